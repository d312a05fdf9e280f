# hybrid two-phase v8 micro (tp8.cu): K_A over dense (blocks < K, shared-memory slices) and cold
# ranges, K_B combine per row.  Checks y against numpy and times both kernels.
import sys, os, ctypes, time
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg

torch.cuda.set_device(0)
L = ctypes.CDLL(os.path.abspath('scratch/micro/libtp8.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
nbg.nbg_finalize(c)
n = rp.shape[0] - 1
nnz = ci.shape[0]
cnt = np.bincount(ci, minlength=n)
order = np.argsort(-cnt, kind='stable')
newid = np.empty(n, np.int64); newid[order] = np.arange(n)
ncols_g = int((cnt > 0).sum())
cg = newid[ci]
row = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
S = 32764
blk = cg // S
x = np.random.default_rng(1).random(ncols_g + 16).astype(np.float32)
x[ncols_g:] = 0
yexp = np.bincount(row, weights=x[cg].astype(np.float64), minlength=n)
Pp = ctypes.c_void_p
NT = int(os.environ.get("TP8_NT", 768))
COLD_W = float(os.environ.get("TP8_COLDW", 2.0))

for K in [int(k) for k in os.environ.get("TP8_K", "8").split(",")]:
    t0 = time.time()
    dmask = blk < K
    # ---- dense stream: (block, row, position) order, u16 local index | flag, lane runs of 64
    di = np.nonzero(dmask)[0]
    o1 = np.argsort(blk[di] * n + row[di], kind='stable')
    di = di[o1]
    db, dr, dl = blk[di], row[di], cg[di] - blk[di] * S
    m = di.shape[0]
    end = np.ones(m, bool)
    end[:-1] = (db[1:] != db[:-1]) | (dr[1:] != dr[:-1])
    nb = K
    eb = np.bincount(db, minlength=nb)
    estart = np.concatenate([[0], np.cumsum(eb)])
    padded = (eb + 2047) // 2048 * 2048
    pstart = np.concatenate([[0], np.cumsum(padded)])
    tot = int(pstart[-1])
    pos = pstart[db] + (np.arange(m) - estart[db])
    st = np.full(tot, 0x7fff, np.uint16)
    st[pos] = (dl | (end.astype(np.int64) << 15)).astype(np.uint16)
    st[63::64] |= 0x8000
    fl = (st & 0x8000) != 0
    prow = np.full(tot, -1, np.int64); prow[pos] = dr
    ndp = int(fl.sum())
    dpiece_row = prow[fl]
    dcs = np.cumsum(fl)
    dlbase = np.concatenate([[0], dcs[63::64][:-1]]).astype(np.int64)
    ndr = tot // 2048
    rblk = np.repeat(np.arange(nb), padded // 2048).astype(np.int32)
    bnext = np.repeat(pstart[1:] // 2048, padded // 2048).astype(np.int32)
    Ephys = st.reshape(ndr, 32, 8, 8).transpose(0, 2, 1, 3).reshape(-1).copy()
    # ---- cold stream: row-major int32 gather index | flag, lane runs of 32
    ck = np.nonzero(~dmask)[0]                  # already row-major (CSR order)
    mc = ck.shape[0]
    cr = row[ck]
    cend = np.ones(mc, bool)
    cend[:-1] = cr[1:] != cr[:-1]
    ctot = (mc + 1023) // 1024 * 1024
    cs = np.zeros(ctot, np.uint32)
    cs[:mc] = cg[ck].astype(np.uint32) | (cend.astype(np.uint32) << 31)
    cs[31::32] |= np.uint32(1 << 31)
    cfl = (cs >> 31) == 1
    crow = np.full(ctot, -1, np.int64); crow[:mc] = cr
    ncp = int(cfl.sum())
    cpiece_row = crow[cfl]
    ccs = np.cumsum(cfl)
    clbase = ndp + np.concatenate([[0], ccs[31::32][:-1]]).astype(np.int64)
    ncr = ctot // 1024
    Cphys = cs.reshape(ncr, 32, 8, 4).transpose(0, 2, 1, 3).reshape(-1).copy()
    lbase = np.concatenate([dlbase, clbase, [ndp + ncp]]).astype(np.int32)
    npieces = ndp + ncp
    # ---- CTA spans balanced by cost
    cost = np.concatenate([np.full(ndr, 2048.0), np.full(ncr, 1024.0 * COLD_W)])
    pre = np.concatenate([[0], np.cumsum(cost)])
    ncta = 148
    cta = np.searchsorted(pre, pre[-1] * np.arange(ncta + 1) / ncta).astype(np.int32)
    cta[-1] = ndr + ncr
    # ---- K_B lists: pieces per row, dense (block order) then cold
    prow_all = np.concatenate([dpiece_row, cpiece_row])
    real = np.nonzero(prow_all >= 0)[0]
    lst = real[np.argsort(prow_all[real], kind='stable')].astype(np.int32)
    rp3 = np.concatenate([[0], np.cumsum(np.bincount(prow_all[real], minlength=n))]).astype(np.int64)
    print(f"K {K}: dense {m} ({m / nnz:.3f}) ranges {ndr}, cold {mc} ranges {ncr}, pieces {ndp}+{ncp}, host {time.time() - t0:.1f}s",
          flush=True)
    g = lambda a: torch.from_numpy(a).cuda()
    dE, dC, dX = g(Ephys.view(np.int16)), g(Cphys.view(np.int32)), g(x)
    drb, dbn, dcta, dlb = g(rblk), g(bnext), g(cta), g(lbase)
    dP = torch.zeros(npieces + 1, dtype=torch.float32, device='cuda')
    drp3, dlst = g(rp3), g(lst)
    dy = torch.empty(n, dtype=torch.float32, device='cuda')
    fa = lambda r=1, tim=0: L.tp8_a(r, NT, Pp(dE.data_ptr()), Pp(dC.data_ptr()), Pp(dX.data_ptr()), Pp(drb.data_ptr()),
                                    Pp(dbn.data_ptr()), Pp(dcta.data_ptr()), ncta, Pp(dlb.data_ptr()), Pp(dP.data_ptr()), S,
                                    ctypes.c_longlong(ncols_g), ndr, Pp(tim))
    fb = lambda r=1: L.tp8_b(r, ctypes.c_longlong(n), Pp(drp3.data_ptr()), Pp(dlst.data_ptr()), Pp(dP.data_ptr()), Pp(dy.data_ptr()))
    assert fa() == 0 and fb() == 0
    torch.cuda.synchronize()
    y = dy.cpu().numpy().astype(np.float64)
    err = np.max(np.abs(y - yexp) / np.maximum(np.abs(yexp), 1e-30))

    def tm(f):
        f(3); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(20); e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 20 * 1000

    ta, tb = tm(fa), tm(fb)
    tim = torch.zeros(4 * ncta, dtype=torch.int64, device='cuda')
    fa(1, tim.data_ptr()); torch.cuda.synchronize()
    tt = tim.cpu().numpy().reshape(-1, 4)
    t00 = tt[:, 0].min()
    en = (tt[:, 1] - t00) / 1e3; sl = tt[:, 2] / 1e3
    kind = np.where(cta[:-1] < ndr, 0, 1)
    print(f"  K_A {ta:.1f} us  K_B {tb:.1f} us  total {ta + tb:.1f}  err {err:.1e} | cta end min/med/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}"
          f" slice med/max {np.median(sl):.1f}/{sl.max():.1f}; dense-start ctas end med {np.median(en[kind == 0]):.1f}, cold-start {np.median(en[kind == 1]) if (kind == 1).any() else 0:.1f}",
          flush=True)
