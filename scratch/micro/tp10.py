# hybrid two-phase v8 micro (tp8.cu): K_A over dense (blocks < K, shared-memory slices) and cold
# ranges, K_B combine per row.  Checks y against numpy and times both kernels.
import sys, os, ctypes, time
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg

torch.cuda.set_device(0)
L = ctypes.CDLL(os.path.abspath('scratch/micro/libtp10.so'))
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
    padded = (eb + 1023) // 1024 * 1024
    pstart = np.concatenate([[0], np.cumsum(padded)])
    tot = int(pstart[-1])
    pos = pstart[db] + (np.arange(m) - estart[db])
    st = np.full(tot, 0x7fff, np.uint16)
    st[pos] = (dl | (end.astype(np.int64) << 15)).astype(np.uint16)
    st[31::32] |= 0x8000
    fl = (st & 0x8000) != 0
    prow = np.full(tot, -1, np.int64); prow[pos] = dr
    ndp = int(fl.sum())
    dpiece_row = prow[fl]
    dcs = np.cumsum(fl)
    dlbase = np.concatenate([[0], dcs[31::32][:-1]]).astype(np.int64)
    ndr = tot // 1024
    rblk = np.repeat(np.arange(nb), padded // 1024).astype(np.int32)
    bnext = np.repeat(pstart[1:] // 1024, padded // 1024).astype(np.int32)
    Ephys = st.reshape(ndr, 32, 4, 8).transpose(0, 2, 1, 3).reshape(-1).copy()
    # ---- cold stream: row-major int32 gather index | flag, lane runs of 32
    ck = np.nonzero(~dmask)[0]                  # already row-major (CSR order)
    mc = ck.shape[0]
    cr = row[ck]
    cend = np.ones(mc, bool)
    cend[:-1] = cr[1:] != cr[:-1]
    ctot = (mc + 511) // 512 * 512
    cs = np.zeros(ctot, np.uint32)
    cs[:mc] = cg[ck].astype(np.uint32) | (cend.astype(np.uint32) << 31)
    cs[15::16] |= np.uint32(1 << 31)
    cfl = (cs >> 31) == 1
    crow = np.full(ctot, -1, np.int64); crow[:mc] = cr
    ncp = int(cfl.sum())
    cpiece_row = crow[cfl]
    ccs = np.cumsum(cfl)
    clbase = ndp + np.concatenate([[0], ccs[15::16][:-1]]).astype(np.int64)
    ncr = ctot // 512
    Cphys = cs.reshape(ncr, 32, 4, 4).transpose(0, 2, 1, 3).reshape(-1).copy()
    lbase = np.concatenate([dlbase, clbase, [ndp + ncp]]).astype(np.int32)
    npieces = ndp + ncp
    # ---- CTA spans balanced by cost
    ncta = 148
    cta = (np.arange(ncta + 1) * ndr // ncta).astype(np.int32)
    ccta = (np.arange(ncta + 1) * ncr // ncta).astype(np.int32)
    MODE = os.environ.get("TP9_MODE", "both")
    if MODE == "dense": ccta[:] = 0
    if MODE == "cold": cta[:] = 0
    # ---- K_B lists: pieces per row, dense (block order) then cold
    prow_all = np.concatenate([dpiece_row, cpiece_row])
    real = np.nonzero(prow_all >= 0)[0]
    nreal = real.shape[0]
    ordr = real[np.argsort(prow_all[real], kind='stable')]
    slot = np.full(npieces, nreal, np.int64); slot[ordr] = np.arange(nreal)
    slot = slot.astype(np.int32)
    items = np.bincount(prow_all[real], minlength=n)
    rs = np.concatenate([[0], np.cumsum(items)]).astype(np.int32)
    lrows = np.nonzero(items > 64)[0].astype(np.int32)
    print(f"long rows {lrows.shape[0]} items in them {items[lrows].sum()} max {items.max()}")
    print(f"K {K}: dense {m} ({m / nnz:.3f}) ranges {ndr}, cold {mc} ranges {ncr}, pieces {ndp}+{ncp}, host {time.time() - t0:.1f}s",
          flush=True)
    g = lambda a: torch.from_numpy(a).cuda()
    dE, dC, dX = g(Ephys.view(np.int16)), g(Cphys.view(np.int32)), g(x)
    drb, dbn, dcta, dlb = g(rblk), g(bnext), g(cta), g(lbase)
    dP = torch.zeros(npieces + 1, dtype=torch.float32, device='cuda')
    if os.environ.get("TP10_NOSLOT") == "1":
        slot = np.arange(npieces, dtype=np.int32)
    dccta, dslot, drs, dlr = g(ccta), g(slot), g(rs), g(lrows)
    dy = torch.empty(n, dtype=torch.float32, device='cuda')
    fa = lambda r=1, tim=0: L.tp8_a(r, NT, Pp(dE.data_ptr()), Pp(dC.data_ptr()), Pp(dX.data_ptr()), Pp(drb.data_ptr()),
                                    Pp(dbn.data_ptr()), Pp(dcta.data_ptr()), ncta, Pp(dlb.data_ptr()), Pp(dP.data_ptr()), S,
                                    ctypes.c_longlong(ncols_g), ndr, Pp(tim), Pp(dccta.data_ptr()), Pp(dslot.data_ptr()))
    fb = lambda r=1: L.tp8_b(r, ctypes.c_longlong(n), Pp(drs.data_ptr()), Pp(dlr.data_ptr()), int(lrows.shape[0]), Pp(dP.data_ptr()), Pp(dy.data_ptr()))
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
    kind = np.zeros(ncta, int)
    rc = np.diff(lbase.astype(np.int64))[::32][:ndr + ncr] if False else (lbase[32::32].astype(np.int64) - lbase[:-1:32].astype(np.int64))
    big = rc[:ndr] > 512
    print("  dense ranges with > 512 pieces:", int(big.sum()), "max pieces", int(rc[:ndr].max()))
    slow = np.argsort(-en)[:6]
    for i in slow:
        a_, b_ = cta[i], cta[i + 1]
        print("   cta", int(i), "end %.1f" % en[i], "dense ranges", int(b_ - a_), "blocks", sorted(set(rblk[a_:b_].tolist())), "big", int(big[a_:b_].sum()))
    print(f"  K_A {ta:.1f} us  K_B {tb:.1f} us  total {ta + tb:.1f}  err {err:.1e} | cta end min/med/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}"
          f" slice med/max {np.median(sl):.1f}/{sl.max():.1f}; dense-start ctas end med {np.median(en[kind == 0]):.1f}, cold-start {np.median(en[kind == 1]) if (kind == 1).any() else 0:.1f}",
          flush=True)
