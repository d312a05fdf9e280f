# two-phase v7 estimate: phase 1 (tp7.cu) on the dense blocks < K, phase 2 = the library's v6 SpMV
# on the residual matrix (row i: its pieces as columns ncols_g + ordinal of V = [x | P], then its cold entries)
import sys, os, ctypes, time
os.environ["NBG_RELABEL"] = "0"
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg

torch.cuda.set_device(0)
L = ctypes.CDLL(os.path.abspath('scratch/micro/libtp7.so'))
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
WR = 2048
blk = cg // S
srt = np.argsort(blk * n + row, kind='stable')
sb, sr, sl, sg = blk[srt], row[srt], (cg - blk * S)[srt], cg[srt]
x = np.random.default_rng(1).random(ncols_g).astype(np.float32)
yexp = np.bincount(row, weights=x[cg].astype(np.float64), minlength=n)
Pp = ctypes.c_void_p


def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


for K in [int(k) for k in os.environ.get("TP7_K", "4,8,12,16,24,64").split(",")]:
    m = int(np.searchsorted(sb, K))              # dense entries: a prefix of the block-sorted order
    db, dr, dl = sb[:m], sr[:m], sl[:m]
    nb = int(db.max()) + 1
    end = np.ones(m, bool)
    end[:-1] = (db[1:] != db[:-1]) | (dr[1:] != dr[:-1])
    eb = np.bincount(db, minlength=nb)
    estart = np.concatenate([[0], np.cumsum(eb)])
    padded = (eb + WR - 1) // WR * WR
    pstart = np.concatenate([[0], np.cumsum(padded)])
    tot = int(pstart[-1])
    pos = pstart[db] + (np.arange(m) - estart[db])
    stream = np.full(tot, 0x7fff, np.uint16)
    stream[pos] = (dl | (end.astype(np.int64) << 15)).astype(np.uint16)
    stream[WR - 1::WR] |= 0x8000
    if os.environ.get("TP7_V3", "1") == "1":
        stream[63::64] |= 0x8000
    flag = (stream & 0x8000) != 0
    csum = np.cumsum(flag)
    npieces = int(csum[-1])
    prow_full = np.full(tot, -1, np.int64); prow_full[pos] = dr
    fpos = np.nonzero(flag)[0]
    piece_row = prow_full[fpos]
    real = np.nonzero(piece_row >= 0)[0]
    nr = tot // WR
    wblk = (np.searchsorted(pstart, np.arange(nr) * WR, side='right') - 1).astype(np.int32)
    pbase = np.concatenate([[0], csum[WR - 1::WR][:-1]]).astype(np.int64)
    ncta = 148
    cta = (np.arange(ncta + 1) * nr // ncta).astype(np.int32)
    # residual matrix: pieces (virtual columns ncols_g + ordinal), then cold entries
    rrow = np.concatenate([piece_row[real], sr[m:]])
    rcol = np.concatenate([ncols_g + real, sg[m:]])
    o2 = np.argsort(rrow, kind='stable')
    rrow, rcol = rrow[o2], rcol[o2]
    rrp = np.concatenate([[0], np.cumsum(np.bincount(rrow, minlength=n))]).astype(np.int64)
    nv = ncols_g + npieces
    lbase = np.concatenate([[0], csum[63::64][:-1]]).astype(np.int32)
    phys = stream.reshape(nr, 32, 8, 8).transpose(0, 2, 1, 3).reshape(-1).copy()   # [range][lane][k][h] -> [range][k][lane][h]
    dE3 = torch.from_numpy(phys.view(np.int16)).cuda()
    dlb = torch.from_numpy(lbase).cuda()
    dE = torch.from_numpy(stream.view(np.int16)).cuda()
    dX = torch.from_numpy(x).cuda()
    dwb = torch.from_numpy(wblk).cuda(); dcta = torch.from_numpy(cta).cuda(); dpb = torch.from_numpy(pbase).cuda()
    dP = torch.zeros(npieces, dtype=torch.float32, device='cuda')
    NT3 = int(os.environ.get("TP7_NT", 768))
    f3 = lambda r=1: L.tp7_p1c(r, NT3, Pp(dE3.data_ptr()), Pp(dX.data_ptr()), Pp(dwb.data_ptr()), Pp(dcta.data_ptr()), ncta,
                               Pp(dlb.data_ptr()), Pp(dP.data_ptr()), S, ctypes.c_longlong(ncols_g), Pp(0))
    f1 = lambda r=1: L.tp7_p1(r, 0, 1024, Pp(dE.data_ptr()), Pp(dX.data_ptr()), Pp(dwb.data_ptr()), Pp(dcta.data_ptr()), ncta,
                          Pp(dpb.data_ptr()), Pp(dP.data_ptr()), S, ctypes.c_longlong(ncols_g))
    assert f1() == 0
    torch.cuda.synchronize()
    if os.environ.get("TP7_V3", "1") == "1":
        f1 = f3
    assert f1() == 0
    f1(3); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); f1(20); e1.record(); torch.cuda.synchronize()
    t1 = e0.elapsed_time(e1) / 20 * 1000
    if os.environ.get("TP7_V3", "1") == "1":
        tim = torch.zeros(4 * ncta, dtype=torch.int64, device='cuda')
        L.tp7_p1c(1, NT3, Pp(dE3.data_ptr()), Pp(dX.data_ptr()), Pp(dwb.data_ptr()), Pp(dcta.data_ptr()), ncta,
                  Pp(dlb.data_ptr()), Pp(dP.data_ptr()), S, ctypes.c_longlong(ncols_g), Pp(tim.data_ptr()))
        tm = tim.cpu().numpy().reshape(-1, 4)
        t0_ = tm[:, 0].min()
        st = (tm[:, 0] - t0_) / 1e3; en = (tm[:, 1] - t0_) / 1e3; sl_ = tm[:, 2] / 1e3
        cb = wblk[cta[:-1]]
        print("  start max %.1f us; end min/med/max %.1f/%.1f/%.1f; slice min/med/max %.1f/%.1f/%.1f" % (st.max(), en.min(), np.median(en), en.max(), sl_.min(), np.median(sl_), sl_.max()))
        for b in range(nb):
            mm = cb == b
            if mm.any(): print("   first-block %d: ctas %d end med %.1f max %.1f" % (b, mm.sum(), np.median(en[mm]), en[mm].max()))
        o_ = np.argsort(-en)[:6]
        print("   slowest ctas", [(int(i), int(tm[i, 3]), round(float(en[i]), 1), int(cta[i + 1] - cta[i])) for i in o_])
    V = np.concatenate([x, dP.cpu().numpy()])
    c2 = nbg.nbg_init(nbg.BLOCKING, 0)
    R = nbg.nbg_matrix_from_csr(c2, n, nv, rrp, rcol.astype(np.int32), type=nbg.FP32)
    u = nbg.nbg_vector_from_dense(c2, nbg.FP32, V)
    y = nbg.nbg_mxv(c2, nbg.FP32, "PLUS", "SECOND", R, u)
    yv = nbg.nbg_vector_export_dense(c2, y)
    err = np.max(np.abs(yv - yexp) / np.maximum(np.abs(yexp), 1e-30))
    nbg.nbg_vector_free(c2, y)
    for _ in range(3):
        nbg.nbg_vector_free(c2, nbg.nbg_mxv(c2, nbg.FP32, "PLUS", "SECOND", R, u))
    nbg.nbg_sync(c2)
    nbg.nbg_set_timing(c2, 1)
    for _ in range(10):
        nbg.nbg_vector_free(c2, nbg.nbg_mxv(c2, nbg.FP32, "PLUS", "SECOND", R, u))
    nbg.nbg_sync(c2)
    ms, k = nbg.nbg_get_timing(c2, "spmv")
    nbg.nbg_finalize(c2)
    print(f"K {K}: dense {m / nnz:.3f} pieces {npieces} residual nnz {rcol.shape[0]} | phase1 {t1:.1f} us  phase2(v6) {ms / k * 1e3:.1f} us"
          f"  total {t1 + ms / k * 1e3:.1f}  err {err:.1e}", flush=True)
