import sys, os, ctypes, time
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg

torch.cuda.set_device(0)
L = ctypes.CDLL(os.path.abspath('scratch/micro/libtp7.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
n = rp.shape[0] - 1
nnz = ci.shape[0]
t0 = time.time()
cnt = np.bincount(ci, minlength=n)
order = np.argsort(-cnt, kind='stable')
newid = np.empty(n, np.int64); newid[order] = np.arange(n)
ncols_g = int((cnt > 0).sum())
cg = newid[ci]
row = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
S = int(os.environ.get('TP7_S', 32767))
WR = 2048
blk = cg // S
key = blk * n + row
srt = np.argsort(key, kind='stable')
sb, sr, sl = blk[srt], row[srt], (cg - blk * S)[srt]
del key
nb = int(sb.max()) + 1
end = np.ones(nnz, bool)
end[:-1] = (sb[1:] != sb[:-1]) | (sr[1:] != sr[:-1])
eb = np.bincount(sb, minlength=nb)
estart = np.concatenate([[0], np.cumsum(eb)])
padded = (eb + WR - 1) // WR * WR
pstart = np.concatenate([[0], np.cumsum(padded)])
tot = int(pstart[-1])
pos = pstart[sb] + (np.arange(nnz) - estart[sb])
stream = np.full(tot, 0x7fff, np.uint16)
stream[pos] = (sl | (end.astype(np.int64) << 15)).astype(np.uint16)
stream[WR - 1::WR] |= 0x8000
flag = (stream & 0x8000) != 0
csum = np.cumsum(flag)
npieces = int(csum[-1])
prow_full = np.full(tot, -1, np.int64); prow_full[pos] = sr
fpos = np.nonzero(flag)[0]
piece_row = prow_full[fpos]
real = np.nonzero(piece_row >= 0)[0]                 # piece ordinals with a row
ordr = real[np.argsort(piece_row[real], kind='stable')]
rp2 = np.concatenate([[0], np.cumsum(np.bincount(piece_row[real], minlength=n))]).astype(np.int64)
nr = tot // WR
wblk = (np.searchsorted(pstart, np.arange(nr) * WR, side='right') - 1).astype(np.int32)
pbase = np.concatenate([[0], csum[WR - 1::WR][:-1]]).astype(np.int64)
ncta = 148
cta = (np.arange(ncta + 1) * nr // ncta).astype(np.int32)
print(f"n {n} nnz {nnz} blocks {nb} stream {tot} (+{tot - nnz} pad) pieces {npieces} real {real.shape[0]} host {time.time() - t0:.1f}s", flush=True)
x = np.random.default_rng(1).random(ncols_g).astype(np.float32)
xe = np.zeros(nb * S + 1, np.float32); xe[:ncols_g] = x
yexp = np.bincount(row, weights=xe[cg].astype(np.float64), minlength=n)

dE = torch.from_numpy(stream.view(np.int16)).cuda()
dX = torch.from_numpy(x).cuda()
dwb = torch.from_numpy(wblk).cuda(); dcta = torch.from_numpy(cta).cuda(); dpb = torch.from_numpy(pbase).cuda()
drp2 = torch.from_numpy(rp2).cuda(); drpc = torch.from_numpy(ordr.astype(np.int32)).cuda()
dy = torch.empty(n, dtype=torch.float32, device='cuda')
Pp = ctypes.c_void_p


def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


for accd in (1, 0):
    dP = torch.zeros(npieces, dtype=torch.float64 if accd else torch.float32, device='cuda')
    for nt in (768, 1024):
        f1 = lambda: L.tp7_p1(accd, nt, Pp(dE.data_ptr()), Pp(dX.data_ptr()), Pp(dwb.data_ptr()), Pp(dcta.data_ptr()), ncta,
                              Pp(dpb.data_ptr()), Pp(dP.data_ptr()), S, ctypes.c_longlong(ncols_g))
        assert f1() == 0
        torch.cuda.synchronize()
        f2 = lambda: L.tp7_p2(accd, ctypes.c_longlong(n), Pp(drp2.data_ptr()), Pp(drpc.data_ptr()), Pp(dP.data_ptr()), Pp(dy.data_ptr()))
        assert f2() == 0
        torch.cuda.synchronize()
        y = dy.cpu().numpy().astype(np.float64)
        err = np.max(np.abs(y - yexp) / np.maximum(np.abs(yexp), 1e-30))
        t1 = timeit(f1); t2 = timeit(f2)
        print(f"acc {'f64' if accd else 'f32'} nt {nt}: phase1 {t1:.1f} us  phase2 {t2:.1f} us  total {t1 + t2:.1f}  max rel err {err:.2e}", flush=True)
