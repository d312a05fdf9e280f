import sys, os, ctypes, time; sys.path.insert(0, '.'); sys.path.insert(0, 'scratch/micro')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libbs.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
P = ctypes.c_void_p
def ev(): return torch.cuda.Event(enable_timing=True)
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0, e1 = ev(), ev(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
LMAX = 2048
t0 = time.time()
order = np.argsort(-d.astype(np.int64), kind='stable'); cperm = np.empty(n, np.int64); cperm[order] = np.arange(n)
ncols = int((d > 0).sum())
g = cperm[ci] + 1                                     # gather layout index, 0 = zero column
lens = np.diff(rp)
short = lens <= LMAX
rowP = np.argsort(-np.where(short, lens, 0), kind='stable')     # long rows treated as empty here (timed separately)
Ls_row = np.where(short, lens, 0)[rowP]
nsl = (n + 31) // 32
Lpad = np.zeros(nsl * 32, np.int64); Lpad[:n] = Ls_row
sL = Lpad.reshape(nsl, 32).max(1)
soff = np.r_[0, np.cumsum(32 * sL)][:-1]
idx = np.zeros(int(32 * sL.sum()), np.uint32)
# fill: for P-position q (row rowP[q]) entries k < len
q = np.repeat(np.arange(n), Ls_row)
kk = np.arange(len(q)) - np.repeat(np.cumsum(Ls_row) - Ls_row, Ls_row)
rows = rowP[q]
idx[soff[q // 32] + 32 * kk + (q % 32)] = g[rp[rows] + kk]
print("plan", time.time() - t0, "slices", nsl, "idx entries", len(idx), "nnz short", int(Ls_row.sum()), flush=True)
y = np.random.rand(n).astype(np.float32)
yg = np.zeros(ncols + 1, np.float32); yg[cperm[d > 0] + 1] = y[d > 0]
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = cs_[rp[1:]] - cs_[rp[:-1]]; ref[~short] = 0
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
tsoff, tsL, tidx, tyg = T(soff.astype(np.int32)), T(sL.astype(np.int32)), T(idx), T(yg)
tP = torch.rand(nsl * 32, device='cuda'); dP = torch.rand(nsl * 32, device='cuda')
gP = torch.zeros(nsl * 32, dtype=torch.int32, device='cuda')
rPt = torch.zeros(nsl * 32, device='cuda'); yn = torch.zeros(ncols + 1, device='cuda')
dsum = torch.zeros(1, dtype=torch.float64, device='cuda'); ctr = torch.zeros(1, dtype=torch.int32, device='cuda')
for U in (4, 8, 16):
    for hc in (0, 16384, 32768, 40960):
        f = lambda: L_.bs_sp8(U, 148, nsl, P(tsoff.data_ptr()), P(tsL.data_ptr()), P(tidx.data_ptr()), P(tyg.data_ptr()), hc,
                              P(tP.data_ptr()), P(dP.data_ptr()), P(gP.data_ptr()), ctypes.c_float(0.0), P(rPt.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()), P(ctr.data_ptr()))
        assert f() == 0; torch.cuda.synchronize()
        got = np.zeros(n); got[rowP] = rPt.cpu().numpy()[:n]
        err = np.max(np.abs(got - ref) / np.maximum(ref, 1e-3))
        t = timeit(f)
        print(f"U {U} hc {hc}: {t:.1f} us (short rows only: {Ls_row.sum()/t/1e3:.0f} GTEPS)  maxrel {err:.2e}", flush=True)
