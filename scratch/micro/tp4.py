import sys, os, ctypes, time; sys.path.insert(0, '.'); sys.path.insert(0, 'scratch/micro')
import torch, numpy as np, tp4plan
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libtp4.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
P = ctypes.c_void_p
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
t0 = time.time(); p = tp4plan.build(rp, ci, d); print("plan", time.time() - t0, "pieces", p['npieces'], "slices", p['nsl'], "tiles", p['ntiles'], flush=True)
T = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in p.items() if isinstance(v, np.ndarray)}
y = np.random.rand(n).astype(np.float32)
yg = np.zeros(p['ncols'] + 64, np.float32); yg[p['perm'][d > 0]] = y[d > 0]
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = cs_[rp[1:]] - cs_[rp[:-1]]
tyg = torch.from_numpy(yg).cuda()
part = torch.zeros(p['npieces'] + 1, dtype=torch.float64, device='cuda')
tt = torch.rand(n, device='cuda'); dinv = torch.rand(n, device='cuda'); gpos = torch.full((n,), -1, dtype=torch.int32, device='cuda')
r = torch.zeros(n, device='cuda'); yn = torch.zeros(p['ncols'] + 1, device='cuda'); dsum = torch.zeros(1, dtype=torch.float64, device='cuda')
dbg = torch.zeros(148 * 4, dtype=torch.int64, device='cuda')
for nt in (768,):
    f1 = lambda: L_.tp4_p1(nt, P(T['cta'].data_ptr()), P(T['sl_blk'].data_ptr()), P(T['sl_off'].data_ptr()), P(T['sl_Ls'].data_ptr()),
                           P(T['spbase'].data_ptr()), P(T['lcol'].data_ptr()), P(T['pos2'].data_ptr()), P(tyg.data_ptr()), p['S'], p['ncols'], P(part.data_ptr()), P(dbg.data_ptr()))
    for grid in (148 * 8,):
        f2 = lambda: L_.tp4_p2(grid, p['ntiles'], P(T['tinfo'].data_ptr()), P(T['rslot'].data_ptr()), P(T['qidx'].data_ptr()), P(part.data_ptr()),
                               P(tt.data_ptr()), P(dinv.data_ptr()), P(gpos.data_ptr()), ctypes.c_float(0.0), P(r.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()))
        r.zero_(); assert f1() == 0; torch.cuda.synchronize(); assert f2() == 0; torch.cuda.synchronize()
        err = np.max(np.abs(r.cpu().numpy() - ref) / np.maximum(ref, 1e-3))
        t1 = timeit(f1); t2 = timeit(f2); t12 = timeit(lambda: (f1(), f2()))
        print(f"nt {nt}: p1 {t1:.1f} us  p2 {t2:.1f} us  both {t12:.1f} us  GTEPS {len(ci) / t12 / 1e3:.0f}  maxrel {err:.2e}", flush=True)

D = dbg.cpu().numpy().reshape(148, 4)
o = np.argsort(-D[:, 0])
for i in o[:10]: print("cta", i, "cycles", D[i, 0], "blocks", D[i, 1], "slices", D[i, 2], "first block", D[i, 3])
print("median cycles", np.median(D[:, 0]))
# slices per block and entries
sb = p['sl_blk']; print("slices in block 0..5:", [int((sb == b).sum()) for b in range(6)])
