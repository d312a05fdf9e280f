import sys, os, ctypes, time; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L = ctypes.CDLL(os.path.abspath('scratch/micro/libmg.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
order = np.argsort(-d.astype(np.int64), kind='stable'); perm = np.empty(n, np.int64); perm[order] = np.arange(n)
cig = torch.from_numpy(perm[ci].astype(np.int32)).cuda()
nnz = cig.numel()
x = torch.rand(n, device='cuda')
out = torch.empty(148 * 1024, device='cuda')
P = ctypes.c_void_p
def ev(): return torch.cuda.Event(enable_timing=True)
def timeit(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0, e1 = ev(), ev(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
SM = 200 * 1024
for mode, cs in ((0, 1), (1, 1), (2, 2), (2, 4), (2, 8), (2, 16)):
    smem = 0 if mode == 0 else SM
    mc = L.mg_maxclusters(mode, cs, smem)
    print("mode", mode, "cs", cs, "max active clusters", mc, "SMs", mc * cs, flush=True)
    if mc <= 0: continue
    hcs = [0] if mode == 0 else ([51200] if mode == 1 else [cs * 51200 // 2, cs * 51200])
    for hc in hcs:
        f = lambda: L.mg_run(mode, cs, mc, P(cig.data_ptr()), ctypes.c_longlong(nnz), P(x.data_ptr()), hc, P(out.data_ptr()), smem)
        rc = f(); torch.cuda.synchronize()
        if rc: print("launch rc", rc); continue
        t = timeit(f)
        print(f"  hc {hc}: {t:.1f} us  hit {(cig < hc).float().mean().item():.3f}  Ggathers/s {nnz / t / 1e3:.0f}", flush=True)
for cs in (1, 2, 4, 8, 16):
    per = 51200
    mc = L.mg_maxclusters(2, cs, per * 4) if cs > 1 else 148
    iters = 2000
    f = lambda: L.mg_rand(cs, mc, per, iters, P(out.data_ptr()))
    rc = f(); torch.cuda.synchronize()
    if rc: print("rand rc", rc, cs); continue
    t = timeit(f, 5)
    tot = mc * cs * 1024 * iters * 4
    print(f"rand cs {cs}: {t:.1f} us, {tot / t / 1e3:.0f} G gathers/s, per SM per cycle {tot / (mc * cs) / (t * 1e-6) / 1.965e9:.2f}", flush=True)
