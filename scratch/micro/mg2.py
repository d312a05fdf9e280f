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
cin = torch.from_numpy(ci.astype(np.int32)).cuda()
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
def run(mode, hc, smem, ci_=cig, label=""):
    f = lambda: L.mg_run(mode, 1, 148, P(ci_.data_ptr()), ctypes.c_longlong(nnz), P(x.data_ptr()), hc, P(out.data_ptr()), smem)
    rc = f(); torch.cuda.synchronize()
    if rc: print("rc", rc); return
    t = timeit(f)
    print(f"{label} mode {mode} hc {hc} smem {smem//1024}KB: {t:.1f} us  Ggathers/s {nnz / t / 1e3:.0f}", flush=True)
run(0, 0, 0, cin, "natural")
run(0, 0, 0)
for sm in (8, 32, 64, 100, 132, 164, 196):
    run(0, 0, sm * 1024, label="carve")
for hc in (4096, 8192, 16384, 24576, 32768, 40960, 51200):
    run(1, hc, hc * 4)
for hc in (8192, 16384, 32768, 57344, 100000, 200000, 400000):
    run(3, hc, 0)
    run(4, hc, 0)
