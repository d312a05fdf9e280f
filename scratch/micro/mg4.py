import sys, os, ctypes; sys.path.insert(0, '.')
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
nnz = cig.numel(); x = torch.rand(n, device='cuda'); out = torch.empty(148 * 1024, device='cuda')
P = ctypes.c_void_p
def timeit(f, reps=10):
    for _ in range(2): f()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
for hc in (0, 32768):
    for mode in (0, 1, 2):
        f = lambda: L.mg_tex(mode, P(cig.data_ptr()), ctypes.c_longlong(nnz), P(x.data_ptr()), ctypes.c_longlong(n), hc, P(out.data_ptr()))
        assert f() == 0
        print(f"hc {hc} mode {mode} ({['ldg','tex','half'][mode]}): {timeit(f):.1f} us (includes texobj create/destroy + sync)", flush=True)
