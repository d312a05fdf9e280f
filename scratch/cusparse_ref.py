import sys; sys.path.insert(0,'.')
import torch, numpy as np, time
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
n = rp.shape[0]-1
crow = torch.from_numpy(rp).cuda(); col = torch.from_numpy(ci.astype(np.int64)).cuda()
vals = torch.ones(ci.shape[0], device='cuda', dtype=torch.float32)
M = torch.sparse_csr_tensor(crow, col, vals, size=(n, n))
x = torch.rand(n, 1, device='cuda')
for _ in range(3): y = torch.sparse.mm(M, x)
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): y = torch.sparse.mm(M, x)
e1.record(); torch.cuda.synchronize()
print("cusparse spmm(n x 1) fp32 us/iter", e0.elapsed_time(e1)/20*1000)
# int32 indices
M32 = torch.sparse_csr_tensor(crow.int(), col.int(), vals, size=(n, n))
for _ in range(3): y = torch.sparse.mm(M32, x)
torch.cuda.synchronize(); e0.record()
for _ in range(20): y = torch.sparse.mm(M32, x)
e1.record(); torch.cuda.synchronize()
print("cusparse int32 us/iter", e0.elapsed_time(e1)/20*1000)
# simple gather bandwidth test: y = x[colidx] sum-free gather
ci_t = torch.from_numpy(ci).cuda().long()
xf = torch.rand(n, device='cuda')
for _ in range(3): g = xf[ci_t]
torch.cuda.synchronize(); e0.record()
for _ in range(10): g = xf[ci_t]
e1.record(); torch.cuda.synchronize()
print("torch gather x[colidx] us", e0.elapsed_time(e1)/10*1000)
