# e2e breakdown on the bench's e2e input (the per-rank data plane's relabelled CSR at P = 1):
# upload, first solve (plan build + solve), second solve (solve only)
import sys, time; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
c = nbg.nbg_init(nbg.NONBLOCKING, 0, torch.cuda.current_stream().cuda_stream)
A, deg, cuts, ncg = nbg.nbg_dist_graph_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1, nranks=1, bytes_per_row=20)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
rp_p = torch.from_numpy(rp).pin_memory(); ci_p = torch.from_numpy(ci).pin_memory(); dg_p = torch.from_numpy(d).pin_memory()
out = torch.empty(n, dtype=torch.float32).pin_memory()
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    A2 = nbg.nbg_matrix_from_csr(c, n, n, rp_p.numpy(), ci_p.numpy(), type=nbg.FP32)
    d2 = nbg.nbg_vector_from_dense(c, nbg.INT32, dg_p.numpy())
    nbg.nbg_sync(c); t1 = time.perf_counter()
    r, s, _ = nbg.nbg_pagerank(c, A2, d2, alpha=0.85, tol=1e-6, itermax=100, type=nbg.FP32)
    nbg.nbg_sync(c); t2 = time.perf_counter()
    nbg.nbg_vector_export_dense(c, r, out.numpy()); t3 = time.perf_counter()
    r2, s2, _ = nbg.nbg_pagerank(c, A2, d2, alpha=0.85, tol=1e-6, itermax=100, type=nbg.FP32)
    nbg.nbg_sync(c); t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms  first solve (plan + solve) {1e3*(t2-t1):.2f} ms  export {1e3*(t3-t2):.2f} ms  second solve {1e3*(t4-t3):.2f} ms  sweeps {s}", flush=True)
    for h in (r, r2, d2): nbg.nbg_vector_free(c, h)
    nbg.nbg_matrix_free(c, A2)
