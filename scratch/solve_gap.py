# where the ~0.3 ms per solve outside the sweep kernels goes: host vs device timeline of one solve
import sys, time; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
c = nbg.nbg_init(nbg.NONBLOCKING, 0, st.cuda_stream)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
for _ in range(3):
    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=1e-6, itermax=100); nbg.nbg_vector_free(c, r)
torch.cuda.synchronize()
for it in range(5):
    nbg.nbg_set_timing(c, 1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=1e-6, itermax=100)
    t1 = time.perf_counter(); e1.record(st); torch.cuda.synchronize(); t2 = time.perf_counter()
    sp, ns = nbg.nbg_get_timing(c, "spmv"); ew, ne = nbg.nbg_get_timing(c, "ewise")
    nbg.nbg_set_timing(c, 0)
    print(f"host call {1e3*(t1-t0):.3f} ms, device span {e0.elapsed_time(e1):.3f} ms, spmv {sp:.3f} ms ({ns}), ewise {ew:.3f} ms ({ne}), sweeps {s}")
    nbg.nbg_vector_free(c, r)
