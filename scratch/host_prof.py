"""C1 host-path profile: wall time per sweep of a fixed-count solve (timing off) vs its device
time, and the planner's phase split (run with NBG_PLAN_PROFILE=1)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
c = nbg.nbg_init(nbg.NONBLOCKING, 0, st.cuda_stream)
scale = int(os.environ.get("SCALE", "10"))
T = nbg.FP64 if os.environ.get("T", "fp64") == "fp64" else nbg.FP32
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, scale, 8, 1)
K = 20
def solve():
    r, s, _ = nbg.nbg_pagerank(c, A, deg, alpha=0.85, tol=-1.0, itermax=K, type=T)
    nbg.nbg_vector_free(c, r)
for _ in range(5): solve()
nbg.nbg_sync(c)
N = int(os.environ.get("N", "300"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(st); t0 = time.perf_counter()
for _ in range(N): solve()
e1.record(st); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"scale {scale}: wall {1e6*(t1-t0)/N/K:.2f} us/sweep  device {1e3*e0.elapsed_time(e1)/N/K:.2f} us/sweep")
nbg.nbg_set_timing(c, 1)
for _ in range(20): solve()
nbg.nbg_sync(c)
for cls in ("spmv", "ewise"):
    ms, cnt = nbg.nbg_get_timing(c, cls)
    if cnt: print(f"  {cls}: {1e3*ms/cnt:.2f} us x {cnt}")
