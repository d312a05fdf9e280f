import sys, time; sys.path.insert(0, '.')
import torch, numpy as np
from torch.profiler import profile, ProfilerActivity
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
c = nbg.nbg_init(nbg.NONBLOCKING, 0, torch.cuda.current_stream().cuda_stream)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
rp_p = torch.from_numpy(rp).pin_memory(); ci_p = torch.from_numpy(ci).pin_memory(); dg_p = torch.from_numpy(d).pin_memory()
out = torch.empty(n, dtype=torch.float32).pin_memory()
def one():
    A2 = nbg.nbg_matrix_from_csr(c, n, n, rp_p.numpy(), ci_p.numpy(), type=nbg.FP32)
    d2 = nbg.nbg_vector_from_dense(c, nbg.INT32, dg_p.numpy())
    r, s, _ = nbg.nbg_pagerank(c, A2, d2, alpha=0.85, tol=1e-6, itermax=100, type=nbg.FP32)
    nbg.nbg_vector_export_dense(c, r, out.numpy())
    for h in (r, d2): nbg.nbg_vector_free(c, h)
    nbg.nbg_matrix_free(c, A2)
one(); one(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    one(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs[:60]:
    print(f"{(e.time_range.start - t0)/1e3:9.3f} ms {e.time_range.elapsed_us()/1e3:8.3f} ms  {e.name[:90]}")
