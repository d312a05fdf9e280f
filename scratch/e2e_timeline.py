# device timeline of one e2e step (upload CSR from pinned host, plan, PageRank, export): which
# kernels / copies fill the ~12 ms
import sys; sys.path.insert(0, '.')
import torch
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
    r, s, _ = nbg.nbg_pagerank(c, A2, d2, tol=1e-6, itermax=100)
    nbg.nbg_vector_export_dense(c, r, out.numpy())
    for h in (r, d2): nbg.nbg_vector_free(c, h)
    nbg.nbg_matrix_free(c, A2)
for _ in range(3): one()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    one(); torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
agg = {}
for e in evs:
    k = e.name[:90]
    if k.startswith("nbg_spmv"): k = "nbg_spmv (sweeps)"
    agg[k] = agg.get(k, 0.0) + e.time_range.elapsed_us()
print(f"span {(evs[-1].time_range.end - t0)/1e3:.2f} ms, busy {sum(agg.values())/1e3:.2f} ms")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{v/1e3:8.3f} ms  {k}")
prev = None
print("-- gaps > 50 us:")
for e in evs:
    if prev is not None and e.time_range.start - prev > 50:
        print(f"  gap {(e.time_range.start - prev)/1e3:.3f} ms before {e.name[:50]} at {(e.time_range.start - t0)/1e3:.2f} ms")
    prev = max(prev or 0, e.time_range.end)
