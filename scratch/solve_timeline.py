# device timeline of back-to-back solves (bench-like): gaps between consecutive kernels
import sys; sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
c = nbg.nbg_init(nbg.NONBLOCKING, 0, st.cuda_stream)
import os
SC = int(os.environ.get('SCALE', '22')); EF = int(os.environ.get('EF', '16'))
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, SC, EF, 1)
TT = nbg.FP64 if os.environ.get('T') == 'fp64' else nbg.FP32
KW = dict(tol=-1.0, itermax=20) if os.environ.get('FIXED') else dict(tol=1e-6, itermax=100)
def solve():
    r, s, h = nbg.nbg_pagerank(c, A, deg, type=TT, **KW); nbg.nbg_vector_free(c, r)
for _ in range(3): solve()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): solve()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and 'Memcpy' not in e.name], key=lambda e: e.time_range.start)
prev = None
for e in evs:
    st_, en = e.time_range.start, e.time_range.end
    gap = (st_ - prev) if prev is not None else 0
    print(f"gap {gap:8.1f} us  dur {en - st_:8.1f} us  {e.name[:50]}")
    prev = en
