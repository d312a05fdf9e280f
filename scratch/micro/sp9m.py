import sys, os, ctypes, time; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libsp9.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
P = ctypes.c_void_p
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
t0 = time.time()
order = np.argsort(-d.astype(np.int64), kind='stable'); cperm = np.empty(n, np.int64); cperm[order] = np.arange(n)
ncols = int((d > 0).sum())
g1 = (cperm[ci] + 1).astype(np.int32)
lens = np.diff(rp).astype(np.int64)
ng = (lens + 3) // 4
grp = np.r_[0, np.cumsum(ng)]
cg = np.zeros(int(grp[-1]) * 4, np.int32)
row = np.repeat(np.arange(n), lens); j = np.arange(len(ci)) - rp[row]
cg[4 * grp[row] + j] = g1
LONGG = 512; CHG = 512              # long rows: > 2048 entries; chunks of 512 groups
tiles = []; i = 0
while i < n:
    if ng[i] > LONGG: i += 1; continue
    st = i; nz = 0
    while i < n and i - st < 32:
        l2 = ng[i]
        if l2 > LONGG: break
        if i > st and nz + l2 > 512: break
        nz += l2; i += 1
    tiles.append((st, i))
tiles = np.array(tiles, np.int32)
lr = np.flatnonzero(ng > LONGG)
chunks = []; longs = []; tot = 0
for jj, rw in enumerate(lr):
    g0, g1_ = grp[rw], grp[rw + 1]; nch = (g1_ - g0 + CHG - 1) // CHG
    longs.append((rw, tot, nch, 0))
    for u in range(nch):
        gb = g0 + u * CHG; chunks.append((jj, gb & 0xffffffff, gb >> 32, min(CHG, g1_ - gb)))
    tot += nch
chunks = np.array(chunks, np.int64).astype(np.uint32).view(np.int32).reshape(-1, 4); longs = np.array(longs, np.int32)
print("plan", time.time() - t0, "tiles", len(tiles), "chunks", len(chunks), "groups", grp[-1], "pad", grp[-1] * 4 / len(ci), flush=True)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
y = np.random.rand(n).astype(np.float32)
yg1 = np.zeros(ncols + 1, np.float32); yg1[cperm[d > 0] + 1] = y[d > 0]
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = cs_[rp[1:]] - cs_[rp[:-1]]
ttiles, tch, tlo, tgrp, tcg, tyg = T(tiles), T(chunks), T(longs), T(grp.astype(np.int64)), T(cg), T(yg1)
counters = torch.zeros(len(longs) + 1, dtype=torch.int32, device='cuda'); partials = torch.zeros(len(chunks) + 1, dtype=torch.float64, device='cuda')
tt = torch.rand(n, device='cuda'); dinv = torch.rand(n, device='cuda'); gpos = T(np.zeros(n, np.int32))
r = torch.zeros(n, device='cuda'); yn = torch.zeros(ncols + 1, device='cuda')
dsum = torch.zeros(1, dtype=torch.float64, device='cuda'); ctr = torch.zeros(2, dtype=torch.int32, device='cuda')
for mode in (0, 1, 2, 3):
  B = 1
  if True:
    for hc in (32768,):
        f = lambda: L_.sp9_run(mode, B, ctypes.c_longlong(len(tiles)), ctypes.c_longlong(len(chunks)), P(ttiles.data_ptr()), P(tch.data_ptr()), P(tlo.data_ptr()),
                               P(counters.data_ptr()), P(partials.data_ptr()), P(tgrp.data_ptr()), P(tcg.data_ptr()), P(tyg.data_ptr()), hc,
                               P(tt.data_ptr()), P(dinv.data_ptr()), P(gpos.data_ptr()), ctypes.c_float(0.0), P(r.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()), P(ctr.data_ptr()))
        r.zero_(); assert f() == 0; torch.cuda.synchronize()
        err = np.max(np.abs(r.cpu().numpy() - ref) / np.maximum(ref, 1e-3))
        tm = timeit(f)
        print(f"mode {mode} hc {hc}: {tm:.1f} us  GTEPS {len(ci) / tm / 1e3:.0f}  maxrel {err:.2e}", flush=True)
