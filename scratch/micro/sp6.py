import sys, os, ctypes, time; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libsp6.so'))
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
order = np.argsort(-d.astype(np.int64), kind='stable'); cperm = np.empty(n, np.int64); cperm[order] = np.arange(n)
ncols = int((d > 0).sum())
cig = cperm[ci].astype(np.int32)
LONG = 2048; CH = 2048
lens = np.diff(rp)
tiles = []; i = 0
while i < n:
    if lens[i] > LONG: i += 1; continue
    st = i; nz = 0
    while i < n and i - st < 32:
        l2 = lens[i]
        if l2 > LONG: break
        if i > st and nz + l2 > 2048: break
        nz += l2; i += 1
    tiles.append((st, i))
tiles = np.array(tiles, np.int32)
lr = np.flatnonzero(lens > LONG)
chunks = []; longs = []; tot = 0
for j, row in enumerate(lr):
    p0, p1 = rp[row], rp[row + 1]; nch = (p1 - p0 + CH - 1) // CH
    longs.append((row, tot, nch, 0))
    for q in range(nch):
        pb = p0 + q * CH; chunks.append((j, pb & 0xffffffff, pb >> 32, min(CH, p1 - pb)))
    tot += nch
chunks = np.array(chunks, np.int64).astype(np.uint32).view(np.int32).reshape(-1, 4); longs = np.array(longs, np.int32)
print("tiles", len(tiles), "chunks", len(chunks), "longs", len(longs), flush=True)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ttiles, tchunks, tlongs = T(tiles), T(chunks), T(longs)
counters = torch.zeros(len(longs) + 1, dtype=torch.int32, device='cuda'); partials = torch.zeros(len(chunks) + 1, dtype=torch.float64, device='cuda')
trp = T(rp.astype(np.int64)); tci = T(np.r_[cig, np.zeros(64, np.int32)])
y = np.random.rand(n).astype(np.float32)
yg = np.zeros(ncols, np.float32); yg[cperm[d > 0]] = y[d > 0]
tyg = T(yg)
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = cs_[rp[1:]] - cs_[rp[:-1]]
tt = torch.rand(n, device='cuda'); dinv = torch.rand(n, device='cuda'); gpos = torch.full((n,), -1, dtype=torch.int32, device='cuda')
r = torch.zeros(n, device='cuda'); yn = torch.zeros(ncols, device='cuda')
dsum = torch.zeros(1, dtype=torch.float64, device='cuda'); ctr = torch.zeros(1, dtype=torch.int32, device='cuda')
for E in (4, 8, 16):
    for hc in (0, 32768, 40960):
        f = lambda: L_.sp6_run(E, len(tiles), len(chunks), P(ttiles.data_ptr()), P(tchunks.data_ptr()), P(tlongs.data_ptr()), P(counters.data_ptr()),
                               P(partials.data_ptr()), P(trp.data_ptr()), P(tci.data_ptr()), ctypes.c_longlong(len(ci)), P(tyg.data_ptr()), hc,
                               P(tt.data_ptr()), P(dinv.data_ptr()), P(gpos.data_ptr()), ctypes.c_float(0.0), P(r.data_ptr()), P(yn.data_ptr()),
                               P(dsum.data_ptr()), P(ctr.data_ptr()))
        r.zero_(); assert f() == 0; torch.cuda.synchronize()
        err = np.max(np.abs(r.cpu().numpy() - ref) / np.maximum(ref, 1e-3))
        t = timeit(f)
        print(f"E {E} hc {hc}: {t:.1f} us  GTEPS {len(ci) / t / 1e3:.0f}  maxrel {err:.2e}", flush=True)
