import sys, os, ctypes, time; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libsp10.so'))
if len(sys.argv) > 1 and sys.argv[1] == 'small':
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 14, 16, 1)
    LONG = 64
else:
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
    LONG = 2048
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
gi = cperm[ci].astype(np.int32)
lens = np.diff(rp).astype(np.int64)
islong = lens > LONG
ng = (lens + 3) // 4
ngs = np.where(islong, 0, ng); ngl = np.where(islong, ng, 0)
grps = np.r_[0, np.cumsum(ngs)]; grpl = np.r_[0, np.cumsum(ngl)]
cgs = np.full(int(grps[-1]) * 4, -1, np.int32); cgl = np.full(max(int(grpl[-1]) * 4, 4), -1, np.int32)
row = np.repeat(np.arange(n), lens); j = np.arange(len(ci)) - rp[row]
sh = ~islong[row]
cgs[4 * grps[row[sh]] + j[sh]] = gi[sh]
cgl[4 * grpl[row[~sh]] + j[~sh]] = gi[~sh]
CHG = 512
lr = np.flatnonzero(islong)
chunks = []; longs = []; tot = 0
for jj, rw in enumerate(lr):
    g0, g1_ = grpl[rw], grpl[rw + 1]; nch = (g1_ - g0 + CHG - 1) // CHG
    longs.append((rw, tot, nch, 0))
    for u in range(nch):
        gb = g0 + u * CHG; chunks.append((jj, gb & 0xffffffff, gb >> 32, min(CHG, g1_ - gb)))
    tot += nch
chunks = np.array(chunks, np.int64).astype(np.uint32).view(np.int32).reshape(-1, 4) if chunks else np.zeros((1, 4), np.int32)
longs = np.array(longs, np.int32).reshape(-1, 4) if longs else np.zeros((1, 4), np.int32)
nb = (n + 31) // 32
nonempty = (~islong) & (lens > 0)
pad = np.zeros(nb * 32, bool); pad[:n] = nonempty; nm = np.packbits(pad.reshape(nb, 32)[:, ::-1], axis=1, bitorder='big').view('>u4').ravel().astype(np.uint32)
pad[:] = False; pad[:n] = islong; lm = np.packbits(pad.reshape(nb, 32)[:, ::-1], axis=1, bitorder='big').view('>u4').ravel().astype(np.uint32)
binfo = np.stack([nm, lm], 1).astype(np.uint32)
bg = ngs[:nb * 32] if n >= nb * 32 else np.r_[ngs, np.zeros(nb * 32 - n, np.int64)]
cost = bg.reshape(nb, 32).sum(1) + 8
cw = np.r_[0, np.cumsum(cost)]
print("plan", time.time() - t0, "n", n, "blocks", nb, "chunks", len(chunks), "short groups", grps[-1], flush=True)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
y = np.random.rand(n).astype(np.float32)
yg = np.zeros(ncols, np.float32); yg[cperm[d > 0]] = y[d > 0]
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = cs_[rp[1:]] - cs_[rp[:-1]]
tch, tlo, tcgl, tgrps, tbinfo, tcgs, tyg = T(chunks), T(longs), T(cgl), T(grps.astype(np.int64)), T(binfo), T(np.r_[cgs, -np.ones(4, np.int32)]), T(yg)
counters = torch.zeros(len(longs) + 1, dtype=torch.int32, device='cuda'); partials = torch.zeros(len(chunks) + 1, dtype=torch.float64, device='cuda')
tt = torch.rand(n, device='cuda'); dinv = torch.rand(n, device='cuda'); gpos = T(np.zeros(n, np.int32))
r = torch.zeros(n, device='cuda'); yn = torch.zeros(ncols + 1, device='cuda')
dsum = torch.zeros(1, dtype=torch.float64, device='cuda'); ctr = torch.zeros(1, dtype=torch.int32, device='cuda')
nchunks = len(lr) and len(chunks)
for nt in (1024, 768, 512):
    NWT = 148 * nt // 32
    wk = np.searchsorted(cw, np.linspace(0, cw[-1], NWT + 1), side='left').astype(np.int32); wk[-1] = nb; wk[0] = 0
    twk = T(wk)
    for hc in (0, 32768):
        hc = min(hc, ncols)
        f = lambda: L_.sp10_run(nt, ctypes.c_longlong(nchunks), P(tch.data_ptr()), P(tlo.data_ptr()), P(counters.data_ptr()), P(partials.data_ptr()), P(tcgl.data_ptr()),
                                P(twk.data_ptr()), P(tgrps.data_ptr()), P(tbinfo.data_ptr()), P(tcgs.data_ptr()), ctypes.c_longlong(n), P(tyg.data_ptr()), hc,
                                P(tt.data_ptr()), P(dinv.data_ptr()), P(gpos.data_ptr()), ctypes.c_float(0.0), P(r.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()), P(ctr.data_ptr()))
        r.fill_(-1.0); assert f() == 0; torch.cuda.synchronize()
        got = r.cpu().numpy()
        err = np.max(np.abs(got - ref) / np.maximum(ref, 1e-3))
        bad = np.flatnonzero(np.abs(got - ref) > 1e-5 * np.maximum(ref, 1e-3))
        tm = timeit(f)
        print(f"nt {nt} hc {hc}: {tm:.1f} us  GTEPS {len(ci) / tm / 1e3:.0f}  maxrel {err:.2e} nbad {len(bad)} first {bad[:5]}", flush=True)
