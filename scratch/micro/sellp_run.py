import sys, os, ctypes, time; sys.path.insert(0, '.'); sys.path.insert(0, 'scratch/micro')
import torch, numpy as np, sellp
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libsellp.so'))
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
t0 = time.time(); p = sellp.build(rp, ci, d); print("plan", time.time() - t0, "slices", p['nslices'], flush=True)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
y = np.random.rand(n).astype(np.float32)
yg1 = np.zeros(p['ncols'] + 1, np.float32); yg1[p['cperm'][d > 0] + 1] = y[d > 0]
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = (cs_[rp[1:]] - cs_[rp[:-1]])[p['rowP']]
ci1 = (p['cperm'][ci] + 1).astype(np.int32)
twt, thdr, tidx, tch, tlo = T(p['wt']), T(p['hdr']), T(p['idx']), T(p['chunks']), T(p['longs'])
counters = torch.zeros(len(p['longs']) + 1, dtype=torch.int32, device='cuda'); partials = torch.zeros(len(p['chunks']) + 1, dtype=torch.float64, device='cuda')
trp = T(rp.astype(np.int64)); tci1 = T(np.r_[ci1, np.zeros(64, np.int32)]); tyg = T(yg1)
tP = torch.rand(n, device='cuda'); dP = torch.rand(n, device='cuda'); gP = T(np.zeros(n, np.int32))
rP = torch.zeros(n, device='cuda'); yn = torch.zeros(p['ncols'] + 1, device='cuda')
dsum = torch.zeros(1, dtype=torch.float64, device='cuda'); ctr = torch.zeros(1, dtype=torch.int32, device='cuda')
for U in (8, 16):
    for hc in (0, 32768, 40960):
        f = lambda: L_.sellp_run(U, p['nslices'], P(twt.data_ptr()), P(thdr.data_ptr()), P(tidx.data_ptr()), ctypes.c_longlong(p['nlong']), ctypes.c_longlong(len(p['chunks'])),
                                 P(tch.data_ptr()), P(tlo.data_ptr()), P(counters.data_ptr()), P(partials.data_ptr()), P(trp.data_ptr()), P(tci1.data_ptr()), P(tyg.data_ptr()), hc,
                                 ctypes.c_longlong(n), ctypes.c_longlong(p['nempty0']), P(tP.data_ptr()), P(dP.data_ptr()), P(gP.data_ptr()), ctypes.c_float(0.0),
                                 P(rP.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()), P(ctr.data_ptr()))
        rP.zero_(); assert f() == 0; torch.cuda.synchronize()
        err = np.max(np.abs(rP.cpu().numpy() - ref) / np.maximum(ref, 1e-3))
        t = timeit(f)
        print(f"U {U} hc {hc}: {t:.1f} us  GTEPS {len(ci) / t / 1e3:.0f}  maxrel {err:.2e}", flush=True)
