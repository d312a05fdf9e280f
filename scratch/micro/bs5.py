import sys, os, ctypes, time; sys.path.insert(0, '.'); sys.path.insert(0, 'scratch/micro')
import torch, numpy as np, bsplan4
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
L_ = ctypes.CDLL(os.path.abspath('scratch/micro/libbs.so'))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
P = ctypes.c_void_p
def ev(): return torch.cuda.Event(enable_timing=True)
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0, e1 = ev(), ev(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps * 1000
y = np.random.rand(n).astype(np.float32)
cs_ = np.r_[0.0, np.cumsum(y[ci].astype(np.float64))]
ref = cs_[rp[1:]] - cs_[rp[:-1]]
for SB, L, C, nt, wp in ((15, 64, 256, 1024, 4),):
    t0 = time.time(); p = bsplan4.build(rp, ci, d, SB=SB, L=L, C=C, wpiece=wp)
    print("plan", SB, L, C, nt, wp, f"{time.time() - t0:.1f}s", "pieces", p['nslots'], "slices", p['nslices'], flush=True)
    T = {k: torch.from_numpy(v).cuda() for k, v in p.items() if isinstance(v, np.ndarray)}
    yg = np.zeros(p['ncols'], np.float32); yg[p['perm'][d > 0]] = y[d > 0]
    ygt = torch.from_numpy(yg).cuda()
    part = torch.zeros(p['nslots'] + 1, dtype=torch.float64, device='cuda')
    tt = torch.rand(n, device='cuda'); dinv = torch.rand(n, device='cuda'); r = torch.empty(n, device='cuda'); yn = torch.empty(p['ncols'], device='cuda')
    dsum = torch.zeros(1, dtype=torch.float64, device='cuda')
    f1 = lambda: L_.bs_p1v4(nt, L, C, 148, P(T['cs'].data_ptr()), P(T['sblk'].data_ptr()), P(T['soff'].data_ptr()), P(T['snv'].data_ptr()),
                           P(T['hdr'].data_ptr()), P(T['lcol'].data_ptr()), P(ygt.data_ptr()), SB, p['ncols'], P(part.data_ptr()))
    TR, PMAX, grid = 512, 3072, 592
    f2 = lambda: L_.bs_p2v3(TR, grid, PMAX, ctypes.c_longlong(n), p['ntiles'], p['nb'], P(T['tiles'].data_ptr()), P(T['rstart'].data_ptr()),
                            P(T['pre'].data_ptr()), P(T['rslot'].data_ptr()), P(T['qidx'].data_ptr()), P(part.data_ptr()), P(tt.data_ptr()), P(dinv.data_ptr()),
                            P(T['gpos'].data_ptr()), ctypes.c_float(0.0), P(r.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()))
    ti = np.stack([p['tiles'][:-1], p['tiles'][1:], p['rslot'][p['tiles'][:-1]], p['rslot'][p['tiles'][1:]]], 1).astype(np.int32)
    tinfo = torch.from_numpy(np.ascontiguousarray(ti)).cuda()
    for grid in (148 * 2, 148 * 4):
        f3 = lambda: L_.bs_p2v5(grid, p['ntiles'], p['nb'], P(tinfo.data_ptr()), P(T['rstart'].data_ptr()), P(T['pre'].data_ptr()), P(T['rslot'].data_ptr()),
                                P(T['qidx'].data_ptr()), P(part.data_ptr()), P(tt.data_ptr()), P(dinv.data_ptr()), P(T['gpos'].data_ptr()), ctypes.c_float(0.0),
                                P(r.data_ptr()), P(yn.data_ptr()), P(dsum.data_ptr()))
        r.zero_(); assert f1() == 0; assert f3() == 0; torch.cuda.synchronize()
        err = np.max(np.abs(r.cpu().numpy() - ref) / np.maximum(ref, 1e-3))
        print(f"  p2v5 grid {grid}: {timeit(f3):.1f} us  both {timeit(lambda: (f1(), f3())):.1f} maxrel {err:.2e}", flush=True)
    r.zero_()
    assert f1() == 0; assert f2() == 0; torch.cuda.synchronize()
    got = r.cpu().numpy()
    err = np.max(np.abs(got - ref) / np.maximum(ref, 1e-3))
    t1 = timeit(f1); t2 = timeit(f2); t12 = timeit(lambda: (f1(), f2()))
    print(f"  p1 {t1:.1f} us  p2 {t2:.1f} us  both {t12:.1f} us  GTEPS {len(ci) / t12 / 1e3:.0f}  maxrel {err:.2e}", flush=True)
