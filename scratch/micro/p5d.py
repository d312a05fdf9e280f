# 2D-staged SpMV micro-benchmark v4 driver: C4 graph from the library's generator, plan in numpy
# (p5d_plan.py), kernel p5d.cu built per variant (P5D_* macros), checked against numpy, timed.
#   python scratch/micro/p5d.py  [env P5D_VARIANTS="tag:SMAX:BLOB:NRMAX:CUT:NS:LTH:PIECE,..."]
import sys, os, ctypes, time, subprocess
sys.path.insert(0, '.')
sys.path.insert(0, 'scratch/micro')
import numpy as np
import torch
from paper_2509_14211_b200 import nbg
import p5d_plan

torch.cuda.set_device(0)
scale = int(os.environ.get("P5D_SCALE", 22))
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, scale, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
nbg.nbg_finalize(c)
n = rp.shape[0] - 1
nnz = ci.shape[0]
print(f"graph n={n} nnz={nnz}", flush=True)


class Args(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("secs", ctypes.c_void_p), ("blob", ctypes.c_void_p), ("tiles", ctypes.c_void_p),
                ("panels", ctypes.c_void_p), ("seqrec", ctypes.c_void_p), ("seqoff", ctypes.c_void_p), ("citems", ctypes.c_void_p), ("ccomb", ctypes.c_void_p), ("cidx", ctypes.c_void_p), ("crows", ctypes.c_void_p), ("gmask", ctypes.c_void_p), ("gbase", ctypes.c_void_p), ("t", ctypes.c_void_p),
                ("dinv", ctypes.c_void_p), ("perm", ctypes.c_void_p), ("r", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("red", ctypes.c_void_p), ("n", ctypes.c_longlong), ("c", ctypes.c_float)]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


variants = os.environ.get("P5D_VARIANTS", "a:1024:24576:8192:262144:2:32:1024").split(",")
rng = np.random.default_rng(1)
cnt = np.bincount(ci, minlength=n)
dinv = np.where(cnt > 0, np.float32(0.85) / np.maximum(cnt, 1).astype(np.float32), 0).astype(np.float32)
tvec = (rng.random(n) / n).astype(np.float32)
cc = np.float32(0.15 / n)
for v in variants:
    tag, SMAX, BLOB, NRMAX, CUT, NS, LTH, PIECE, NT = (v.split(":") + ["1024"])[:9]
    SMAX, BLOB, NRMAX, CUT, NS, LTH, PIECE, NT = int(SMAX), int(BLOB), int(NRMAX), int(CUT), int(NS), int(LTH), int(PIECE), int(NT)
    H = 0
    so = f"scratch/micro/libp5d_{tag}.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared", "-Xcompiler",
                           "-fPIC", f"-DP5D_SMAX={SMAX}", f"-DP5D_BLOB={BLOB}", f"-DP5D_NRMAX={NRMAX}",
                           f"-DP5D_NS={NS}", f"-DP5D_NT={NT}", "-o", so, "scratch/micro/p5d.cu"])
    L = ctypes.CDLL(os.path.abspath(so))
    t0 = time.time()
    grid = torch.cuda.get_device_properties(0).multi_processor_count * (1024 // NT)
    pl = p5d_plan.build(rp, ci, CUT=CUT, NRMAX=NRMAX, SMAX=SMAX, BLOBMAX=BLOB, LTH=LTH, PIECE=PIECE, G=grid,
                        WMAX=int(os.environ.get("P5D_WMAX", BLOB // 2)))
    st = pl['stats']
    print(f"[{tag}] plan {time.time() - t0:.1f}s {st}", flush=True)
    assert max(st['pmax'], st['cold_pmax']) <= 256 and max(st['cmax'], st['cold_cmax']) <= 64 and pl['maxseq'] <= 256, (st, pl['maxseq'])
    ncg = pl['ncols_g']
    xg = np.zeros(ncg + 64, np.float32)
    # gathered values y = t * dinv in the gather layout
    perm = pl['perm']
    m_ = perm >= 0
    xg[perm[m_]] = tvec[m_] * dinv[m_]
    exp_m = np.bincount(pl['row'], weights=xg[pl['g']].astype(np.float64), minlength=n)
    exp_r = (exp_m.astype(np.float32) + cc).astype(np.float32)
    D = dict(x=dev(xg), secs=dev(pl['secs']), blob=dev(pl['blob']), tiles=dev(pl['tiles']), panels=dev(pl['panels']),
             seqrec=dev(pl['seqrec']), seqoff=dev(pl['seqoff']), citems=dev(pl['citems'] if pl['citems'].size else np.zeros((1,4),np.int32)), ccomb=dev(pl['ccomb'] if pl['ccomb'].size else np.zeros((1,4),np.int32)), cidx=dev(pl['cidx'].view(np.int32) if pl['cidx'].size else np.zeros(4,np.int32)), crows=dev(pl['crows'].view(np.int16) if pl['crows'].size else np.zeros(32,np.int16)),
             gmask=dev(pl['gmask'].view(np.int32)), gbase=dev(pl['gbase']), t=dev(tvec), dinv=dev(dinv), perm=dev(perm),
             r=torch.zeros(n, dtype=torch.float32, device='cuda'), y=torch.zeros(ncg + 64, dtype=torch.float32, device='cuda'),
             red=torch.zeros(2, dtype=torch.float64, device='cuda'))
    a = Args(D['x'].data_ptr(), D['secs'].data_ptr(), D['blob'].data_ptr(), D['tiles'].data_ptr(), D['panels'].data_ptr(),
             D['seqrec'].data_ptr(), D['seqoff'].data_ptr(), D['citems'].data_ptr(), D['ccomb'].data_ptr(), D['cidx'].data_ptr(), D['crows'].data_ptr(), D['gmask'].data_ptr(), D['gbase'].data_ptr(), D['t'].data_ptr(), D['dinv'].data_ptr(), D['perm'].data_ptr(),
             D['r'].data_ptr(), D['y'].data_ptr(), D['red'].data_ptr(), n, float(cc))
    s = torch.cuda.current_stream().cuda_stream
    err = L.p5d_launch(ctypes.byref(a), grid, ctypes.c_void_p(s))
    torch.cuda.synchronize()
    assert err == 0, err
    r = D['r'].cpu().numpy()
    rel = np.abs(r.astype(np.float64) - exp_r) / np.maximum(np.abs(exp_r), 1e-30)
    nbad = int((r != exp_r).sum())
    red = D['red'].cpu().numpy() / 1.0
    exp_dl = np.abs(exp_r.astype(np.float64) - tvec.astype(np.float64)).sum()
    ydev = D['y'].cpu().numpy()[:ncg]
    exp_y = np.zeros(ncg, np.float32)
    exp_y[perm[m_]] = exp_r[m_] * dinv[m_]
    print(f"[{tag}] max rel {rel.max():.3e}, {nbad} of {n} not bit-equal; delta {red[0]:.10e} vs {exp_dl:.10e} (after 1 launch); "
          f"y ok {np.array_equal(ydev, exp_y)}", flush=True)
    # timing
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        L.p5d_launch(ctypes.byref(a), grid, ctypes.c_void_p(s))
    K = 20
    ts = []
    for _ in range(K):
        e0.record()
        L.p5d_launch(ctypes.byref(a), grid, ctypes.c_void_p(s))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = np.array(ts)
    bns = 4 * nnz + 8 * (n + 1) + 2 * 4 * n
    print(f"[{tag}] us per launch: median {np.median(ts):.1f} min {ts.min():.1f}    "
          f"B_ns/t = {bns / np.median(ts) / 1e3:.0f} GB/s  GTEPS {nnz / np.median(ts) / 1e3:.0f}", flush=True)
    del D
