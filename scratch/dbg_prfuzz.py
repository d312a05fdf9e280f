import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2509_14211_b200 import nbg
for seed in range(16):
    rng = np.random.default_rng(1100 + seed)
    n = int(rng.integers(1, 3000)); m = int(rng.integers(0, 8 * n + 1))
    src = rng.integers(0, n, m).astype(np.int32)
    dst = (rng.integers(0, max(1, n // 50), m) if seed % 3 == 0 else rng.integers(0, n, m)).astype(np.int32)
    T = np.float32 if seed % 2 else np.float64
    t = nbg.FP32 if T is np.float32 else nbg.FP64
    tol = -1.0 if seed % 4 < 2 else (1e-6 if T is np.float32 else 1e-12)
    uniform = seed % 5 != 0
    c = nbg.nbg_init(nbg.NONBLOCKING if seed % 7 else nbg.BLOCKING, 0)
    A, deg = nbg.nbg_matrix_from_edges(c, n, src, dst)
    orp, oci, odeg = oracle.build_csr(n, src, dst)
    r, sw, hist = nbg.nbg_pagerank(c, A, deg, tol=tol, itermax=60, type=t, dangling=nbg.PR_UNIFORM if uniform else nbg.PR_DROP)
    ro, so, dho, _ = oracle.pagerank(orp, oci, odeg, dtype=T, itermax=60, tol=tol, uniform=uniform)
    got = nbg.nbg_vector_export_dense(c, r)
    atol = 4.0 * float(np.spacing(np.abs(np.asarray(ro, T))).astype(np.float64).sum())
    h = np.asarray(hist); d = np.asarray(dho)
    bad = np.nonzero(np.abs(h - d) > np.maximum(1e-9 * np.abs(d), atol))[0]
    print(seed, n, m, T.__name__, tol, uniform, 'sw', sw, so, 'rel', float(np.max(np.abs(got - ro) / np.abs(ro))) if n else 0, 'atol', atol, 'bad', bad[:5], h[bad[:3]], d[bad[:3]])
    nbg.nbg_finalize(c)
