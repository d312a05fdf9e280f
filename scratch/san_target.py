# compute-sanitizer target (DESIGN.md §4 "sanitizers"): config 1 (R-MAT s10 fp64, 20 sweeps, both
# dangling variants), a small graph whose hub rows are cut into chunks (long-row tickets), the
# elementwise chain, a convergence loop, and the loopback 2-rank data plane -- every skeleton once.
import sys
import threading
sys.path.insert(0, ".")
import numpy as np
import inputs
from paper_2509_14211_b200 import nbg

c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 10, 8, 1)
for dang in (nbg.PR_UNIFORM, nbg.PR_DROP):
    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=20, dangling=dang, type=nbg.FP64)
    print("c1", dang, s, float(nbg.nbg_vector_export_dense(c, r).sum()))
# hubs: 3 vertices with ~20k in-edges each (chunked long rows, tickets), 4000 vertices
rng = np.random.default_rng(1)
n, m = 4000, 60000
src = rng.integers(0, n, m).astype(np.int32)
dst = np.where(rng.random(m) < 0.9, rng.integers(0, 3, m), rng.integers(0, n, m)).astype(np.int32)
B, bdeg = nbg.nbg_matrix_from_edges(c, n, src, dst)
for T in (nbg.FP32, nbg.FP64):
    r, s, h = nbg.nbg_pagerank(c, B, bdeg, tol=1e-9, itermax=50, type=T)
    print("hubs", T, s, float(nbg.nbg_vector_export_dense(c, r).sum()))
x, y = inputs.uniform_vectors(1 << 16, 3, np.float32)
vx = nbg.nbg_vector_from_dense(c, nbg.FP32, x)
vy = nbg.nbg_vector_from_dense(c, nbg.FP32, y)
a = nbg.nbg_apply(c, nbg.FP32, "ADD_C", vy, 1.0)
z = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", vx, a)
print("chain", nbg.nbg_scalar_get(c, nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, z)))
nbg.nbg_finalize(c)
ctxs = [nbg.nbg_init(nbg.NONBLOCKING, 0) for _ in range(2)]
nbg.nbg_dist_init_loopback(ctxs)
out = [None, None]


def rank(q):
    Ad, d, cuts, ncg = nbg.nbg_dist_graph_from_generator(ctxs[q], nbg.GRAPH_RMAT, 11, 8, 2, nranks=2)
    r, s, h = nbg.nbg_pagerank_dist(ctxs[q], Ad, d, cuts, ncg, tol=-1.0, itermax=5, type=nbg.FP32)
    out[q] = (s, h[-1])


th = [threading.Thread(target=rank, args=(q,)) for q in range(2)]
[t.start() for t in th]
[t.join() for t in th]
print("dist", out)
for cc in ctxs:
    nbg.nbg_finalize(cc)
print("SAN_TARGET_OK")
