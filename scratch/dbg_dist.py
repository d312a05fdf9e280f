# reproducer for a host crash in tests/test_gpu_dist.py (debug aid)
import sys, os, ctypes
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2509_14211_b200 import nbg
from test_dist_gloo import relabel


def oracle_graph(kind, scale, ef, seed):
    f = oracle.rmat_edges if kind == "rmat" else oracle.er_edges
    src, dst = f(scale, ef, seed)
    return oracle.build_csr(1 << scale, src, dst)


if os.environ.get("SELFTEST"):
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    print("deliberate segv", flush=True)
    ctypes.string_at(0)
for kind, scale, ef, seed in [("rmat", 12, 16, 5), ("er", 11, 8, 2), ("rmat", 10, 8, 1)]:
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    k = nbg.GRAPH_RMAT if kind == "rmat" else nbg.GRAPH_ER
    A, d, cuts, ncg = nbg.nbg_dist_graph_from_generator(c, k, scale, ef, seed, nranks=1)
    rp, ci, deg = oracle_graph(kind, scale, ef, seed)
    order, pi, rp2, ci2, ncols_g = relabel(rp, ci, deg)
    grp, gci = nbg.nbg_matrix_export_csr(c, A)
    print("setup", kind, np.array_equal(grp, rp2), np.array_equal(gci, ci2), flush=True)
    nbg.nbg_finalize(c)
print("setup tests done", flush=True)
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, d, cuts, ncg = nbg.nbg_dist_graph_from_generator(c, nbg.GRAPH_RMAT, 13, 16, 7, nranks=1)
print("a", flush=True)
S, sdeg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 13, 16, 7)
print("b", flush=True)
rp, ci, deg = oracle_graph("rmat", 13, 16, 7)
order, pi, _, _, _ = relabel(rp, ci, deg)
print("c", flush=True)
r1, s1, h1 = nbg.nbg_pagerank(c, S, sdeg, tol=-1.0, itermax=12, type=nbg.FP32)
print("d", flush=True)
nbg.nbg_pagerank_dist(c, A, d, cuts, ncg, tol=-1.0, itermax=12, type=nbg.FP32)
print("e", flush=True)
nbg.nbg_reset_stats(c)
r2, s2, h2 = nbg.nbg_pagerank_dist(c, A, d, cuts, ncg, tol=-1.0, itermax=12, type=nbg.FP32)
print("f", flush=True)
v1 = nbg.nbg_vector_export_dense(c, r1)[order]
v2 = nbg.nbg_vector_export_dense(c, r2)
print("max rel", np.max(np.abs(v2 - v1) / v1), flush=True)
nbg.nbg_finalize(c)
print("done", flush=True)
