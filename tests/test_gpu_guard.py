"""Guard mode (NBG_GUARD=1, include/nbg.h nbg_guard_selftest): red zones after every pool buffer,
checked after each generated kernel and each wait -- the out-of-bounds-write check that replaces
compute-sanitizer, which is closed on the GPU pool (profiles/r2_sanitizer_closed.txt).

A subprocess with NBG_GUARD=1 (the mode is read once per process) checks that an intentional
one-byte overflow is reported, then runs every skeleton once -- PageRank at C1 (both dangling
variants), a chunked-hub-row graph, the config-2 chain, sparse ops and the 2-rank loopback data
plane in both exchange modes -- which must finish without a guard report."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SCRIPT = r'''
import sys, threading
sys.path.insert(0, ".")
import numpy as np
import inputs
from paper_2509_14211_b200 import nbg

c = nbg.nbg_init(nbg.NONBLOCKING, 0)
try:
    nbg.nbg_guard_selftest(c)
    print("SELFTEST_MISSED")
except nbg.NbgError as e:
    assert "guard" in str(e), e
    print("SELFTEST_CAUGHT")
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 10, 8, 1)
for dang in (nbg.PR_UNIFORM, nbg.PR_DROP):
    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=20, dangling=dang, type=nbg.FP64)
    nbg.nbg_vector_export_dense(c, r)
rng = np.random.default_rng(1)
n, m = 4000, 60000
src = rng.integers(0, n, m).astype(np.int32)
dst = np.where(rng.random(m) < 0.9, rng.integers(0, 3, m), rng.integers(0, n, m)).astype(np.int32)
H, hdeg = nbg.nbg_matrix_from_edges(c, n, src, dst)
for T in (nbg.FP32, nbg.FP64):
    r, s, h = nbg.nbg_pagerank(c, H, hdeg, tol=1e-9, itermax=50, type=T)
    nbg.nbg_vector_export_dense(c, r)
x, y = inputs.uniform_vectors(1 << 16, 3)
u = nbg.nbg_vector_from_dense(c, nbg.FP32, x)
v = nbg.nbg_vector_from_dense(c, nbg.FP32, y)
z = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", u, nbg.nbg_apply(c, nbg.FP32, "ADD_C", v, 1.0))
nbg.nbg_scalar_get(c, nbg.nbg_reduce(c, nbg.FP64, "PLUS", z))
sp = nbg.nbg_vector_from_sparse(c, nbg.FP32, 1 << 16, np.array([3, 70, 9000], np.int32), np.ones(3, np.float32))
nbg.nbg_vector_export_sparse(c, nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", sp, u))
nbg.nbg_vector_export_dense(c, nbg.nbg_ewise_add(c, nbg.FP32, "PLUS", sp, u))
nbg.nbg_sync(c)
nbg.nbg_finalize(c)
for mode in (nbg.DIST_EXCHANGE_COLLECTIVE, nbg.DIST_EXCHANGE_PEER):
    ctxs = [nbg.nbg_init(nbg.NONBLOCKING, 0) for _ in range(2)]
    nbg.nbg_dist_init_loopback(ctxs)
    errs = []
    def rank(q):
        try:
            cq = ctxs[q]
            nbg.nbg_dist_set_exchange(cq, mode)
            Aq, dq, cuts, ncg = nbg.nbg_dist_graph_from_generator(cq, nbg.GRAPH_RMAT, 11, 16, 3, nranks=2)
            r, s, h = nbg.nbg_pagerank_dist(cq, Aq, dq, cuts, ncg, tol=-1.0, itermax=6)
            nbg.nbg_vector_export_dense(cq, r)
            nbg.nbg_sync(cq)
        except Exception as e:
            errs.append(e)
    th = [threading.Thread(target=rank, args=(q,)) for q in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    for cq in ctxs:
        nbg.nbg_finalize(cq)
print("GUARD_RUN_OK")
'''


def test_guard_mode_catches_overflow_and_every_skeleton_runs_clean():
    env = dict(os.environ, NBG_GUARD="1")
    p = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    assert "SELFTEST_CAUGHT" in p.stdout, out[-3000:]
    assert "GUARD_RUN_OK" in p.stdout and "guard:" not in p.stderr, out[-3000:]
