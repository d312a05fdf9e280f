"""User-defined operators on the GPU: spliced into
the generated kernels by NVRTC, evaluated in the operation's type with one rounding per step (the
expected values are the same expression written in numpy in that type), fused with the rest of a
region, usable as a semiring multiply; the persistent cubin cache (NBG_JIT_CACHE, the paper's
future work PAPER.md:310) lets a second process run the same program with zero NVRTC compiles."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


@pytest.mark.parametrize("tname", ["fp32", "fp64", "int32", "int64"])
@pytest.mark.parametrize("mode", ["NONBLOCKING", "BLOCKING"])
def test_user_unop_and_binop_values(nbg, tname, mode):
    sq = nbg.nbg_unop_define("sq_plus", "x * x + c0")
    ad = nbg.nbg_binop_define("scaled_absdiff", "nbg_abs(x - y) * c0")
    t = nbg.TYPE_OF[tname]
    T = nbg.NP_OF[t]
    c = nbg.nbg_init(getattr(nbg, mode), 0)
    try:
        n = 5003
        if T in (np.float32, np.float64):
            x, y = inputs.uniform_vectors(n, 7, T)
            x = (x * 4 - 2).astype(T)
        else:
            rng = np.random.default_rng(7)
            x = rng.integers(-1000, 1000, n).astype(T)
            y = rng.integers(-1000, 1000, n).astype(T)
        vx = nbg.nbg_vector_from_dense(c, t, x)
        vy = nbg.nbg_vector_from_dense(c, t, y)
        a = nbg.nbg_apply(c, t, sq, vx, 3.0)
        b = nbg.nbg_ewise_mult(c, t, ad, a, vy, 2.0)
        iso = nbg.nbg_vector_new_const(c, t, n, 5.0)
        d = nbg.nbg_ewise_add(c, t, ad, iso, vy, 1.0)          # iso operand: not folded on the host
        k3, k2, k1 = T(3), T(2), T(1)
        exp_a = (x * x + k3).astype(T)
        exp_b = (np.abs(exp_a - y) * k2).astype(T)
        exp_d = (np.abs(T(5) - y) * k1).astype(T)
        assert np.array_equal(nbg.nbg_vector_export_dense(c, a), exp_a)
        assert np.array_equal(nbg.nbg_vector_export_dense(c, b), exp_b)
        assert np.array_equal(nbg.nbg_vector_export_dense(c, d), exp_d)
    finally:
        nbg.nbg_finalize(c)


def test_user_ops_fuse_into_one_kernel(nbg):
    sq = nbg.nbg_unop_define("sq_plus", "x * x + c0")
    ad = nbg.nbg_binop_define("scaled_absdiff", "nbg_abs(x - y) * c0")
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        x, y = inputs.uniform_vectors(1 << 16, 3, np.float64)
        vx = nbg.nbg_vector_from_dense(c, nbg.FP64, x)
        vy = nbg.nbg_vector_from_dense(c, nbg.FP64, y)
        nbg.nbg_reset_stats(c)
        a = nbg.nbg_apply(c, nbg.FP64, sq, vx, 0.5)
        b = nbg.nbg_ewise_mult(c, nbg.FP64, ad, a, vy, 3.0)
        nbg.nbg_vector_free(c, a)
        s = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, b)
        nbg.nbg_vector_free(c, b)
        got = nbg.nbg_scalar_get(c, s)
        st = nbg.nbg_get_stats(c)
        assert st["kernels_launched"] == 1 and st["vectors_materialized"] == 0
        import math
        exp = math.fsum(np.abs((x * x + 0.5) - y) * 3.0)
        assert abs(got - exp) <= 1e-12 * abs(exp)
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_user_semiring_multiply(nbg, T):
    """mxv(PLUS, user mul (a, x) -> a * x + c0) over a valued matrix vs the dense definition."""
    mul = nbg.nbg_binop_define("affine_times", "x * y + c0")
    t = nbg.TYPE_OF[T]
    npT = nbg.NP_OF[t]
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        rng = np.random.default_rng(5)
        n = 300
        dense = rng.random((n, n)) < 0.05
        rp = np.concatenate([[0], np.cumsum(dense.sum(1))]).astype(np.int64)
        ci = np.nonzero(dense)[1].astype(np.int32)
        vals = rng.integers(1, 5, ci.shape[0]).astype(npT)
        x = rng.integers(0, 9, n).astype(npT)
        A = nbg.nbg_matrix_from_csr(c, n, n, rp, ci, vals=vals, type=t)
        vx = nbg.nbg_vector_from_dense(c, t, x)
        w = nbg.nbg_mxv(c, t, nbg.PLUS, mul, A, vx, 0.25)
        got = nbg.nbg_vector_export_dense(c, w)
        exp = np.zeros(n, npT)
        for i in range(n):
            acc = 0.0
            for p in range(rp[i], rp[i + 1]):
                acc += float(npT(vals[p] * x[ci[p]] + npT(0.25)))
            exp[i] = npT(acc)
        assert np.array_equal(got, exp)
    finally:
        nbg.nbg_finalize(c)


_PROG = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import inputs
from paper_2509_14211_b200 import nbg
sq = nbg.nbg_unop_define("sq_plus", "x * x + c0")
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
x, y = inputs.uniform_vectors(1 << 14, 9, np.float32)
vx = nbg.nbg_vector_from_dense(c, nbg.FP32, x)
a = nbg.nbg_apply(c, nbg.FP32, sq, vx, 1.0)
s = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, a)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 10, 8, 1)
r, sw, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=5, type=nbg.FP64)
v = float(nbg.nbg_scalar_get(c, s))
st = nbg.nbg_get_stats(c)
print(json.dumps({"v": v, "r0": float(nbg.nbg_vector_export_dense(c, r)[0]), "jit": st["jit_compiles"],
                  "disk": st["jit_disk_hits"], "plans": st["plans_built"]}))
"""


def test_persistent_cache_second_process_compiles_nothing(tmp_path):
    env = dict(os.environ, NBG_JIT_CACHE=str(tmp_path / "jit"))
    outs = []
    for _ in range(2):
        p = subprocess.run([sys.executable, "-c", _PROG % ROOT], env=env, capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    first, second = outs
    assert first["jit"] > 0 and first["plans"] > 0
    assert second["jit"] == 0 and second["disk"] == first["jit"] and second["plans"] == first["plans"]
    assert second["v"] == first["v"] and second["r0"] == first["r0"]
