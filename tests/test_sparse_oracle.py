"""Pins of the sparse-vector oracle (oracle/sparse.py) -- CPU only.

* the worked examples of SPEC.md:186-203 and 211-217 (apply, intersection, union, reduce, empty);
* brute force on tiny random vectors against an independent dict formulation of the GraphBLAS
  definitions (intersection / union of stored positions);
* mxv with a partially present x: a 2x2 hand example and brute force against the dense oracle on
  a zero-filled x (PLUS/TIMES, where an absent x contributes exactly 0);
* the estimator formulas: leaf = nnz / size, ewise_mult = product.
"""
import numpy as np

from oracle import ops
from oracle import sparse as S


def d(sv):
    return {int(i): float(v) for i, v in zip(sv.idx, sv.vals)}


def test_spec_examples():
    f32 = np.float32
    u = S.sparse(4, [0, 2], np.array([1.0, 3.0], f32))
    assert d(S.apply("ADD_C", u, f32, 1.0)) == {0: 2.0, 2: 4.0}
    v = S.sparse(4, [0, 1], np.array([2.0, 2.0], f32))
    assert d(S.ewise_mult("TIMES", u, v, f32)) == {0: 2.0}
    a = S.sparse(4, [0], np.array([1.0], f32))
    b = S.sparse(4, [0, 1], np.array([2.0, 5.0], f32))
    assert d(S.ewise_add("PLUS", a, b, f32)) == {0: 3.0, 1: 5.0}
    e = S.sparse(4, [], np.array([], f32))
    assert d(S.ewise_mult("TIMES", u, e, f32)) == {}
    assert d(S.ewise_add("PLUS", u, e, f32)) == d(u)
    w = S.sparse(5, [0, 2, 3], np.array([1.0, 2.0, 3.0], f32))
    assert S.reduce("PLUS", w, f32) == 6.0
    assert S.reduce("PLUS", e, f32) == 0.0 and S.reduce("MAX", e, np.float64) == -np.inf


def _rand_sv(rng, n, fill, T):
    m = rng.random(n) < fill
    idx = np.nonzero(m)[0]
    vals = rng.integers(-8, 9, idx.shape[0]).astype(T)
    return S.sparse(n, idx, vals)


def test_brute_force_intersection_union():
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(1, 40))
        T = [np.float32, np.float64, np.int32, np.int64][trial % 4]
        u = _rand_sv(rng, n, rng.random(), T)
        v = _rand_sv(rng, n, rng.random(), T)
        du, dv = d(u), d(v)
        m = S.ewise_mult("TIMES", u, v, T)
        assert d(m) == {k: du[k] * dv[k] for k in du if k in dv}
        a = S.ewise_add("MAX", u, v, T)
        exp = {}
        for k in set(du) | set(dv):
            exp[k] = max(du[k], dv[k]) if (k in du and k in dv) else (du[k] if k in du else dv[k])
        assert d(a) == exp
        assert list(a.idx) == sorted(exp)
        b = S.bind2nd("MINUS", u, 3.0, T)
        assert d(b) == {k: x - 3.0 for k, x in du.items()}
        assert S.reduce("PLUS", u, np.float64) == sum(du.values())
        if du:
            assert S.reduce("MIN", u, np.float64) == min(du.values())


def test_mxv_partial_x():
    # A = [[0, 2], [1, 0]] stored nonzeros (SPEC.md:207 example) with x = {1: 4} only
    rp = np.array([0, 1, 2])
    ci = np.array([1, 0], np.int32)
    vals = np.array([2.0, 1.0], np.float64)
    x = S.sparse(2, [1], np.array([4.0]))
    w = S.mxv("PLUS", "TIMES", rp, ci, vals, x, np.float64)
    assert list(w) == [8.0, 0.0]          # row 1 meets no present x entry -> identity 0
    wm = S.mxv("MIN", "TIMES", rp, ci, vals, x, np.float64)
    assert wm[0] == 8.0 and wm[1] == np.inf
    rng = np.random.default_rng(3)
    for _ in range(10):
        n = int(rng.integers(2, 30))
        dense = rng.random((n, n)) < 0.3
        rp = np.concatenate([[0], np.cumsum(dense.sum(1))])
        ci = np.nonzero(dense)[1].astype(np.int32)
        av = rng.integers(1, 5, ci.shape[0]).astype(np.float64)
        x = _rand_sv(rng, n, 0.5, np.float64)
        xz = np.zeros(n)
        xz[x.idx] = x.vals
        assert np.array_equal(S.mxv("PLUS", "TIMES", rp, ci, av, x, np.float64),
                              ops.mxv("PLUS", "TIMES", rp, ci, av, xz, np.float64))


def test_estimator_formulas():
    u = S.sparse(10, [0, 3, 5, 9], np.ones(4))
    assert S.fill(u) == 0.4
    assert abs(S.fill_mult(0.3, 0.5) - 0.15) < 1e-15          # PAPER.md:237 (product)
    assert S.fill_add(0.0, 0.25) == 0.25 and S.fill_add(1.0, 0.3) == 1.0
    # independence: the expected fill of a union of independent random supports
    rng = np.random.default_rng(1)
    a, b = rng.random(200000) < 0.3, rng.random(200000) < 0.2
    assert abs((a | b).mean() - S.fill_add(0.3, 0.2)) < 5e-3 and abs((a & b).mean() - S.fill_mult(0.3, 0.2)) < 5e-3
