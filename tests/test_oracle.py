"""Pins for the CPU oracle (oracle/): each test ties an oracle function to something other than
itself -- a published value, a closed form, brute force, a textbook routine, an exact rational
solve or an invariant -- chosen so that a dropped term, a wrong sign/index or a transposed
operand fails at least one of them.  DESIGN.md "Oracle pins" lists which test pins what."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import ops

ALPHA = 0.85


# ------------------------------------------------------------------ SplitMix64 (reading Q9)

def test_sm64_published_vector():
    # SplitMix64 seeded with 0 (Steele et al. 2014 reference generator): the published first
    # three outputs.  Our output k uses state key + (k+1)*gamma, i.e. exactly that stream.
    assert oracle.sm64(0, 0) == 0xE220A8397B1DCDAF
    assert oracle.sm64(0, 1) == 0x6E789E6AA1B965F4
    assert oracle.sm64(0, 2) == 0x06C45D188009454F


def test_sm64_matches_shared_input_generator():
    # inputs/ is the only module both sides may share; its vectorised SplitMix64 must be the
    # same stream (this pins inputs.uniform_vectors to the published vector transitively).
    import inputs
    ks = np.array([0, 1, 2, 12345, 2**40 + 7], dtype=np.uint64)
    got = inputs.sm64_np(99, ks)
    assert [int(v) for v in got] == [oracle.sm64(99, int(k)) for k in ks]


# ------------------------------------------------------------------ generators

def test_rmat_counts_and_range():
    src, dst = oracle.rmat_edges(10, 8, seed=1)
    assert src.shape == (8192,) and dst.shape == (8192,)
    assert src.min() >= 0 and src.max() < 1024 and dst.min() >= 0 and dst.max() < 1024


def test_rmat_quadrant_probabilities():
    # Every level draws one quadrant with P = (0.57, 0.19, 0.19, 0.05) (BASELINE configs).
    scale = 12
    src, dst = oracle.rmat_edges(scale, 16, seed=3)
    m = src.shape[0]
    for bit in (scale - 1, scale // 2, 0):
        s = (src >> bit) & 1
        d = (dst >> bit) & 1
        p = [np.mean((s == a) & (d == b)) for a, b in ((0, 0), (0, 1), (1, 0), (1, 1))]
        sd = np.sqrt(0.25 / m)
        assert abs(p[0] - 0.57) < 6 * sd and abs(p[1] - 0.19) < 6 * sd
        assert abs(p[2] - 0.19) < 6 * sd and abs(p[3] - 0.05) < 6 * sd


def test_er_uniform_targets():
    src, dst = oracle.er_edges(12, 16, seed=5)
    assert src.shape[0] == 16 << 12
    counts = np.bincount(dst, minlength=4096)
    # Poisson(16) in-degree: mean 16, variance ~16
    assert abs(counts.mean() - 16) < 1e-9
    assert 12 < counts.var() < 20


# ------------------------------------------------------------------ CSR build (P1 brute force)

@pytest.mark.parametrize("seed", range(6))
def test_csr_build_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 65))
    m = int(rng.integers(0, 4 * n + 1))
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    if m > 3:   # force duplicates and self-loops
        src[1], dst[1] = src[0], dst[0]
        dst[2] = src[2]
    rowptr, colidx, deg = oracle.build_csr(n, src, dst)
    dense = np.zeros((n, n), bool)          # dense AT: AT[v, u] = 1 for edge u -> v, u != v
    for u, v in zip(src, dst):
        if u != v:
            dense[v, u] = True
    rows, cols = np.nonzero(dense)          # row-major order == CSR order
    assert np.array_equal(colidx, cols.astype(np.int32))
    assert np.array_equal(rowptr, np.concatenate([[0], np.cumsum(dense.sum(1))]).astype(np.int64))
    assert np.array_equal(deg, dense.sum(0).astype(np.int32))   # out-degree = column count of AT


def test_csr_invariants_rmat():
    src, dst = oracle.rmat_edges(10, 8, seed=1)
    rowptr, colidx, deg = oracle.build_csr(1024, src, dst)
    nnz = colidx.shape[0]
    assert rowptr[0] == 0 and rowptr[-1] == nnz == deg.sum()
    assert np.all(np.diff(rowptr) >= 0)
    for i in range(1024):
        c = colidx[rowptr[i]:rowptr[i + 1]]
        assert np.all(np.diff(c) > 0) and not np.any(c == i)
    # plausibility (dedup ratio ~0.81, ~31% dangling at s10 ef8)
    assert 0.75 < nnz / 8192 < 0.87
    assert 0.25 < np.mean(deg == 0) < 0.38


# ------------------------------------------------------------------ PageRank pins

def _csr_from_edges(n, edges):
    src = np.array([u for u, v in edges], np.int32)
    dst = np.array([v for u, v in edges], np.int32)
    return oracle.build_csr(n, src, dst)


@pytest.mark.parametrize("n", [3, 7, 64])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("uniform", [True, False])
def test_cycle_is_uniform(n, dtype, uniform):
    # P3: a directed n-cycle's ranks are all equal and stay at 1/n (symmetry).
    rp, ci, deg = _csr_from_edges(n, [(i, (i + 1) % n) for i in range(n)])
    r, sweeps, dh, _ = oracle.pagerank(rp, ci, deg, dtype=dtype, uniform=uniform, itermax=30)
    assert sweeps == 30
    assert np.all(r == r[0])
    one_n = dtype(1.0 / n)
    assert abs(float(r[0]) - float(one_n)) <= float(np.spacing(one_n))


def test_four_node_closed_form():
    # P4 (SPEC.md:453 graph 0->1, 1->2, 2->0, 3->0): r3 = t, r0 = t(1+a)^2/(1-a^3),
    # r1 = t + a r0, r2 = t + a r1, t = (1-a)/4.  Exact rationals, a = 17/20.
    a = Fraction(17, 20)
    t = (1 - a) / 4
    r0 = t * (1 + a) ** 2 / (1 - a ** 3)
    r1 = t + a * r0
    r2 = t + a * r1
    exact = np.array([float(r0), float(r1), float(r2), float(t)])
    rp, ci, deg = _csr_from_edges(4, [(0, 1), (1, 2), (2, 0), (3, 0)])
    r, sweeps, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, itermax=400)
    assert np.max(np.abs(r - exact) / exact) < 1e-14
    assert abs(r.sum() - 1.0) < 1e-14


def test_star_dangling_closed_forms():
    # P5: star i -> 0 (i = 1..5), n = 6; vertex 0 is dangling.
    rp, ci, deg = _csr_from_edges(6, [(i, 0) for i in range(1, 6)])
    ru, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, uniform=True, itermax=400)
    assert abs(ru[0] - 21 / 41) < 1e-14 and np.max(np.abs(ru[1:] - 4 / 41)) < 1e-14
    rd, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, uniform=False, itermax=400)
    assert abs(rd[0] - 0.13125) < 1e-15 and np.max(np.abs(rd[1:] - 0.025)) < 1e-15


def _random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    A = rng.random((n, n)) < p
    np.fill_diagonal(A, False)
    edges = [(int(u), int(v)) for u, v in zip(*np.nonzero(A))]   # A[u, v]: edge u -> v
    return A, edges


@pytest.mark.parametrize("seed", range(4))
def test_dense_google_matrix_power_iteration(seed):
    # P6: the sweep is the textbook power iteration with the column-stochastic Google matrix
    # G = a*P + (1-a)/n 11^T, P[v,u] = 1/deg(u) for u -> v, dangling columns = 1/n (UNIFORM).
    n = 9
    A, edges = _random_graph(n, 0.25, seed)
    A[0, :] = False                      # make vertex 0 dangling
    edges = [(u, v) for (u, v) in edges if u != 0]
    rp, ci, deg = _csr_from_edges(n, edges)
    P = np.zeros((n, n))
    for u in range(n):
        d = A[u].sum()
        if d == 0:
            P[:, u] = 1.0 / n
        else:
            P[A[u], u] = 1.0 / d
    G = ALPHA * P + (1 - ALPHA) / n * np.ones((n, n))
    x = np.full(n, 1.0 / n)
    for _ in range(20):
        x = G @ x
    r, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, itermax=20)
    assert np.max(np.abs(r - x) / x) < 1e-13


@pytest.mark.parametrize("seed", range(3))
def test_exact_rational_fixed_point(seed):
    # P7: the converged sweep solves (I - a M) r = (1-a)/n 1 exactly, with M = P (UNIFORM).
    n = 6
    A, edges = _random_graph(n, 0.3, 10 + seed)
    rp, ci, deg = _csr_from_edges(n, edges)
    a = Fraction(17, 20)
    M = [[Fraction(0)] * n for _ in range(n)]
    for u in range(n):
        d = int(A[u].sum())
        for v in range(n):
            M[v][u] = Fraction(1, n) if d == 0 else (Fraction(1, d) if A[u, v] else Fraction(0))
    # Gaussian elimination on (I - aM) r = b
    S = [[(1 if i == j else 0) - a * M[i][j] for j in range(n)] + [(1 - a) / n] for i in range(n)]
    for c in range(n):
        piv = next(i for i in range(c, n) if S[i][c] != 0)
        S[c], S[piv] = S[piv], S[c]
        for i in range(n):
            if i != c and S[i][c] != 0:
                f = S[i][c] / S[c][c]
                S[i] = [x - f * y for x, y in zip(S[i], S[c])]
    exact = np.array([float(S[i][n] / S[i][i]) for i in range(n)])
    r, sweeps, dh, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, itermax=1000, tol=1e-15)
    assert dh[-1] <= 1e-15 or sweeps == 1000
    assert np.max(np.abs(r - exact) / exact) < 1e-12


def test_mass_conservation_and_drop_equivalence():
    # P8: UNIFORM conserves mass; DROP == UNIFORM bit-exactly when nothing dangles.
    src, dst = oracle.rmat_edges(10, 8, seed=1)
    rp, ci, deg = oracle.build_csr(1024, src, dst)
    r64, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, itermax=20)
    r32, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float32, itermax=20)
    assert abs(r64.sum() - 1) < 1e-12
    assert abs(float(r32.astype(np.float64).sum()) - 1) < 1e-5
    assert np.max(np.abs(r32 - r64) / r64) < 1e-5          # fp32(fp64-acc) vs fp64
    rd, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, uniform=False, itermax=20)
    assert rd.sum() < 1 - 1e-3                              # dangling mass leaks under DROP
    rpc, cic, degc = _csr_from_edges(50, [(i, (i + 1) % 50) for i in range(50)] + [(3, 7), (9, 2)])
    assert np.all(degc > 0)
    a, _, _, _ = oracle.pagerank(rpc, cic, degc, dtype=np.float32, uniform=True, itermax=25)
    b, _, _, _ = oracle.pagerank(rpc, cic, degc, dtype=np.float32, uniform=False, itermax=25)
    assert np.array_equal(a, b)


def test_delta_and_ds_history_definitions():
    # rdiff_k = sum_i |r_k - r_{k-1}| (Fig. 6); ds_k = sum over dangling of r_{k-1}.
    src, dst = oracle.rmat_edges(9, 8, seed=4)
    rp, ci, deg = oracle.build_csr(512, src, dst)
    prev = np.full(512, 1.0 / 512)
    _, _, dh, sh = oracle.pagerank(rp, ci, deg, dtype=np.float64, itermax=6)
    for k in range(1, 7):
        rk, _, _, _ = oracle.pagerank(rp, ci, deg, dtype=np.float64, itermax=k)
        assert abs(dh[k - 1] - np.abs(rk - prev).sum()) <= 1e-13 * max(dh[k - 1], 1e-300)
        assert abs(sh[k - 1] - prev[deg == 0].sum()) <= 1e-15
        prev = rk


def test_loop_semantics():
    # Fig. 6 / SPEC.md:454: itermax = 1 -> exactly one sweep (iter = 2); tol stops at the first
    # sweep whose rdiff <= tol.
    src, dst = oracle.rmat_edges(10, 8, seed=2)
    rp, ci, deg = oracle.build_csr(1024, src, dst)
    _, s1, _, _ = oracle.pagerank(rp, ci, deg, itermax=1, tol=1e-9)
    assert s1 == 1
    _, s, dh, _ = oracle.pagerank(rp, ci, deg, itermax=100, tol=1e-6)
    assert dh[-1] <= 1e-6 and np.all(dh[:-1] > 1e-6)
    assert np.all(np.diff(dh) < 0)                      # contraction by ~alpha per sweep


def test_mxv_plus_vs_dense():
    src, dst = oracle.rmat_edges(8, 8, seed=7)
    rp, ci, deg = oracle.build_csr(256, src, dst)
    x = np.arange(256, dtype=np.float64) % 17          # small integers: every sum is exact
    dense = np.zeros((256, 256))
    for i in range(256):
        dense[i, ci[rp[i]:rp[i + 1]]] = 1
    assert np.array_equal(oracle.mxv_plus(rp, ci, x), dense @ x)


# ------------------------------------------------------------------ ops.py pins (SPEC examples)

def test_ops_spec_examples():
    f64 = np.float64
    assert np.array_equal(ops.unop("ADD_C", np.full(3, 1.0), f64, 1.0), np.full(3, 2.0))
    assert np.array_equal(ops.ewise_mult("TIMES", np.array([1., 2.]), np.array([3., 4.]), f64),
                          [3., 8.])
    assert ops.ewise_mult("TIMES", np.ones(2), None, f64) is None
    got = ops.ewise_add("ABSDIFF", np.array([0.2, 0.4]), np.array([0.3, 0.1]), f64)
    assert np.allclose(got, [0.1, 0.3], rtol=1e-15, atol=1e-16)
    assert np.array_equal(ops.ewise_add("PLUS", np.ones(2), None, f64), np.ones(2))
    rp = np.array([0, 1, 2], np.int64)
    ci = np.array([1, 0], np.int32)
    vals = np.array([2.0, 1.0])
    assert np.array_equal(ops.mxv("PLUS", "TIMES", rp, ci, vals, np.array([3., 4.]), f64), [8., 3.])
    rp2 = np.array([0, 2], np.int64)
    ci2 = np.array([0, 1], np.int32)
    assert ops.mxv("PLUS", "SECOND", rp2, ci2, None, np.array([5., 7.]), f64)[0] == 12.0
    rp3 = np.array([0, 0], np.int64)
    assert ops.mxv("PLUS", "TIMES", rp3, np.zeros(0, np.int32), None, np.ones(1), f64)[0] == 0.0
    assert ops.reduce("PLUS", np.array([1., 2., 3.]), f64) == 6.0
    assert ops.reduce("PLUS", None, f64) == 0.0
    assert ops.reduce("MAX", np.array([3., 9., 1.]), f64) == 9.0


def test_ops_fp32_rounding_is_single_step():
    # Each fp32 operator result equals the fp64-exact result rounded once (Sterbenz/exact
    # products): checks that ops.py computes in T, not in a wider type with a late rounding.
    rng = np.random.default_rng(0)
    a = rng.random(1000).astype(np.float32)
    b = rng.random(1000).astype(np.float32)
    f32 = np.float32
    assert np.array_equal(ops.binop("TIMES", a, b, f32), (a.astype(np.float64) * b).astype(f32))
    assert np.array_equal(ops.binop("ABSDIFF", a, b, f32), np.abs(a.astype(np.float64) - b).astype(f32))
    assert np.array_equal(ops.binop("DIV", a, b, f32), (a.astype(np.float64) / b).astype(f32))


def test_ops_reduce_exact():
    v = np.array([1e16, 1.0, -1e16, 1.0])
    assert ops.reduce("PLUS", v, np.float64) == 2.0     # exact sum (a sequential sum gives 1.0 or 0.0)


def test_ops_mxv_vs_dense_random():
    rng = np.random.default_rng(3)
    n = 20
    dense = (rng.random((n, n)) < 0.3).astype(np.float64)
    rp = np.concatenate([[0], np.cumsum(dense.sum(1))]).astype(np.int64)
    ci = np.nonzero(dense)[1].astype(np.int32)
    x = rng.integers(0, 9, n).astype(np.float64)
    assert np.array_equal(ops.mxv("PLUS", "TIMES", rp, ci, None, x, np.float64), dense @ x)
    assert np.array_equal(ops.mxv("MAX", "SECOND", rp, ci, None, x, np.float64),
                          np.array([x[dense[i] > 0].max() if dense[i].any() else -np.inf for i in range(n)]))


def test_ops_empty_fold_identities():
    """An empty fold yields the monoid's identity in the result type (SPEC.md:206 for mxv rows,
    SPEC.md:211-217 for reduce): 0, +/-inf for floats, the extreme values of an integer type --
    checked against numpy's own integer limits and a brute-force min/max over the whole type."""
    for T in (np.int32, np.int64):
        info = np.iinfo(T)
        assert ops.reduce("MIN", None, T) == info.max and ops.reduce("MAX", None, T) == info.min
        assert ops.reduce("MIN", None, T).dtype == np.dtype(T)
        # identity property: min(identity, v) == v for the extremes of the type
        for v in (info.min, -1, 0, 1, info.max):
            assert min(int(ops.reduce("MIN", None, T)), v) == v and max(int(ops.reduce("MAX", None, T)), v) == v
    assert ops.reduce("MIN", None, np.float32) == np.inf and ops.reduce("PLUS", None, np.float64) == 0.0
    # mxv: an empty row takes the identity, a non-empty one its fold
    rp = np.array([0, 0, 2], np.int64)
    ci = np.array([0, 1], np.int32)
    x = np.array([4, -3], np.int32)
    assert list(ops.mxv("MIN", "SECOND", rp, ci, None, x, np.int32)) == [np.iinfo(np.int32).max, -3]
    assert list(ops.mxv("MAX", "SECOND", rp, ci, None, x, np.int64)) == [np.iinfo(np.int64).min, 4]


def test_ops_integer_division_exact():
    """C truncating division (toward zero) for integers, x / 0 = 0 (reading R2), exact beyond 2^53."""
    a = np.array([7, -7, 7, -7, 0, 5, 2**62 + 1, -(2**62) - 3, -2**63, 1], np.int64)
    b = np.array([2, 2, -2, -2, 3, 0, 3, 7, 3, -2**63], np.int64)
    exp = [3, -3, -3, 3, 0, 0, (2**62 + 1) // 3, -((2**62 + 3) // 7), -(2**63 // 3), 0]
    assert list(ops.binop("DIV", a, b, np.int64)) == exp
    assert list(ops.unop("MINV", np.array([1, -1, 2, 0, -2**31], np.int32), np.int32)) == [1, -1, 0, 0, 0]


def test_openmp_build_is_identical():
    # bench.py's all-core baseline runs the same orc.c built with -fopenmp (rows split over
    # threads, each row's sum in ascending order): results must equal the single-threaded build
    src, dst = oracle.rmat_edges(12, 8, seed=2)
    rp, ci, deg = oracle.build_csr(4096, src, dst)
    for dt in (np.float32, np.float64):
        a = oracle.pagerank(rp, ci, deg, dtype=dt, itermax=6)
        b = oracle.pagerank(rp, ci, deg, dtype=dt, itermax=6, threads=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2]) and a[1] == b[1]
