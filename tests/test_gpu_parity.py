"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): bit-exact graph structure, out-degrees and sweep counts; ranks
within max relative error 1e-10 (fp64) / 1e-5 (fp32) after the same sweep count; blocking ==
nonblocking bit for bit (fused kernels keep the blocking rounding points).
"""
import numpy as np
import pytest

import oracle
from oracle import ops

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


@pytest.fixture(scope="module")
def ctx(nbg):
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    yield c
    nbg.nbg_finalize(c)


@pytest.fixture(scope="module")
def bctx(nbg):
    c = nbg.nbg_init(nbg.BLOCKING, 0)
    yield c
    nbg.nbg_finalize(c)


def delta_close(got, exp, r_final, npT):
    """Delta_k = sum_i |r_k - r_{k-1}| is a sum of cancelling differences: a 1-ulp change of any
    rank moves it by ulp(r_i).  Bound: rel 1e-9 or 4 * sum_i ulp_T(r_i) absolute (derived,
    DESIGN.md "tolerances")."""
    atol = 4.0 * float(np.spacing(np.abs(np.asarray(r_final, npT))).astype(np.float64).sum())
    got = np.asarray(got)
    exp = np.asarray(exp)
    return bool(np.all(np.abs(got - exp) <= np.maximum(1e-9 * np.abs(exp), atol)))


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.abs(b))) if a.size else 0.0


# ------------------------------------------------------------------ a0: generation + CSR build

@pytest.mark.parametrize("kind,scale,ef,seed", [("rmat", 10, 8, 1), ("rmat", 10, 8, 2), ("rmat", 10, 8, 3),
                                                ("rmat", 14, 16, 5), ("er", 12, 16, 4)])
def test_edges_and_csr_bit_exact(nbg, ctx, kind, scale, ef, seed):
    k = nbg.GRAPH_RMAT if kind == "rmat" else nbg.GRAPH_ER
    src, dst = nbg.nbg_graph_edges(ctx, k, scale, ef, seed)
    osrc, odst = (oracle.rmat_edges if kind == "rmat" else oracle.er_edges)(scale, ef, seed)
    assert np.array_equal(src, osrc) and np.array_equal(dst, odst)
    A, deg = nbg.nbg_matrix_from_generator(ctx, k, scale, ef, seed)
    rp, ci = nbg.nbg_matrix_export_csr(ctx, A)
    orp, oci, odeg = oracle.build_csr(1 << scale, osrc, odst)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert np.array_equal(nbg.nbg_vector_export_dense(ctx, deg), odeg)
    nbg.nbg_vector_free(ctx, deg)
    nbg.nbg_matrix_free(ctx, A)


def test_csr_from_host_edges_with_dups_and_loops(nbg, ctx):
    rng = np.random.default_rng(0)
    n = 300
    src = rng.integers(0, n, 5000).astype(np.int32)
    dst = rng.integers(0, n, 5000).astype(np.int32)
    src[:50] = dst[:50]                      # self loops
    src[50:100], dst[50:100] = src[100:150], dst[100:150]   # duplicates
    A, deg = nbg.nbg_matrix_from_edges(ctx, n, src, dst)
    rp, ci = nbg.nbg_matrix_export_csr(ctx, A)
    orp, oci, odeg = oracle.build_csr(n, src, dst)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert np.array_equal(nbg.nbg_vector_export_dense(ctx, deg), odeg)


def test_edges_out_of_range(nbg, ctx):
    with pytest.raises(nbg.NbgError) as e:
        nbg.nbg_matrix_from_edges(ctx, 10, np.array([1, 2], np.int32), np.array([3, 10], np.int32))
    assert e.value.status == nbg.INDEX_OUT_OF_BOUNDS


# ------------------------------------------------------------------ PageRank sweeps

def _graph(nbg, ctx, kind, scale, ef, seed):
    k = nbg.GRAPH_RMAT if kind == "rmat" else nbg.GRAPH_ER
    A, deg = nbg.nbg_matrix_from_generator(ctx, k, scale, ef, seed)
    src, dst = (oracle.rmat_edges if kind == "rmat" else oracle.er_edges)(scale, ef, seed)
    orp, oci, odeg = oracle.build_csr(1 << scale, src, dst)
    return A, deg, (orp, oci, odeg)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("uniform", [True, False])
def test_config1_fp64_20_sweeps(nbg, ctx, seed, uniform):
    A, deg, (orp, oci, odeg) = _graph(nbg, ctx, "rmat", 10, 8, seed)
    r, sweeps, hist = nbg.nbg_pagerank(ctx, A, deg, tol=-1.0, itermax=20, type=nbg.FP64,
                                       dangling=nbg.PR_UNIFORM if uniform else nbg.PR_DROP)
    ro, so, dho, _ = oracle.pagerank(orp, oci, odeg, dtype=np.float64, uniform=uniform, itermax=20)
    rv = nbg.nbg_vector_export_dense(ctx, r)
    assert sweeps == so == 20
    assert rel(rv, ro) <= 1e-10
    assert delta_close(hist, dho, ro, np.float64)
    if uniform:
        assert abs(rv.sum() - 1.0) < 1e-12


@pytest.mark.parametrize("scale,ef,kind", [(12, 16, "rmat"), (14, 8, "er"), (16, 16, "rmat")])
def test_fp32_fixed_sweeps(nbg, ctx, scale, ef, kind):
    A, deg, (orp, oci, odeg) = _graph(nbg, ctx, kind, scale, ef, 1)
    r, sweeps, hist = nbg.nbg_pagerank(ctx, A, deg, tol=-1.0, itermax=30, type=nbg.FP32)
    ro, so, dho, _ = oracle.pagerank(orp, oci, odeg, dtype=np.float32, itermax=30)
    rv = nbg.nbg_vector_export_dense(ctx, r)
    assert sweeps == so
    assert rel(rv, ro) <= 1e-5


def test_convergence_sweep_count_exact(nbg, ctx):
    A, deg, (orp, oci, odeg) = _graph(nbg, ctx, "rmat", 16, 16, 1)
    r, sweeps, hist = nbg.nbg_pagerank(ctx, A, deg, tol=1e-6, itermax=100, type=nbg.FP32)
    ro, so, dho, _ = oracle.pagerank(orp, oci, odeg, dtype=np.float32, itermax=100, tol=1e-6)
    assert sweeps == so
    assert rel(nbg.nbg_vector_export_dense(ctx, r), ro) <= 1e-5
    assert delta_close(hist, dho, ro, np.float32)


@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_blocking_equals_nonblocking_bitwise(nbg, ctx, bctx, T):
    t = nbg.FP32 if T == "fp32" else nbg.FP64
    res = []
    for c in (ctx, bctx):
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 12, 8, 9)
        r, sweeps, hist = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=12, type=t)
        res.append((nbg.nbg_vector_export_dense(c, r), hist))
    # ranks and deltas bit for bit in both types: the fused and the per-op kernels keep
    # the same rounding points, and the dangling mass / delta -- summed per SpMV task in the fused
    # kernel, per ewise thread in the per-op reduce -- are exact sums (fp64 terms: per-thread exact
    # accumulators), so their grouping does not matter
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])


def test_long_rows_star(nbg, ctx):
    # a hub with 50k in-edges: exercises the long-row chunk path + its ticket combine
    n = 60000
    src = np.arange(1, n, dtype=np.int32)
    dst = np.zeros(n - 1, np.int32)
    src = np.concatenate([src, np.array([0, 0], np.int32)])
    dst = np.concatenate([dst, np.array([1, 2], np.int32)])
    A, deg = nbg.nbg_matrix_from_edges(ctx, n, src, dst)
    orp, oci, odeg = oracle.build_csr(n, src, dst)
    for T, np_t, tol in ((nbg.FP64, np.float64, 1e-10), (nbg.FP32, np.float32, 1e-5)):
        r, sweeps, _ = nbg.nbg_pagerank(ctx, A, deg, tol=-1.0, itermax=10, type=T)
        ro, _, _, _ = oracle.pagerank(orp, oci, odeg, dtype=np_t, itermax=10)
        assert rel(nbg.nbg_vector_export_dense(ctx, r), ro) <= tol


def test_cycle_uniform_gpu(nbg, ctx):
    n = 1001
    src = np.arange(n, dtype=np.int32)
    dst = ((np.arange(n) + 1) % n).astype(np.int32)
    A, deg = nbg.nbg_matrix_from_edges(ctx, n, src, dst)
    r, _, _ = nbg.nbg_pagerank(ctx, A, deg, tol=-1.0, itermax=25, type=nbg.FP32)
    rv = nbg.nbg_vector_export_dense(ctx, r)
    assert np.all(rv == rv[0])
    assert abs(float(rv[0]) - float(np.float32(1 / n))) <= float(np.spacing(np.float32(1 / n)))


# ------------------------------------------------------------------ mxv semirings

@pytest.mark.parametrize("add", ["PLUS", "MIN", "MAX"])
@pytest.mark.parametrize("mul", ["TIMES", "SECOND", "FIRST", "PLUS"])
@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_mxv_semirings(nbg, ctx, add, mul, T):
    rng = np.random.default_rng(hash((add, mul, T)) % 2**32)
    n, m = 700, 4000                                  # ragged, several tiles
    lens = rng.integers(0, 40, n)
    lens[5] = 3000                                    # a long row (chunks)
    lens[7] = 200                                     # a medium row (warp path)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(m, int(l), replace=False)) for l in lens]).astype(np.int32)
    npT = np.float32 if T == "fp32" else np.float64
    vals = rng.random(ci.shape[0]).astype(npT)
    x = rng.random(m).astype(npT)
    t = nbg.TYPE_OF[T]
    A = nbg.nbg_matrix_from_csr(ctx, n, m, rp, ci, vals=vals, type=t)
    u = nbg.nbg_vector_from_dense(ctx, t, x)
    w = nbg.nbg_mxv(ctx, t, add, mul, A, u)
    got = nbg.nbg_vector_export_dense(ctx, w)
    exp = ops.mxv(add, mul, rp, ci, vals, x, npT)
    if add == "PLUS":
        assert rel(got[lens > 0], exp[lens > 0]) <= (2e-7 if T == "fp32" else 1e-14)
        assert np.all(got[lens == 0] == 0)
    else:
        assert np.array_equal(got, exp)


def test_mxv_iso_and_empty_input(nbg, ctx):
    rp = np.array([0, 2, 2, 5], np.int64)
    ci = np.array([0, 3, 1, 2, 3], np.int32)
    A = nbg.nbg_matrix_from_csr(ctx, 3, 4, rp, ci, type=nbg.FP64, iso=2.0)
    x = nbg.nbg_vector_new_const(ctx, nbg.FP64, 4, 1.5)
    w = nbg.nbg_mxv(ctx, nbg.FP64, "PLUS", "TIMES", A, x)
    assert np.array_equal(nbg.nbg_vector_export_dense(ctx, w), [6.0, 0.0, 9.0])
    e = nbg.nbg_vector_new(ctx, nbg.FP64, 4)
    w2 = nbg.nbg_mxv(ctx, nbg.FP64, "PLUS", "TIMES", A, e)      # dense output: identity everywhere
    assert np.array_equal(nbg.nbg_vector_export_dense(ctx, w2), [0.0, 0.0, 0.0])
    with pytest.raises(nbg.NbgError) as ex:
        nbg.nbg_mxv(ctx, nbg.FP64, "PLUS", "TIMES", A, nbg.nbg_vector_new_const(ctx, nbg.FP64, 5, 1.0))
    assert ex.value.status == nbg.DIMENSION_MISMATCH


# ------------------------------------------------------------------ elementwise chain (config 2)

def _chain(nbg, c, x, y, T, free=True):
    """z = ewise_mult(*, x, apply(v+1, y)); c1..c5; s = reduce(+)."""
    vx = nbg.nbg_vector_from_dense(c, T, x)
    vy = nbg.nbg_vector_from_dense(c, T, y)
    a = nbg.nbg_apply(c, T, "ADD_C", vy, 1.0)
    z = nbg.nbg_ewise_mult(c, T, "TIMES", vx, a)
    c1 = nbg.nbg_apply(c, T, "MUL_C", z, 0.5)
    c2 = nbg.nbg_ewise_add(c, T, "PLUS", c1, vx)
    c3 = nbg.nbg_ewise_mult(c, T, "TIMES", c2, vy)
    c4 = nbg.nbg_apply(c, T, "ABS_SUB_C", c3, 0.25)
    c5 = nbg.nbg_ewise_add(c, T, "MAX", c4, z)
    hs = [a, c1, c2, c3, c4]
    if free:
        for h in hs:
            nbg.nbg_vector_free(c, h)
    s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", c5)
    return s, z, c5, vx, vy


def _chain_oracle(x, y, npT):
    z = ops.ewise_mult("TIMES", x, ops.unop("ADD_C", y, npT, 1.0), npT)
    c1 = ops.unop("MUL_C", z, npT, 0.5)
    c2 = ops.ewise_add("PLUS", c1, x, npT)
    c3 = ops.ewise_mult("TIMES", c2, y, npT)
    c4 = ops.unop("ABS_SUB_C", c3, npT, 0.25)
    c5 = ops.ewise_add("MAX", c4, z, npT)
    return ops.reduce("PLUS", c5, np.float64), z, c5


@pytest.mark.parametrize("T", ["fp32", "fp64"])
@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_chain_fused_vs_blocking_vs_oracle(nbg, ctx, bctx, T, n):
    import inputs
    npT = np.float32 if T == "fp32" else np.float64
    x, y = inputs.uniform_vectors(n, 11, npT)
    t = nbg.TYPE_OF[T]
    outs = []
    for c in (ctx, bctx):
        s, z, c5, vx, vy = _chain(nbg, c, x, y, t)
        outs.append((nbg.nbg_scalar_get(c, s), nbg.nbg_vector_export_dense(c, z), nbg.nbg_vector_export_dense(c, c5)))
    so, zo, c5o = _chain_oracle(x, y, npT)
    for sv, zv, c5v in outs:
        assert np.array_equal(zv, zo) and np.array_equal(c5v, c5o)    # every element bit-exact (P11)
        assert abs(sv - so) <= 1e-12 * abs(so)
    assert np.array_equal(outs[0][1], outs[1][1])


def test_chain_fusion_counters(nbg):
    import inputs
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        x, y = inputs.uniform_vectors(1 << 16, 3, np.float32)
        nbg.nbg_reset_stats(c)
        s, z, c5, vx, vy = _chain(nbg, c, x, y, nbg.FP32)
        nbg.nbg_vector_free(c, c5)
        nbg.nbg_vector_free(c, z)
        nbg.nbg_scalar_get(c, s)
        st = nbg.nbg_get_stats(c)
        assert st["kernels_launched"] == 1            # one fused pass (Figs. 1-2)
        assert st["vectors_materialized"] == 0        # only the scalar: every intermediate elided
        assert st["plans_built"] == 1
        for _ in range(5):                            # same signature: cache hits only
            s2, z2, c52, vx2, vy2 = _chain(nbg, c, x, y, nbg.FP32)
            for h in (z2, c52, vx2, vy2):
                nbg.nbg_vector_free(c, h)
            nbg.nbg_scalar_get(c, s2)
        st = nbg.nbg_get_stats(c)
        assert st["plans_built"] == 1 and st["plan_hits"] == 5
    finally:
        nbg.nbg_finalize(c)


def test_pagerank_steady_state_one_kernel_per_sweep(nbg):
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 14, 16, 1)
        for _ in range(2):   # warm-up: plans, hints, hinted plans
            nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=10, type=nbg.FP32)
        nbg.nbg_reset_stats(c)
        r, sweeps, _ = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=10, type=nbg.FP32)
        st = nbg.nbg_get_stats(c)
        assert st["plans_built"] == 0 and st["jit_compiles"] == 0
        # dinv once + first sweep's prologue (y1, ds1 from the iso r0) + one fused kernel per sweep
        assert st["kernels_launched"] <= sweeps + 2, st
        assert st["side_outputs"] >= 2 * (sweeps - 1)
    finally:
        nbg.nbg_finalize(c)


# ------------------------------------------------------------------ gather layout (column relabel)

@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_relabel_is_bit_exact(nbg, T, monkeypatch):
    """The degree-sorted gather layout keeps every row's summation order: results with and
    without it are identical bit for bit."""
    t = nbg.TYPE_OF[T]
    out = {}
    monkeypatch.setenv("NBG_SPMV_TP", "0")      # the single-pass plan (the two-phase plan reorders sums)
    for flag in ("0", "1"):
        monkeypatch.setenv("NBG_RELABEL", flag)
        c = nbg.nbg_init(nbg.NONBLOCKING, 0)
        try:
            A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 13, 16, 4)
            res = []
            for _ in range(2):          # second run uses the speculative scattered side output
                r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=12, type=t)
                res.append((nbg.nbg_vector_export_dense(c, r), h))
            x = nbg.nbg_vector_from_dense(c, t, np.linspace(0, 1, 1 << 13).astype(nbg.NP_OF[t]))
            m = nbg.nbg_mxv(c, t, "PLUS", "SECOND", A, x)
            out[flag] = (res, nbg.nbg_vector_export_dense(c, m), nbg.nbg_get_stats(c))
        finally:
            nbg.nbg_finalize(c)
    for (r0, h0), (r1, h1) in zip(out["0"][0], out["1"][0]):
        assert np.array_equal(r0, r1)
        assert np.array_equal(h0, h1) if T == "fp32" else rel(h0, h1) <= 1e-12
    assert np.array_equal(out["0"][1], out["1"][1])
    assert out["1"][2]["side_outputs"] > 0


@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_two_phase_matches_oracle(nbg, T, monkeypatch):
    """The opt-in two-phase column-blocked SpMV against the oracle, and
    deterministic: two solves give identical bits."""
    monkeypatch.setenv("NBG_SPMV_TP", "1")
    t = nbg.TYPE_OF[T]
    npT = nbg.NP_OF[t]
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 16, 16, 5)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        odeg = nbg.nbg_vector_export_dense(c, deg)
        runs = []
        for _ in range(2):
            r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=10, type=t)
            runs.append((nbg.nbg_vector_export_dense(c, r), h))
        ro, so, dho, _ = oracle.pagerank(rp, ci, odeg, dtype=npT, itermax=10)
        assert np.array_equal(runs[0][0], runs[1][0])
        assert rel(runs[0][0], ro) <= (1e-5 if T == "fp32" else 1e-10)
        assert delta_close(runs[0][1], dho, ro, npT)
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("kind,scale,force", [("er", 12, None), ("er", 12, "0"), ("rmat", 12, "1"), ("rmat", 10, "1")])
def test_lane_per_row_spmv(nbg, monkeypatch, kind, scale, force):
    """The lane-per-row SpMV skeleton (low-skew matrices) -- chosen by skew for ER,
    forced on skewed R-MAT -- against the oracle, fused (nonblocking) and per-op (blocking)
    results identical for fp32 and within 1e-15 for fp64 (P9), both dangling variants."""
    if force is None:
        monkeypatch.delenv("NBG_SPMV_LPR", raising=False)
    else:
        monkeypatch.setenv("NBG_SPMV_LPR", force)
    g = nbg.GRAPH_ER if kind == "er" else nbg.GRAPH_RMAT
    res = {}
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            A, deg = nbg.nbg_matrix_from_generator(c, g, scale, 16, 2)
            rp, ci = nbg.nbg_matrix_export_csr(c, A)
            d = nbg.nbg_vector_export_dense(c, deg)
            for T, tol in (("fp32", 1e-5), ("fp64", 1e-10)):
                for dang in (nbg.PR_UNIFORM, nbg.PR_DROP):
                    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=12, dangling=dang, type=nbg.TYPE_OF[T])
                    v = nbg.nbg_vector_export_dense(c, r)
                    ro, so, dho, _ = oracle.pagerank(rp, ci, d, dtype=nbg.NP_OF[nbg.TYPE_OF[T]], itermax=12,
                                                     uniform=dang == nbg.PR_UNIFORM)
                    assert s == so == 12
                    assert rel(v, ro) <= tol
                    res[(mode, T, dang)] = v
        finally:
            nbg.nbg_finalize(c)
    for dang in (nbg.PR_UNIFORM, nbg.PR_DROP):
        assert np.array_equal(res[(nbg.NONBLOCKING, "fp32", dang)], res[(nbg.BLOCKING, "fp32", dang)])
        # fp64: the dangling sum's last bit may differ (see test_blocking_equals_nonblocking_bitwise)
        assert rel(res[(nbg.NONBLOCKING, "fp64", dang)], res[(nbg.BLOCKING, "fp64", dang)]) <= 1e-15


def test_mxv_degenerate_and_int(nbg, ctx):
    """Edge cases of the SpMV plan: no stored entries, a 1 x 1 matrix, integer semirings, and a
    wide iso matrix (>= 2^15 columns: the relabelled gather layout) against the oracle."""
    # nnz = 0: dense output, identity everywhere
    A0 = nbg.nbg_matrix_from_csr(ctx, 5, 3, np.zeros(6, np.int64), np.zeros(0, np.int32), type=nbg.FP32, iso=1.0)
    w0 = nbg.nbg_mxv(ctx, nbg.FP32, "MIN", "TIMES", A0, nbg.nbg_vector_from_dense(ctx, nbg.FP32, np.ones(3, np.float32)))
    assert np.all(nbg.nbg_vector_export_dense(ctx, w0) == np.inf)
    # 1 x 1
    A1 = nbg.nbg_matrix_from_csr(ctx, 1, 1, np.array([0, 1], np.int64), np.array([0], np.int32), type=nbg.FP64, iso=3.0)
    w1 = nbg.nbg_mxv(ctx, nbg.FP64, "PLUS", "TIMES", A1, nbg.nbg_vector_from_dense(ctx, nbg.FP64, np.array([2.5])))
    assert nbg.nbg_vector_export_dense(ctx, w1)[0] == 7.5
    rng = np.random.default_rng(17)
    # integer semirings on a ragged valued matrix
    n, m = 300, 500
    lens = rng.integers(0, 30, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(m, int(l), replace=False)) for l in lens]).astype(np.int32)
    for T, npT in ((nbg.INT32, np.int32), (nbg.INT64, np.int64)):
        vals = rng.integers(-5, 6, ci.shape[0]).astype(npT)
        x = rng.integers(-5, 6, m).astype(npT)
        A = nbg.nbg_matrix_from_csr(ctx, n, m, rp, ci, vals=vals, type=T)
        u = nbg.nbg_vector_from_dense(ctx, T, x)
        for add in ("PLUS", "MIN", "MAX"):
            got = nbg.nbg_vector_export_dense(ctx, nbg.nbg_mxv(ctx, T, add, "TIMES", A, u))
            assert np.array_equal(got, ops.mxv(add, "TIMES", rp, ci, vals, x, npT)), (T, add)
    # wide iso matrix: relabelled gather layout, hot cache + L2 gathers
    n, m = 2000, 70000
    lens = rng.integers(0, 60, n)
    lens[3] = 5000
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(m, int(l), replace=False)) for l in lens]).astype(np.int32)
    x = rng.random(m).astype(np.float32)
    A = nbg.nbg_matrix_from_csr(ctx, n, m, rp, ci, type=nbg.FP32, iso=1.0)
    got = nbg.nbg_vector_export_dense(ctx, nbg.nbg_mxv(ctx, nbg.FP32, "PLUS", "TIMES", A, nbg.nbg_vector_from_dense(ctx, nbg.FP32, x)))
    exp = ops.mxv("PLUS", "TIMES", rp, ci, None, x, np.float32)
    assert rel(got[lens > 0], exp[lens > 0]) <= 2e-7 and np.all(got[lens == 0] == 0)


@pytest.mark.parametrize("tname", ["bool", "int32", "int64", "fp32", "fp64"])
@pytest.mark.parametrize("mode", ["NONBLOCKING", "BLOCKING"])
def test_every_operator_every_type(nbg, tname, mode):
    """Every unary and binary operator of the ABI in every type against the oracle, element by
    element (one rounding in the output type on both sides; integer division by zero = 0, R2),
    on edge values: zeros, signs, large magnitudes, the integer extremes (wrapping arithmetic)."""
    npT = {"bool": np.bool_, "int32": np.int32, "int64": np.int64, "fp32": np.float32, "fp64": np.float64}[tname]
    t = nbg.TYPE_OF[tname]
    if np.dtype(npT).kind == "f":
        base = np.array([0.0, -0.0, 1.0, -2.5, 3.0, 1e-3, 7.25, -1e30, 1e30, 0.85], np.float64)
        c0, c1 = 2.5, -1.0
    elif npT is np.bool_:
        base = np.array([0, 1, 1, 0, 1], np.int64)
        c0, c1 = 1.0, 0.0
    else:
        info = np.iinfo(npT)
        base = np.array([0, 1, -1, 2, -7, 5, 1000, -1000, info.max, info.min], np.int64)
        c0, c1 = 3.0, -2.0
    u = np.resize(base, 97).astype(npT)
    v = np.resize(np.roll(base, 3), 97).astype(npT)
    dev_t = nbg.NP_OF[t]
    c = nbg.nbg_init(getattr(nbg, mode), 0)
    try:
        du = nbg.nbg_vector_from_dense(c, t, u.astype(dev_t))
        dv = nbg.nbg_vector_from_dense(c, t, v.astype(dev_t))
        for code in nbg.UNOPS:
            got = nbg.nbg_vector_export_dense(c, nbg.nbg_apply(c, t, code, du, c0, c1)).astype(npT)
            exp = ops.unop(code, u, npT, c0, c1)
            assert np.array_equal(got, exp, equal_nan=np.dtype(npT).kind == "f"), (tname, code)
        for code in nbg.BINOPS:
            for rec, fn in ((nbg.nbg_ewise_add, ops.ewise_add), (nbg.nbg_ewise_mult, ops.ewise_mult)):
                got = nbg.nbg_vector_export_dense(c, rec(c, t, code, du, dv, 0.85)).astype(npT)
                exp = fn(code, u, v, npT, 0.85)
                assert np.array_equal(got, exp, equal_nan=np.dtype(npT).kind == "f"), (tname, code)
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("mode", ["NONBLOCKING", "BLOCKING"])
def test_convert_and_reduce_every_type(nbg, mode):
    """convert between every pair of types (in-range values: C conversion rules, float -> int
    truncates toward zero; out-of-range float -> int is undefined in C and not tested) and reduce
    with every monoid in every type (integer sums exact, float sums within 1e-12 of the exact sum)."""
    names = ["bool", "int32", "int64", "fp32", "fp64"]
    npT = {"bool": np.bool_, "int32": np.int32, "int64": np.int64, "fp32": np.float32, "fp64": np.float64}
    rng = np.random.default_rng(4)
    src = {"bool": rng.integers(0, 2, 301).astype(np.bool_),
           "int32": rng.integers(-100000, 100000, 301).astype(np.int32),
           "int64": rng.integers(-100000, 100000, 301).astype(np.int64),
           "fp32": ((rng.random(301) - 0.5) * 2e4).astype(np.float32),
           "fp64": (rng.random(301) - 0.5) * 2e4}
    c = nbg.nbg_init(getattr(nbg, mode), 0)
    try:
        for a in names:
            ta = nbg.TYPE_OF[a]
            du = nbg.nbg_vector_from_dense(c, ta, src[a].astype(nbg.NP_OF[ta]))
            for b in names:
                tb = nbg.TYPE_OF[b]
                got = nbg.nbg_vector_export_dense(c, nbg.nbg_convert(c, tb, du)).astype(npT[b])
                assert np.array_equal(got, ops.convert(src[a], npT[b])), (a, b)
            for mono in ("PLUS", "MIN", "MAX"):
                for rt in ("int64", "fp64") if mono == "PLUS" else (a,):
                    s = nbg.nbg_reduce(c, nbg.TYPE_OF[rt], mono, du)
                    exp = float(ops.reduce(mono, ops.convert(src[a], npT[rt]), npT[rt]))
                    got = nbg.nbg_scalar_get(c, s)
                    if mono == "PLUS" and rt == "fp64":
                        assert abs(got - exp) <= 1e-12 * float(np.abs(src[a].astype(np.float64)).sum()), (a, mono, rt)
                    else:
                        assert got == exp, (a, mono, rt)
    finally:
        nbg.nbg_finalize(c)


def test_degenerate_sizes(nbg):
    """Length-0 vectors through every op (both modes), graphs with no edges / only self-loops /
    only duplicates, and PageRank on a 1-vertex graph: bit-exact against the oracle."""
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            z = nbg.nbg_vector_from_dense(c, nbg.FP64, np.zeros(0, np.float64))
            e = nbg.nbg_ewise_add(c, nbg.FP64, "PLUS", nbg.nbg_apply(c, nbg.FP64, "ABS", z), z)
            assert nbg.nbg_vector_export_dense(c, e).shape[0] == 0
            assert nbg.nbg_scalar_get(c, nbg.nbg_reduce(c, nbg.FP64, "PLUS", e)) == 0.0
            assert nbg.nbg_scalar_get(c, nbg.nbg_reduce(c, nbg.FP64, "MAX", z)) == -np.inf
            sp = nbg.nbg_vector_from_sparse(c, nbg.FP32, 0, np.zeros(0, np.int32), np.zeros(0, np.float32))
            assert nbg.nbg_vector_nvals(c, sp) == 0
            # graphs
            for n, src, dst in ((5, [], []), (4, [0, 1, 2, 3], [0, 1, 2, 3]), (3, [0, 0, 0, 2], [1, 1, 1, 1]), (1, [0], [0])):
                s = np.array(src, np.int32)
                d = np.array(dst, np.int32)
                A, deg = nbg.nbg_matrix_from_edges(c, n, s, d)
                rp, ci = nbg.nbg_matrix_export_csr(c, A)
                orp, oci, odeg = oracle.build_csr(n, s, d)
                assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
                assert np.array_equal(nbg.nbg_vector_export_dense(c, deg), odeg)
                r, sw, _ = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=5, type=nbg.FP64)
                ro, so, _, _ = oracle.pagerank(orp, oci, odeg, dtype=np.float64, itermax=5)
                assert sw == so and rel(nbg.nbg_vector_export_dense(c, r), ro) <= 1e-14, (n, src, dst)
        finally:
            nbg.nbg_finalize(c)


@pytest.mark.parametrize("n,hubs,m", [(4000, 3, 60000), (5000, 1, 40000), (9000, 2, 70000)])
def test_small_matrix_with_long_rows(nbg, ctx, n, hubs, m):
    """Small matrices (fewer than 4 x SMs 128-row tasks) run 32-row warp tasks; rows longer than
    512 groups (2048 entries) are still cut into chunks combined by a ticket: both together, fp32
    and fp64, PageRank and plain mxv against the oracle."""
    rng = np.random.default_rng(n + m)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = np.where(rng.random(m) < 0.8, rng.integers(0, hubs, m), rng.integers(0, n, m)).astype(np.int32)
    A, deg = nbg.nbg_matrix_from_edges(ctx, n, src, dst)
    orp, oci, odeg = oracle.build_csr(n, src, dst)
    lens = np.diff(orp)
    assert int(lens.max()) > 2048                                  # at least one chunked row
    for T, npT, tolr in ((nbg.FP32, np.float32, 1e-5), (nbg.FP64, np.float64, 1e-12)):
        r, sw, hist = nbg.nbg_pagerank(ctx, A, deg, tol=-1.0, itermax=15, type=T)
        ro, so, dho, _ = oracle.pagerank(orp, oci, odeg, dtype=npT, itermax=15)
        assert sw == so
        assert rel(nbg.nbg_vector_export_dense(ctx, r), ro) <= tolr
        x = rng.random(n).astype(npT)
        got = nbg.nbg_vector_export_dense(ctx, nbg.nbg_mxv(ctx, T, "PLUS", "TIMES", A, nbg.nbg_vector_from_dense(ctx, T, x)))
        exp = ops.mxv("PLUS", "TIMES", orp, oci, None, x, npT)
        assert rel(got[lens > 0], exp[lens > 0]) <= (2e-7 if T == nbg.FP32 else 1e-14) and np.all(got[lens == 0] == 0)


# ------------------------------------------------------------------ C ABI: wait_all, deterministic flag

def test_wait_all_materialises_live_pending_nodes_only(nbg):
    """nbg_wait_all: every pending node a handle reaches is materialised in one
    planning pass; nodes no handle reaches stay elided; values match the oracle."""
    import inputs
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        x, y = inputs.uniform_vectors(1 << 14, 5, np.float64)
        vx = nbg.nbg_vector_from_dense(c, nbg.FP64, x)
        vy = nbg.nbg_vector_from_dense(c, nbg.FP64, y)
        a = nbg.nbg_apply(c, nbg.FP64, "ADD_C", vy, 1.0)              # freed below: elided
        z = nbg.nbg_ewise_mult(c, nbg.FP64, "TIMES", vx, a)           # live
        w = nbg.nbg_ewise_add(c, nbg.FP64, "MAX", z, vx)              # live
        s = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, w)                  # live scalar
        nbg.nbg_vector_free(c, a)
        assert not nbg.nbg_vector_is_materialized(c, z) and not nbg.nbg_vector_is_materialized(c, w)
        nbg.nbg_reset_stats(c)
        nbg.nbg_wait_all(c)
        st = nbg.nbg_get_stats(c)
        assert nbg.nbg_vector_is_materialized(c, z) and nbg.nbg_vector_is_materialized(c, w)
        assert st["kernels_launched"] == 1 and st["vectors_materialized"] == 2, st   # one fused pass, `a` elided
        nbg.nbg_wait_all(c)                                            # idempotent: nothing left
        assert nbg.nbg_get_stats(c)["kernels_launched"] == 1
        zo = ops.binop("TIMES", x, ops.unop("ADD_C", y, np.float64, 1.0), np.float64)
        wo = ops.binop("MAX", zo, x, np.float64)
        assert np.array_equal(nbg.nbg_vector_export_dense(c, z), zo)
        assert np.array_equal(nbg.nbg_vector_export_dense(c, w), wo)
        assert rel([nbg.nbg_scalar_get(c, s)], [ops.reduce("PLUS", wo, np.float64)]) <= 1e-12
    finally:
        nbg.nbg_finalize(c)


def test_deterministic_flag_and_run_to_run_bits(nbg):
    """nbg_config.flags = NBG_FLAG_DETERMINISTIC is accepted; results are bit-reproducible run to
    run with or without it (exact cross-block combine, plan-fixed row order)."""
    outs = []
    for flags in (nbg.FLAG_DETERMINISTIC, 0, nbg.FLAG_DETERMINISTIC):
        c = nbg.nbg_init(nbg.NONBLOCKING, 0, flags=flags)
        try:
            A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 14, 16, 4)
            r, sweeps, hist = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=8, type=nbg.FP64)
            outs.append((nbg.nbg_vector_export_dense(c, r), np.asarray(hist)))
        finally:
            nbg.nbg_finalize(c)
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


@pytest.mark.parametrize("mode", ["NONBLOCKING", "BLOCKING"])
def test_fp64_plus_reduce_is_the_exactly_rounded_sum(nbg, mode):
    """fp64 PLUS reductions are exact sums rounded once (per-thread exact accumulators + exact
    cross-block limbs): equal to math.fsum bit for bit, also with cancellation and wide exponent
    ranges, standalone and fused behind elementwise operators."""
    import math
    c = nbg.nbg_init(getattr(nbg, mode), 0)
    try:
        rng = np.random.default_rng(21)
        for n, spread in ((1, 10), (1000, 5), (100003, 60), (1 << 20, 30), (77777, 100)):   # inside [2^-160, 2^128)
            v = np.ldexp(rng.standard_normal(n), rng.integers(-spread, spread, n))
            if n > 10:
                v[::7] = -v[1::7][: v[::7].shape[0]] if v[1::7].shape[0] >= v[::7].shape[0] else v[::7]
            u = nbg.nbg_vector_from_dense(c, nbg.FP64, v)
            s = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, u)
            assert nbg.nbg_scalar_get(c, s) == math.fsum(v), n
            w = nbg.nbg_apply(c, nbg.FP64, "ABS", u)
            s2 = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, w)
            assert nbg.nbg_scalar_get(c, s2) == math.fsum(np.abs(v)), n
    finally:
        nbg.nbg_finalize(c)


def test_deferred_scalar_readbacks_any_order(nbg):
    """Scalar readbacks are deferred to the first host read and copied in bulk (runtime.cpp
    issue_readback): many held reductions read in reverse, interleaved with new launches, with
    freed neighbours in the same slab and more than the deferred list's compaction threshold --
    every value is its own exactly rounded sum (math.fsum), whatever order the copies happen in."""
    import math
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        rng = np.random.default_rng(5)
        vecs = [np.ldexp(rng.standard_normal(1000 + 37 * k), rng.integers(-20, 20, 1000 + 37 * k)) for k in range(300)]
        held, expect = [], []
        for k, v in enumerate(vecs):
            u = nbg.nbg_vector_from_dense(c, nbg.FP64, v)
            s = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, u)
            nbg.nbg_scalar_wait(c, s)                       # materialised: marked readable, not copied
            nbg.nbg_vector_free(c, u)
            if k % 3 == 2:
                nbg.nbg_scalar_free(c, s)                   # a freed neighbour inside the copied range
                continue
            held.append(s)
            expect.append(math.fsum(v))
            if k % 50 == 49:                                # read a middle one while later ones exist
                j = len(held) // 2
                assert nbg.nbg_scalar_get(c, held[j]) == expect[j]
        for s, e in reversed(list(zip(held, expect))):
            assert nbg.nbg_scalar_get(c, s) == e
        for s, e in zip(held, expect):                      # second reads hit the copied mirror
            assert nbg.nbg_scalar_get(c, s) == e
            nbg.nbg_scalar_free(c, s)
    finally:
        nbg.nbg_finalize(c)


def test_tma_staged_ewise_skeleton_matches(nbg, monkeypatch):
    """The opt-in TMA-staged elementwise skeleton (NBG_EWISE_TMA=1: inputs staged in shared
    memory by cp.async.bulk on mbarriers) gives the register skeleton's results bit for bit, with
    whole tiles, a ragged vector tail and a scalar tail, fp32 / fp64 / int32 inputs and an exact
    fp64 reduction."""
    import math
    rng = np.random.default_rng(8)
    data = []
    for n in (1 << 20, (1 << 20) + 2048 * 3 + 4 * 7 + 3, 4099):
        data.append((rng.standard_normal(n).astype(np.float32), rng.standard_normal(n), rng.integers(-5, 5, n).astype(np.int32)))
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("NBG_EWISE_TMA", mode)
        c = nbg.nbg_init(nbg.NONBLOCKING, 0)     # the mode is read at every region (planner.cpp)
        try:
            out = []
            for x, y, k in data:
                u = nbg.nbg_vector_from_dense(c, nbg.FP32, x)
                v = nbg.nbg_vector_from_dense(c, nbg.FP64, y)
                w = nbg.nbg_vector_from_dense(c, nbg.INT32, k)
                z = nbg.nbg_ewise_mult(c, nbg.FP64, "TIMES", nbg.nbg_ewise_add(c, nbg.FP64, "PLUS", u, v), w)
                s = nbg.nbg_reduce(c, nbg.FP64, nbg.PLUS, z)
                zz = nbg.nbg_vector_export_dense(c, z)
                ref = (x.astype(np.float64) + y) * k
                assert np.array_equal(zz, ref)
                assert nbg.nbg_scalar_get(c, s) == math.fsum(ref)
                out.append(zz)
            res[mode] = out
        finally:
            nbg.nbg_finalize(c)
    for a, b in zip(res["0"], res["1"]):
        assert np.array_equal(a, b)
