"""GPU parity of sparse / bitset vectors through the C ABI against
oracle/sparse.py: every element bit-exact (each value is one rounding in its type on both sides),
structure (present indices) exact, reductions exact (fixed-point accumulation vs math.fsum), in
blocking and nonblocking mode, over fills that exercise both loops (index list / full range) and
all three output representations; the estimator formulas through nbg_vector_estimated_fill.
"""
import numpy as np
import pytest

from oracle import ops
from oracle import sparse as S

pytestmark = pytest.mark.gpu
N = 100_003          # not a multiple of 32: ragged last bitset word


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


def rsv(rng, n, fill, T):
    idx = np.nonzero(rng.random(n) < fill)[0]
    if np.dtype(T).kind == "f":
        vals = (rng.random(idx.shape[0]) * 4 - 2).astype(T)
    else:
        vals = rng.integers(-50, 50, idx.shape[0]).astype(T)
    return S.sparse(n, idx, vals)


def put(nbg, c, t, sv):
    return nbg.nbg_vector_from_sparse(c, t, sv.n, sv.idx.astype(np.int32), np.ascontiguousarray(sv.vals))


def get(nbg, c, v, n):
    i, x = nbg.nbg_vector_export_sparse(c, v)
    return S.SV(n, i.astype(np.int64), x)


def same(a, b):
    assert np.array_equal(a.idx, b.idx), f"structure differs ({a.idx.shape[0]} vs {b.idx.shape[0]} entries)"
    assert a.vals.dtype == b.vals.dtype
    assert np.array_equal(a.vals.view(np.uint8), np.ascontiguousarray(b.vals).view(np.uint8)), "values differ"


def test_roundtrip_formats_and_errors(nbg):
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        rng = np.random.default_rng(1)
        for fill in (0.0, 0.001, 0.3, 1.0):
            u = rsv(rng, N, fill, np.float32)
            v = put(nbg, c, nbg.FP32, u)
            same(get(nbg, c, v, N), u)
            assert nbg.nbg_vector_nvals(c, v) == u.idx.shape[0]
            fmt = nbg.nbg_vector_format(c, v)
            assert fmt == (nbg.FORMAT_EMPTY if fill == 0.0 else nbg.FORMAT_FULL if fill == 1.0 else nbg.FORMAT_SPARSE)
        f = nbg.nbg_vector_from_dense(c, nbg.FP64, np.arange(7, dtype=np.float64))
        same(get(nbg, c, f, 7), S.full(np.arange(7, dtype=np.float64)))
        bad = [(np.array([3, 1], np.int32), nbg.INVALID_VALUE), (np.array([1, 1], np.int32), nbg.INVALID_VALUE),
               (np.array([0, 10], np.int32), nbg.INDEX_OUT_OF_BOUNDS), (np.array([-1, 2], np.int32), nbg.INDEX_OUT_OF_BOUNDS)]
        for idx, st in bad:
            with pytest.raises(nbg.NbgError) as e:
                nbg.nbg_vector_from_sparse(c, nbg.FP32, 10, idx, np.ones(2, np.float32))
            assert e.value.status == st
        s = put(nbg, c, nbg.FP32, S.sparse(10, [2], np.ones(1, np.float32)))
        with pytest.raises(nbg.NbgError) as e:
            nbg.nbg_vector_export_dense(c, s)
        assert e.value.status == nbg.INVALID_OBJECT
    finally:
        nbg.nbg_finalize(c)


FILLS = [(0.002, 0.01), (0.04, 0.3), (0.45, 0.9)]


@pytest.mark.parametrize("mode", ["BLOCKING", "NONBLOCKING"])
@pytest.mark.parametrize("tname", ["fp32", "fp64", "int32"])
@pytest.mark.parametrize("fu,fv", FILLS)
def test_ops_match_oracle(nbg, mode, tname, fu, fv):
    T = {"fp32": np.float32, "fp64": np.float64, "int32": np.int32}[tname]
    t = nbg.TYPE_OF[tname]
    rng = np.random.default_rng(int(fu * 1000) + 7 * int(fv * 1000))
    u, v = rsv(rng, N, fu, T), rsv(rng, N, fv, T)
    fvals = rsv(rng, N, 1.0, T).vals
    f = S.full(fvals)
    c = nbg.nbg_init(getattr(nbg, mode), 0)
    try:
        du, dv = put(nbg, c, t, u), put(nbg, c, t, v)
        df = nbg.nbg_vector_from_dense(c, t, fvals)
        st0 = nbg.nbg_get_stats(c)
        # intersection, union, mixed chain, bind2nd, union with a full vector
        g1 = nbg.nbg_ewise_mult(c, t, "TIMES", du, dv)
        g2 = nbg.nbg_ewise_add(c, t, "PLUS", du, dv)
        g3 = nbg.nbg_ewise_add(c, t, "MAX", nbg.nbg_apply(c, t, "MUL_C", du, 3.0), nbg.nbg_ewise_mult(c, t, "MINUS", dv, df))
        s = nbg.nbg_scalar_new(c, t, 2.0)
        g4 = nbg.nbg_apply_bind2nd(c, t, "MINUS", du, s)
        g5 = nbg.nbg_ewise_add(c, t, "PLUS", du, df)
        r1 = nbg.nbg_reduce(c, nbg.FP64, "PLUS", nbg.nbg_ewise_mult(c, t, "TIMES", du, df))
        r2 = nbg.nbg_reduce(c, t, "MAX", g2)
        e1 = S.ewise_mult("TIMES", u, v, T)
        e2 = S.ewise_add("PLUS", u, v, T)
        e3 = S.ewise_add("MAX", S.apply("MUL_C", u, T, 3.0), S.ewise_mult("MINUS", v, f, T), T)
        e4 = S.bind2nd("MINUS", u, 2.0, T)
        e5 = S.ewise_add("PLUS", u, f, T)
        for g, e in ((g1, e1), (g2, e2), (g3, e3), (g4, e4), (g5, e5)):
            same(get(nbg, c, g, N), e)
        assert nbg.nbg_vector_format(c, g5) == nbg.FORMAT_FULL
        fmt1 = nbg.nbg_vector_format(c, g1)
        exp_fill = S.fill_mult(S.fill(u), S.fill(v))
        if e1.idx.shape[0] == 0:
            assert fmt1 == nbg.FORMAT_EMPTY
        else:
            assert fmt1 == (nbg.FORMAT_SPARSE if exp_fill <= 1 / 16 else nbg.FORMAT_BITSET)
        # float PLUS: per-thread fp64 partials, exact combine -> within 1e-12 of the exact sum's scale
        # (the C2 reduce tolerance); integer sums are exact
        prod = S.ewise_mult("TIMES", u, f, T)
        scale = float(np.abs(prod.vals.astype(np.float64)).sum())
        assert abs(nbg.nbg_scalar_get(c, r1) - S.reduce("PLUS", prod, np.float64)) <= 1e-12 * max(scale, 1e-300)
        assert nbg.nbg_scalar_get(c, r2) == float(S.reduce("MAX", e2, T))
        st1 = nbg.nbg_get_stats(c)
        assert st1["structured_regions"] > st0["structured_regions"]
        if fu + fv < 0.5:
            assert st1["structured_index_loops"] > st0["structured_index_loops"]     # sparse driver chosen
    finally:
        nbg.nbg_finalize(c)


def test_estimated_fill(nbg):
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        rng = np.random.default_rng(5)
        u, v = rsv(rng, N, 0.2, np.float32), rsv(rng, N, 0.05, np.float32)
        du, dv = put(nbg, c, nbg.FP32, u), put(nbg, c, nbg.FP32, v)
        fu, fv = S.fill(u), S.fill(v)
        assert nbg.nbg_vector_estimated_fill(c, du) == fu
        m = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", du, dv)
        a = nbg.nbg_ewise_add(c, nbg.FP32, "PLUS", nbg.nbg_apply(c, nbg.FP32, "ABS", du), dv)
        assert nbg.nbg_vector_estimated_fill(c, m) == pytest.approx(S.fill_mult(fu, fv), rel=1e-15)
        assert nbg.nbg_vector_estimated_fill(c, a) == pytest.approx(S.fill_add(fu, fv), rel=1e-15)
        assert not nbg.nbg_vector_is_materialized(c, m)          # the estimate does not materialise
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("add,mul", [("PLUS", "TIMES"), ("PLUS", "SECOND"), ("MIN", "PLUS"), ("MAX", "TIMES")])
def test_mxv_structured_x(nbg, add, mul):
    import oracle
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, _ = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 12, 8, 3)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        n = rp.shape[0] - 1
        rng = np.random.default_rng(11)
        for fill in (0.01, 0.5):
            x = rsv(rng, n, fill, np.float64)
            x.vals[:] = np.round(x.vals * 8)                  # small integers: every fp64 sum is exact
            dx = put(nbg, c, nbg.FP64, x)
            y = nbg.nbg_mxv(c, nbg.FP64, add, mul, A, dx)
            got = nbg.nbg_vector_export_dense(c, y)
            exp = S.mxv(add, mul, rp, ci, None, x, np.float64)
            assert np.array_equal(got, exp)
            # a structured x feeding a fused dense region: z = 0.5 * (A x) + 1 reduced
            z = nbg.nbg_apply(c, nbg.FP64, "AXPB", nbg.nbg_mxv(c, nbg.FP64, add, mul, A, dx), 0.5, 1.0)
            zs = nbg.nbg_reduce(c, nbg.FP64, "PLUS", z)
            assert nbg.nbg_scalar_get(c, zs) == ops.reduce("PLUS", ops.unop("AXPB", exp, np.float64, 0.5, 1.0), np.float64)
    finally:
        nbg.nbg_finalize(c)


def test_empty_and_disjoint(nbg):
    c = nbg.nbg_init(nbg.BLOCKING, 0)
    try:
        a = put(nbg, c, nbg.FP32, S.sparse(64, [1, 3, 5], np.ones(3, np.float32)))
        b = put(nbg, c, nbg.FP32, S.sparse(64, [0, 2, 4], np.ones(3, np.float32)))
        m = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", a, b)
        assert nbg.nbg_vector_format(c, m) == nbg.FORMAT_EMPTY and nbg.nbg_vector_nvals(c, m) == 0
        assert nbg.nbg_vector_export_sparse(c, m)[0].shape[0] == 0
        assert nbg.nbg_scalar_get(c, nbg.nbg_reduce(c, nbg.FP32, "MIN", m)) == np.inf
        u = nbg.nbg_ewise_add(c, nbg.FP32, "PLUS", a, b)
        i, v = nbg.nbg_vector_export_sparse(c, u)
        assert list(i) == [0, 1, 2, 3, 4, 5] and np.all(v == 1)
    finally:
        nbg.nbg_finalize(c)


def test_pending_result_materialised_empty(nbg):
    """A pending structured node that materialises with no entries, used afterwards by operations
    recorded before it was materialised (empty operand inside a region, reduce of it, mxv of it)."""
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        n = 1024
        a = put(nbg, c, nbg.FP32, S.sparse(n, [1, 3, 5], np.ones(3, np.float32)))
        b = put(nbg, c, nbg.FP32, S.sparse(n, [0, 2, 4], np.ones(3, np.float32)))
        f = nbg.nbg_vector_from_dense(c, nbg.FP32, np.full(n, 2.0, np.float32))
        m = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", a, b)             # empty, still pending
        u = nbg.nbg_ewise_add(c, nbg.FP32, "PLUS", m, b)               # recorded on the pending m
        w = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", m, f)
        s = nbg.nbg_reduce(c, nbg.FP32, "MIN", m)
        A, _ = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_ER, 10, 4, 1)
        y = nbg.nbg_mxv(c, nbg.FP32, "PLUS", "TIMES", A, m)
        assert nbg.nbg_vector_format(c, m) == nbg.FORMAT_EMPTY         # m materialised now
        i, v = nbg.nbg_vector_export_sparse(c, u)
        assert list(i) == [0, 2, 4] and np.all(v == 1)
        assert nbg.nbg_vector_nvals(c, w) == 0
        assert nbg.nbg_scalar_get(c, s) == np.inf
        assert np.all(nbg.nbg_vector_export_dense(c, y) == 0)
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("mode", ["BLOCKING", "NONBLOCKING"])
@pytest.mark.parametrize("tname", ["fp64", "int64"])
def test_bitset_operands_chain(nbg, mode, tname):
    """Results kept as bitsets (fill above 1/16) feeding later regions: a bitset operand in the
    index loop (bit test at the driver's indices) and in the full-range loop, user-held
    intermediates, int64 values."""
    T = {"fp64": np.float64, "int64": np.int64}[tname]
    t = nbg.TYPE_OF[tname]
    rng = np.random.default_rng(21)
    u, v, w = rsv(rng, N, 0.3, T), rsv(rng, N, 0.35, T), rsv(rng, N, 0.01, T)
    c = nbg.nbg_init(getattr(nbg, mode), 0)
    try:
        du, dv, dw = put(nbg, c, t, u), put(nbg, c, t, v), put(nbg, c, t, w)
        b = nbg.nbg_ewise_add(c, t, "MIN", du, dv)                          # fill ~0.55: bitset
        eb = S.ewise_add("MIN", u, v, T)
        same(get(nbg, c, b, N), eb)
        assert nbg.nbg_vector_format(c, b) == nbg.FORMAT_BITSET
        m = nbg.nbg_ewise_mult(c, t, "PLUS", b, dw)                         # driven by w (1 %)
        e = nbg.nbg_apply(c, t, "AINV", b)
        x = nbg.nbg_ewise_add(c, t, "MAX", e, dw)
        s = nbg.nbg_reduce(c, nbg.INT64 if tname == "int64" else nbg.FP64, "PLUS", b)
        same(get(nbg, c, m, N), S.ewise_mult("PLUS", eb, w, T))
        ee = S.apply("AINV", eb, T)
        same(get(nbg, c, e, N), ee)
        same(get(nbg, c, x, N), S.ewise_add("MAX", ee, w, T))
        exp = S.reduce("PLUS", eb, np.int64 if tname == "int64" else np.float64)
        got = nbg.nbg_scalar_get(c, s)
        if tname == "int64":
            assert got == exp
        else:
            assert abs(got - exp) <= 1e-12 * float(np.abs(eb.vals).sum())
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("tname", ["bool", "int32", "fp32", "fp64"])
def test_every_operator_structured(nbg, tname):
    """Every unary and binary operator over sparse operands (structure and values vs the oracle),
    both representations of the result (fills around the sparse / bitset threshold)."""
    T = {"bool": np.bool_, "int32": np.int32, "fp32": np.float32, "fp64": np.float64}[tname]
    t = nbg.TYPE_OF[tname]
    rng = np.random.default_rng(33)
    n = 5000
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        for fill in (0.02, 0.4):
            u, v = rsv(rng, n, fill, np.float64), rsv(rng, n, fill, np.float64)
            if T is np.bool_:
                u.vals[:] = rng.integers(0, 2, u.vals.shape[0]); v.vals[:] = rng.integers(0, 2, v.vals.shape[0])
            u.vals = u.vals.astype(T); v.vals = v.vals.astype(T)
            dev = nbg.NP_OF[t]
            du = nbg.nbg_vector_from_sparse(c, t, n, u.idx.astype(np.int32), u.vals.astype(dev))
            dv = nbg.nbg_vector_from_sparse(c, t, n, v.idx.astype(np.int32), v.vals.astype(dev))
            eq = (lambda a, b: np.array_equal(a, b, equal_nan=True)) if np.dtype(T).kind == "f" else np.array_equal
            for code in nbg.UNOPS:
                i, x = nbg.nbg_vector_export_sparse(c, nbg.nbg_apply(c, t, code, du, 2.5, -1.0))
                e = S.apply(code, u, T, 2.5, -1.0)
                assert np.array_equal(i, e.idx) and eq(x.astype(T), e.vals), (tname, fill, code)
            for code in nbg.BINOPS:
                for rec, fn in ((nbg.nbg_ewise_add, S.ewise_add), (nbg.nbg_ewise_mult, S.ewise_mult)):
                    i, x = nbg.nbg_vector_export_sparse(c, rec(c, t, code, du, dv, 0.85))
                    e = fn(code, u, v, T, 0.85)
                    assert np.array_equal(i, e.idx) and eq(x.astype(T), e.vals), (tname, fill, code, fn.__name__)
    finally:
        nbg.nbg_finalize(c)
