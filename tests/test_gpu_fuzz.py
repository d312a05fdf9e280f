"""Random operation DAGs through the planner (fusion, liveness, memo, scalar operands) against the
oracle: every requested vector element by element, every requested reduction within 1e-12 of the
exact sum scale; nonblocking (fused) and blocking (one kernel per op) in one run per program.
Includes sparse operands, so structured regions and dense regions meet in one DAG.
"""
import numpy as np
import pytest

from oracle import ops
from oracle import sparse as S

pytestmark = pytest.mark.gpu
UN = ["IDENTITY", "AINV", "ABS", "ADD_C", "MUL_C", "AXPB", "ABS_SUB_C", "ISZERO"]
BIN = ["PLUS", "MINUS", "TIMES", "MIN", "MAX", "FIRST", "SECOND", "ABSDIFF"]


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


def _program(rng, n_ops):
    """A random SSA program: ('leaf', k) | ('un', code, a, c0, c1) | ('bin', kind, code, a, b) |
    ('bind', code, a, s) with s a reduce of an earlier vector."""
    prog = [("leaf", 0), ("leaf", 1), ("leaf", 2)]
    for _ in range(n_ops):
        r = rng.random()
        a = int(rng.integers(0, len(prog)))
        if r < 0.35:
            prog.append(("un", UN[rng.integers(0, len(UN))], a, float(rng.integers(-3, 4)) / 2, float(rng.integers(-3, 4)) / 4))
        elif r < 0.85:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bin", "add" if rng.random() < 0.5 else "mult", BIN[rng.integers(0, len(BIN))], a, b))
        else:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bind", BIN[rng.integers(0, 5)], a, b))
    return prog


def _oracle(prog, leaves, T):
    vals = []
    for ins in prog:
        if ins[0] == "leaf":
            vals.append(leaves[ins[1]])
        elif ins[0] == "un":
            vals.append(S.apply(ins[1], vals[ins[2]], T, ins[3], ins[4]))
        elif ins[0] == "bin":
            f = S.ewise_add if ins[1] == "add" else S.ewise_mult
            vals.append(f(ins[2], vals[ins[3]], vals[ins[4]], T))
        else:
            s = S.reduce("PLUS", vals[ins[3]], np.float64)
            vals.append(S.bind2nd(ins[1], vals[ins[2]], T.type(s) if hasattr(T, "type") else np.dtype(T).type(s), T))
    return vals


@pytest.mark.parametrize("seed", range(12))
def test_random_dags(nbg, seed):
    rng = np.random.default_rng(1000 + seed)
    T = np.float64
    n = 3001
    leaves = [S.full((rng.integers(-8, 9, n) / 4.0).astype(T)), S.full((rng.integers(-8, 9, n) / 4.0).astype(T))]
    sp = seed % 2 == 1                     # odd seeds: the third leaf is sparse
    if sp:
        idx = np.nonzero(rng.random(n) < 0.1)[0]
        leaves.append(S.sparse(n, idx, (rng.integers(-8, 9, idx.shape[0]) / 4.0).astype(T)))
    else:
        leaves.append(S.full((rng.integers(-8, 9, n) / 4.0).astype(T)))
    prog = _program(rng, 14)
    exp = _oracle(prog, leaves, T)
    want = sorted(set(int(k) for k in rng.integers(3, len(prog), 4)))
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            h = []
            for ins in prog:
                if ins[0] == "leaf":
                    L = leaves[ins[1]]
                    if L.idx.shape[0] == n:
                        h.append(nbg.nbg_vector_from_dense(c, nbg.FP64, L.vals))
                    else:
                        h.append(nbg.nbg_vector_from_sparse(c, nbg.FP64, n, L.idx.astype(np.int32), L.vals))
                elif ins[0] == "un":
                    h.append(nbg.nbg_apply(c, nbg.FP64, ins[1], h[ins[2]], ins[3], ins[4]))
                elif ins[0] == "bin":
                    f = nbg.nbg_ewise_add if ins[1] == "add" else nbg.nbg_ewise_mult
                    h.append(f(c, nbg.FP64, ins[2], h[ins[3]], h[ins[4]]))
                else:
                    s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", h[ins[3]])
                    h.append(nbg.nbg_apply_bind2nd(c, nbg.FP64, ins[1], h[ins[2]], s))
            # drop some handles (elided intermediates), then read the wanted ones in shuffled order
            for k in range(3, len(prog)):
                if k not in want and rng.random() < 0.5:
                    nbg.nbg_vector_free(c, h[k])
                    h[k] = None
            for k in rng.permutation(want):
                i, x = nbg.nbg_vector_export_sparse(c, h[k])
                e = exp[k]
                assert np.array_equal(i, e.idx), (seed, mode, k, prog[k])
                scale = np.maximum(np.abs(e.vals), 1.0)
                # values: bit-exact except where a reduce-derived scalar enters (fp64 partial sums)
                assert np.all(np.abs(x - e.vals) <= 1e-12 * scale), (seed, mode, k, prog[k])
        finally:
            nbg.nbg_finalize(c)


@pytest.mark.parametrize("seed", range(30))
def test_random_dags_with_mxv_and_waits(nbg, seed):
    """As above with mxv nodes (a fixed random matrix: the fused SpMV epilogue), waits at random
    points in the recording (partially materialised DAGs), fp32 or fp64."""
    rng = np.random.default_rng(5000 + seed)
    T = np.float64 if seed % 3 else np.float32
    t = nbg.FP64 if T is np.float64 else nbg.FP32
    n = 2049
    lens = rng.integers(0, 12, n)
    lens[7] = 700
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, int(l), replace=False)) for l in lens]).astype(np.int32)
    leaves = [S.full((rng.integers(-8, 9, n) / 4.0).astype(T)) for _ in range(3)]
    prog = [("leaf", 0), ("leaf", 1), ("leaf", 2)]
    for _ in range(12):
        r = rng.random()
        a = int(rng.integers(0, len(prog)))
        if r < 0.15:
            prog.append(("mxv", "SECOND" if rng.random() < 0.5 else "TIMES", a))
        elif r < 0.4:
            prog.append(("un", UN[rng.integers(0, len(UN))], a, float(rng.integers(-3, 4)) / 2, float(rng.integers(-3, 4)) / 4))
        elif r < 0.85:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bin", "add" if rng.random() < 0.5 else "mult", BIN[rng.integers(0, len(BIN))], a, b))
        else:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bind", BIN[rng.integers(0, 5)], a, b))
    # oracle, one instruction at a time
    exp = []
    for ins in prog:
        if ins[0] == "leaf":
            exp.append(leaves[ins[1]])
        elif ins[0] == "mxv":
            exp.append(S.full(S.mxv("PLUS", ins[1], rp, ci, None, exp[ins[2]], T)))
        elif ins[0] == "un":
            exp.append(S.apply(ins[1], exp[ins[2]], T, ins[3], ins[4]))
        elif ins[0] == "bin":
            f = S.ewise_add if ins[1] == "add" else S.ewise_mult
            exp.append(f(ins[2], exp[ins[3]], exp[ins[4]], T))
        else:
            s = S.reduce("PLUS", exp[ins[3]], np.float64)
            exp.append(S.bind2nd(ins[1], exp[ins[2]], np.dtype(T).type(s), T))
    want = sorted(set(int(k) for k in rng.integers(3, len(prog), 4)))
    waits = set(int(k) for k in np.nonzero(rng.random(len(prog)) < 0.15)[0] if k >= 3)
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            A = nbg.nbg_matrix_from_csr(c, n, n, rp, ci, type=t, iso=1.0)
            h = []
            for k, ins in enumerate(prog):
                if ins[0] == "leaf":
                    h.append(nbg.nbg_vector_from_dense(c, t, leaves[ins[1]].vals))
                elif ins[0] == "mxv":
                    h.append(nbg.nbg_mxv(c, t, "PLUS", ins[1], A, h[ins[2]]))
                elif ins[0] == "un":
                    h.append(nbg.nbg_apply(c, t, ins[1], h[ins[2]], ins[3], ins[4]))
                elif ins[0] == "bin":
                    f = nbg.nbg_ewise_add if ins[1] == "add" else nbg.nbg_ewise_mult
                    h.append(f(c, t, ins[2], h[ins[3]], h[ins[4]]))
                else:
                    s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", h[ins[3]])
                    h.append(nbg.nbg_apply_bind2nd(c, t, ins[1], h[ins[2]], s))
                if k in waits:
                    nbg.nbg_vector_wait(c, h[k])
            for k in range(3, len(prog)):
                if k not in want and rng.random() < 0.5:
                    nbg.nbg_vector_free(c, h[k])
                    h[k] = None
            for k in rng.permutation(want):
                x = nbg.nbg_vector_export_dense(c, h[k])
                e = exp[k].vals
                # mxv row sums and reduce-derived scalars round in fp64 partial order: relative bound
                tol = (1e-5 if T is np.float32 else 1e-12) * np.maximum(np.abs(e), 1.0) * 64
                assert np.all(np.abs(x.astype(np.float64) - e.astype(np.float64)) <= tol), (seed, mode, k, prog[k])
        finally:
            nbg.nbg_finalize(c)


@pytest.mark.parametrize("seed", range(24))
def test_random_structured_dags(nbg, seed):
    """Random DAGs over two sparse leaves (fills 1-30 %) and one full leaf: structured regions,
    structured mxv, reductions read in the middle of the recording, partial waits."""
    rng = np.random.default_rng(9000 + seed)
    T = np.float64
    n = 2500
    lens = rng.integers(0, 10, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, int(l), replace=False)) for l in lens]).astype(np.int32)
    leaves = []
    for fill in (rng.choice([0.01, 0.05, 0.3]), rng.choice([0.01, 0.05, 0.3])):
        idx = np.nonzero(rng.random(n) < fill)[0]
        leaves.append(S.sparse(n, idx, (rng.integers(-8, 9, idx.shape[0]) / 4.0).astype(T)))
    leaves.append(S.full((rng.integers(-8, 9, n) / 4.0).astype(T)))
    prog = [("leaf", 0), ("leaf", 1), ("leaf", 2)]
    for _ in range(12):
        r = rng.random()
        a = int(rng.integers(0, len(prog)))
        if r < 0.1:
            prog.append(("mxv", "TIMES", a))
        elif r < 0.35:
            prog.append(("un", UN[rng.integers(0, len(UN))], a, float(rng.integers(-3, 4)) / 2, float(rng.integers(-3, 4)) / 4))
        elif r < 0.85:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bin", "add" if rng.random() < 0.5 else "mult", BIN[rng.integers(0, len(BIN))], a, b))
        else:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bind", BIN[rng.integers(0, 5)], a, b))
    exp = []
    for ins in prog:
        if ins[0] == "leaf":
            exp.append(leaves[ins[1]])
        elif ins[0] == "mxv":
            exp.append(S.full(S.mxv("PLUS", ins[1], rp, ci, None, exp[ins[2]], T)))
        elif ins[0] == "un":
            exp.append(S.apply(ins[1], exp[ins[2]], T, ins[3], ins[4]))
        elif ins[0] == "bin":
            f = S.ewise_add if ins[1] == "add" else S.ewise_mult
            exp.append(f(ins[2], exp[ins[3]], exp[ins[4]], T))
        else:
            s = S.reduce("PLUS", exp[ins[3]], np.float64)
            exp.append(S.bind2nd(ins[1], exp[ins[2]], np.dtype(T).type(s), T))
    want = sorted(set(int(k) for k in rng.integers(3, len(prog), 4)))
    waits = set(int(k) for k in np.nonzero(rng.random(len(prog)) < 0.15)[0] if k >= 3)
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            A = nbg.nbg_matrix_from_csr(c, n, n, rp, ci, type=nbg.FP64, iso=1.0)
            h, sc = [], {}
            for k, ins in enumerate(prog):
                if ins[0] == "leaf":
                    L = leaves[ins[1]]
                    if L.idx.shape[0] == n:
                        h.append(nbg.nbg_vector_from_dense(c, nbg.FP64, L.vals))
                    else:
                        h.append(nbg.nbg_vector_from_sparse(c, nbg.FP64, n, L.idx.astype(np.int32), L.vals))
                elif ins[0] == "mxv":
                    h.append(nbg.nbg_mxv(c, nbg.FP64, "PLUS", ins[1], A, h[ins[2]]))
                elif ins[0] == "un":
                    h.append(nbg.nbg_apply(c, nbg.FP64, ins[1], h[ins[2]], ins[3], ins[4]))
                elif ins[0] == "bin":
                    f = nbg.nbg_ewise_add if ins[1] == "add" else nbg.nbg_ewise_mult
                    h.append(f(c, nbg.FP64, ins[2], h[ins[3]], h[ins[4]]))
                else:
                    s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", h[ins[3]])
                    sc[k] = (s, ins[3])
                    h.append(nbg.nbg_apply_bind2nd(c, nbg.FP64, ins[1], h[ins[2]], s))
                    if rng.random() < 0.3:         # read the scalar now (materialises its region)
                        v = nbg.nbg_scalar_get(c, s)
                        ref = float(S.reduce("PLUS", exp[ins[3]], np.float64))
                        assert abs(v - ref) <= 1e-12 * max(1.0, float(np.abs(exp[ins[3]].vals).sum())), (seed, mode, k)
                if k in waits:
                    nbg.nbg_vector_wait(c, h[k])
            for k in rng.permutation(want):
                i, x = nbg.nbg_vector_export_sparse(c, h[k])
                e = exp[k]
                assert np.array_equal(i, e.idx), (seed, mode, k, prog[k])
                assert np.all(np.abs(x - e.vals) <= 64e-12 * np.maximum(np.abs(e.vals), 1.0)), (seed, mode, k, prog[k])
        finally:
            nbg.nbg_finalize(c)


@pytest.mark.parametrize("seed", range(12))
def test_random_loops_speculation(nbg, seed):
    """Loops of a random sweep body t <- f(t) (mxv of a scaled t, random elementwise epilogue,
    a reduce-derived constant, a delta reduction read each iteration): after the first iterations
    the planner learns loop-carried side outputs (speculation hints) and memoised invariants; every
    iterate and every delta must still match the oracle, in both modes."""
    rng = np.random.default_rng(7000 + seed)
    T = np.float64
    n = 1500
    lens = rng.integers(0, 9, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, int(l), replace=False)) for l in lens]).astype(np.int32)
    d = (rng.integers(0, 5, n) / 8.0).astype(T)            # zeros act as a "dangling" mask
    t0 = (rng.integers(1, 9, n) / 64.0).astype(T)
    u1 = UN[rng.integers(0, len(UN))]
    b1 = BIN[rng.integers(0, 5)]
    k0, k1 = float(rng.integers(-3, 4)) / 4, float(rng.integers(-3, 4)) / 8
    iters = 8

    def body_oracle(t):
        y = S.ewise_mult("TIMES", S.full(t), S.full(d), T)
        m = S.full(S.mxv("PLUS", "SECOND", rp, ci, None, y, T))
        z = S.ewise_mult("TIMES", S.full(t), S.apply("ISZERO", S.full(d), T), T)
        s = S.reduce("PLUS", z, np.float64)
        r = S.bind2nd(b1, S.apply(u1, m, T, k0, k1), np.dtype(T).type(s * 0.5), T)
        delta = S.reduce("PLUS", S.ewise_add("ABSDIFF", S.full(t), r, T), np.float64)
        return r.vals, float(delta)

    ts, ds = [t0], []
    for _ in range(iters):
        nt, dl = body_oracle(ts[-1])
        ts.append(nt)
        ds.append(dl)
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            A = nbg.nbg_matrix_from_csr(c, n, n, rp, ci, type=nbg.FP64, iso=1.0)
            dv = nbg.nbg_vector_from_dense(c, nbg.FP64, d)
            t = nbg.nbg_vector_from_dense(c, nbg.FP64, t0)
            for it in range(iters):
                y = nbg.nbg_ewise_mult(c, nbg.FP64, "TIMES", t, dv)
                m = nbg.nbg_mxv(c, nbg.FP64, "PLUS", "SECOND", A, y)
                nbg.nbg_vector_free(c, y)
                mask = nbg.nbg_apply(c, nbg.FP64, "ISZERO", dv)
                z = nbg.nbg_ewise_mult(c, nbg.FP64, "TIMES", t, mask)
                nbg.nbg_vector_free(c, mask)
                s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", z)
                nbg.nbg_vector_free(c, z)
                sh = nbg.nbg_scalar_apply(c, nbg.FP64, "MUL_C", s, 0.5)
                um = nbg.nbg_apply(c, nbg.FP64, u1, m, k0, k1)
                nbg.nbg_vector_free(c, m)
                r = nbg.nbg_apply_bind2nd(c, nbg.FP64, b1, um, sh)
                nbg.nbg_vector_free(c, um)
                e = nbg.nbg_ewise_add(c, nbg.FP64, "ABSDIFF", t, r)
                dl = nbg.nbg_reduce(c, nbg.FP64, "PLUS", e)
                nbg.nbg_vector_free(c, e)
                got_d = nbg.nbg_scalar_get(c, dl)
                assert got_d == ds[it] or abs(got_d - ds[it]) <= 1e-10 * max(1.0, abs(ds[it])), (seed, mode, it)
                nbg.nbg_vector_free(c, t)
                t = r
                got = nbg.nbg_vector_export_dense(c, t)
                ex = ts[it + 1]
                with np.errstate(invalid="ignore"):
                    ok = (got == ex) | (np.abs(got - ex) <= 1e-10 * np.maximum(1.0, np.abs(ex))) | (np.isnan(got) & np.isnan(ex))
                assert np.all(ok), (seed, mode, it)
        finally:
            nbg.nbg_finalize(c)


@pytest.mark.parametrize("seed", range(12))
def test_random_dags_integer(nbg, seed):
    """Random DAGs in int32 / int64 (wrapping arithmetic, integer division excluded by the op
    list): every element exact, reductions (int64 PLUS) exact; sparse leaves on odd seeds."""
    rng = np.random.default_rng(3000 + seed)
    T = np.int32 if seed % 2 == 0 else np.int64
    t = nbg.INT32 if T is np.int32 else nbg.INT64
    n = 1777
    leaves = [S.full(rng.integers(-50, 51, n).astype(T)), S.full(rng.integers(-50, 51, n).astype(T))]
    idx = np.nonzero(rng.random(n) < (0.08 if seed % 4 == 1 else 1.0))[0]
    leaves.append(S.sparse(n, idx, rng.integers(-50, 51, idx.shape[0]).astype(T)))
    prog = [("leaf", 0), ("leaf", 1), ("leaf", 2)]
    for _ in range(14):
        r = rng.random()
        a = int(rng.integers(0, len(prog)))
        if r < 0.35:
            prog.append(("un", UN[rng.integers(0, len(UN))], a, float(rng.integers(-3, 4)), float(rng.integers(-3, 4))))
        elif r < 0.85:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bin", "add" if rng.random() < 0.5 else "mult", BIN[rng.integers(0, len(BIN))], a, b))
        else:
            b = int(rng.integers(0, len(prog)))
            prog.append(("bind", BIN[rng.integers(0, 5)], a, b))
    exp = []
    for ins in prog:
        if ins[0] == "leaf":
            exp.append(leaves[ins[1]])
        elif ins[0] == "un":
            exp.append(S.apply(ins[1], exp[ins[2]], T, ins[3], ins[4]))
        elif ins[0] == "bin":
            f = S.ewise_add if ins[1] == "add" else S.ewise_mult
            exp.append(f(ins[2], exp[ins[3]], exp[ins[4]], T))
        else:
            s = S.reduce("PLUS", exp[ins[3]], np.int64)
            exp.append(S.bind2nd(ins[1], exp[ins[2]], int(s), T))
    want = sorted(set(int(k) for k in rng.integers(3, len(prog), 4)))
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            h = []
            for ins in prog:
                if ins[0] == "leaf":
                    L = leaves[ins[1]]
                    if L.idx.shape[0] == n:
                        h.append(nbg.nbg_vector_from_dense(c, t, L.vals))
                    else:
                        h.append(nbg.nbg_vector_from_sparse(c, t, n, L.idx.astype(np.int32), L.vals))
                elif ins[0] == "un":
                    h.append(nbg.nbg_apply(c, t, ins[1], h[ins[2]], ins[3], ins[4]))
                elif ins[0] == "bin":
                    f = nbg.nbg_ewise_add if ins[1] == "add" else nbg.nbg_ewise_mult
                    h.append(f(c, t, ins[2], h[ins[3]], h[ins[4]]))
                else:
                    s = nbg.nbg_reduce(c, nbg.INT64, "PLUS", h[ins[3]])
                    h.append(nbg.nbg_apply_bind2nd(c, t, ins[1], h[ins[2]], s))
            for k in rng.permutation(want):
                i, x = nbg.nbg_vector_export_sparse(c, h[k])
                assert np.array_equal(i, exp[k].idx) and np.array_equal(x, exp[k].vals), (seed, mode, k, prog[k])
        finally:
            nbg.nbg_finalize(c)


@pytest.mark.parametrize("seed", range(16))
def test_random_pagerank(nbg, seed):
    """nbg_pagerank on random small graphs (random sizes, duplicate edges, self-loops, isolated
    and dangling vertices, hubs), both dangling variants, fp32 / fp64, fixed-count and converged:
    sweep counts exact, ranks within 1e-5 / 1e-10, delta history within the derived bound."""
    import oracle
    rng = np.random.default_rng(1100 + seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 8 * n + 1))
    src = rng.integers(0, n, m).astype(np.int32)
    dst = (rng.integers(0, max(1, n // 50), m) if seed % 3 == 0 else rng.integers(0, n, m)).astype(np.int32)   # hubs
    T = np.float32 if seed % 2 else np.float64
    t = nbg.FP32 if T is np.float32 else nbg.FP64
    tol = -1.0 if seed % 4 < 2 else (1e-6 if T is np.float32 else 1e-12)
    uniform = seed % 5 != 0
    c = nbg.nbg_init(nbg.NONBLOCKING if seed % 7 else nbg.BLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_edges(c, n, src, dst)
        orp, oci, odeg = oracle.build_csr(n, src, dst)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
        r, sw, hist = nbg.nbg_pagerank(c, A, deg, tol=tol, itermax=60, type=t,
                                       dangling=nbg.PR_UNIFORM if uniform else nbg.PR_DROP)
        ro, so, dho, _ = oracle.pagerank(orp, oci, odeg, dtype=T, itermax=60, tol=tol, uniform=uniform)
        assert sw == so, (seed, sw, so)
        got = nbg.nbg_vector_export_dense(c, r)
        assert np.max(np.abs(got - ro) / np.abs(ro)) <= (1e-5 if T is np.float32 else 1e-10), seed
        # A priori bound (DESIGN.md §4 "tolerances"): Delta_k moves by at most ||e_k||_1 + ||e_k-1||_1
        # (triangle inequality, e = rank error vector).  Per sweep each rank picks up at most one
        # ulp_T (m_i + c rounded to T) plus the error of c = alpha ds / n + (1 - alpha) / n, which
        # enters EVERY rank with the same sign: ds (<= 1) is the exactly rounded sum on the GPU and a
        # sequential fp64 sum in the oracle, |d ds| <= n eps64, so |d c| <= alpha eps64 and the sweep
        # adds at most sum_i ulp_T(r_i) + alpha n eps64 in L1.  A sweep maps errors through alpha x
        # (a column-stochastic matrix), L1 norm alpha, so ||e_k||_1 <= that / (1 - alpha) and
        # |Delta_gpu - Delta_oracle| <= 2 / (1 - alpha) (sum_i ulp_T(r_i) + alpha n eps64)
        # = 13.3 (...) at alpha = 0.85 (16 used; Delta's own fp64 sums add far less).
        eps64 = float(np.finfo(np.float64).eps)
        atol = 16.0 * (float(np.spacing(np.abs(np.asarray(ro, T))).astype(np.float64).sum()) + 0.85 * n * eps64)
        assert np.all(np.abs(np.asarray(hist) - np.asarray(dho)) <= np.maximum(1e-9 * np.abs(dho), atol)), seed
    finally:
        nbg.nbg_finalize(c)
