"""GPU parity of the row-binned SpMV skeleton (DESIGN.md §7 "row-binned SpMV"; plan RbPlan, kernel
gen_spmv_rb): short rows lane-per-row from length-sorted 32-row slices, long rows one warp each,
hub rows (> 2048 entries) in 512-group chunks combined in order, then the fused epilogue after a
grid barrier.

* Short rows are summed sequentially in fp64 in ascending stored order -- the oracle's own order
  (oracle/ops.py mxv, reading Q4) -- so with every non-hub row short (NBG_RB_T=512) the PLUS mxv
  equals the oracle bit for bit.
* Long rows and hub chunks use a fixed lane-strided order + shuffle tree; ``_warp_row_sum`` below
  restates that order in numpy and the kernel must match it bit for bit.
* A row's sum depends on its length only: permuting the rows of a matrix permutes the result.
* PageRank through the skeleton against the oracle (tolerances of the north star), fused ==
  blocking bit for bit, for several short-row bounds T and task budgets.
"""
import numpy as np
import pytest

import oracle
from oracle import ops

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["b", "p", "i"])
def rb_mode(request, monkeypatch):
    """Every epilogue mode: b = row totals + grid barrier + epilogue pass (default), p = epilogue
    chunks of a row group taken once its totals are complete, i = the epilogue where each row's
    total completes."""
    monkeypatch.setenv("NBG_RB_MODE", request.param)
    return request.param


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.abs(b))) if a.size else 0.0


def _warp_row_sum(terms):
    """The order of a warp-processed row: the row padded to 4-entry groups, lane l
    sums groups l, l + 32, l + 64, ... (each group's 4 entries in order) into an fp64 partial, then
    lane 0 takes the shuffle-down tree v[l] += v[l + d], d = 16, 8, 4, 2, 1."""
    t = np.asarray(terms, np.float64)
    g = (t.shape[0] + 3) // 4
    pad = np.zeros(4 * g)
    pad[:t.shape[0]] = t
    grp = pad.reshape(g, 4)
    v = np.zeros(32)
    for lane in range(32):
        acc = 0.0
        for k in range(lane, g, 32):
            for e in range(4):
                acc += grp[k, e]
        v[lane] = acc
    d = 16
    while d > 0:
        v = np.concatenate([v[:32 - d] + v[d:], v[32 - d:]])
        d >>= 1
    return v[0]


def _rb_row_sum(terms, T):
    g = (len(terms) + 3) // 4
    if g <= T:                                     # lane-per-row: sequential fp64
        acc = 0.0
        for z in terms:
            acc += float(z)
        return acc
    if g <= 512:
        return _warp_row_sum(terms)
    acc = 0.0                                      # hub: chunks of 512 groups, combined in order
    for c0 in range(0, len(terms), 2048):
        acc += _warp_row_sum(terms[c0:c0 + 2048])
    return acc


def _matrix(rng, n, m, lens):
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(m, int(l), replace=False)) for l in lens]).astype(np.int32)
    return rp, ci


def _lens(rng, n):
    # power-law-ish: most rows short, some long (warp path), two hubs (chunked), empty rows
    lens = np.minimum(rng.zipf(1.6, n), 1500).astype(np.int64)
    lens[rng.random(n) < 0.3] = 0
    lens[3] = 5000
    lens[n // 2] = 2049
    lens[n - 1] = 600
    return lens


@pytest.mark.parametrize("T", ["fp32", "fp64"])
@pytest.mark.parametrize("rbT", [1, 16, 64, 512])
def test_rb_mxv_bits(nbg, monkeypatch, T, rbT):
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    monkeypatch.setenv("NBG_RB_T", str(rbT))
    rng = np.random.default_rng(rbT)
    n, m = 3000, 6000
    lens = _lens(rng, n)
    rp, ci = _matrix(rng, n, m, lens)
    t = nbg.TYPE_OF[T]
    npT = nbg.NP_OF[t]
    x = rng.random(m).astype(npT)
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A = nbg.nbg_matrix_from_csr(c, n, m, rp, ci, type=t)
        got = nbg.nbg_vector_export_dense(c, nbg.nbg_mxv(c, t, "PLUS", "SECOND", A, nbg.nbg_vector_from_dense(c, t, x)))
    finally:
        nbg.nbg_finalize(c)
    exp = ops.mxv("PLUS", "SECOND", rp, ci, None, x, npT)
    assert rel(got[lens > 0], exp[lens > 0]) <= (2e-7 if T == "fp32" else 1e-14)
    assert np.all(got[lens == 0] == 0)
    model = np.array([_rb_row_sum(x[ci[rp[i]:rp[i + 1]]].astype(np.float64), rbT) for i in range(n)]).astype(npT)
    assert np.array_equal(got, model)
    if rbT == 512:                                  # every non-hub row sequential: the oracle's bits
        short = (lens + 3) // 4 <= 512
        assert np.array_equal(got[short], exp[short])


@pytest.mark.parametrize("add", ["MIN", "MAX", "PLUS"])
@pytest.mark.parametrize("T", ["int32", "int64", "fp32"])
def test_rb_mxv_semirings(nbg, monkeypatch, add, T):
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    rng = np.random.default_rng(7)
    n, m = 2500, 5000
    lens = _lens(rng, n)
    rp, ci = _matrix(rng, n, m, lens)
    t = nbg.TYPE_OF[T]
    npT = nbg.NP_OF[t]
    x = (rng.integers(-1000, 1000, m) if T.startswith("int") else rng.random(m) - 0.5).astype(npT)
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A = nbg.nbg_matrix_from_csr(c, n, m, rp, ci, type=t, iso=3.0)
        got = nbg.nbg_vector_export_dense(c, nbg.nbg_mxv(c, t, add, "TIMES", A, nbg.nbg_vector_from_dense(c, t, x)))
    finally:
        nbg.nbg_finalize(c)
    exp = ops.mxv(add, "TIMES", rp, ci, None, x, npT, iso=3.0)
    if add == "PLUS" and T == "fp32":
        assert rel(got[lens > 0], exp[lens > 0]) <= 2e-7
    else:
        assert np.array_equal(got, exp)


def test_rb_row_sums_depend_on_length_only(nbg, monkeypatch):
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    rng = np.random.default_rng(11)
    n, m = 4000, 6000
    lens = _lens(rng, n)
    rp, ci = _matrix(rng, n, m, lens)
    perm = rng.permutation(n)
    lp = lens[perm]
    rp2 = np.concatenate([[0], np.cumsum(lp)]).astype(np.int64)
    ci2 = np.concatenate([ci[rp[i]:rp[i + 1]] for i in perm]).astype(np.int32)
    x = rng.random(m).astype(np.float32)
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        out = []
        for r_, c_ in ((rp, ci), (rp2, ci2)):
            A = nbg.nbg_matrix_from_csr(c, n, m, r_, c_, type=nbg.FP32)
            out.append(nbg.nbg_vector_export_dense(c, nbg.nbg_mxv(c, nbg.FP32, "PLUS", "SECOND", A,
                                                                  nbg.nbg_vector_from_dense(c, nbg.FP32, x))))
    finally:
        nbg.nbg_finalize(c)
    assert np.array_equal(out[0][perm], out[1])


@pytest.mark.parametrize("rbT,tg", [(16, 512), (1, 32), (64, 4096)])
@pytest.mark.parametrize("kind,scale,ef", [("rmat", 14, 16), ("rmat", 10, 8), ("er", 12, 16)])
def test_rb_pagerank(nbg, monkeypatch, rbT, tg, kind, scale, ef):
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    monkeypatch.setenv("NBG_RB_T", str(rbT))
    monkeypatch.setenv("NBG_RB_TG", str(tg))
    g = nbg.GRAPH_RMAT if kind == "rmat" else nbg.GRAPH_ER
    res = {}
    for mode in (nbg.NONBLOCKING, nbg.BLOCKING):
        c = nbg.nbg_init(mode, 0)
        try:
            A, deg = nbg.nbg_matrix_from_generator(c, g, scale, ef, 3)
            rp, ci = nbg.nbg_matrix_export_csr(c, A)
            d = nbg.nbg_vector_export_dense(c, deg)
            for T, tol in (("fp32", 1e-5), ("fp64", 1e-10)):
                for dang in (nbg.PR_UNIFORM, nbg.PR_DROP):
                    t = nbg.TYPE_OF[T]
                    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=12, dangling=dang, type=t)
                    v = nbg.nbg_vector_export_dense(c, r)
                    ro, so, dho, _ = oracle.pagerank(rp, ci, d, dtype=nbg.NP_OF[t], itermax=12, uniform=dang == nbg.PR_UNIFORM)
                    assert s == so == 12
                    assert rel(v, ro) <= tol
                    res[(mode, T, dang)] = (v, h)
        finally:
            nbg.nbg_finalize(c)
    for T in ("fp32", "fp64"):
        for dang in (nbg.PR_UNIFORM, nbg.PR_DROP):
            a, b = res[(nbg.NONBLOCKING, T, dang)], res[(nbg.BLOCKING, T, dang)]
            assert np.array_equal(a[0], b[0])


def test_rb_convergence_and_determinism(nbg, monkeypatch):
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 16, 16, 1)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        d = nbg.nbg_vector_export_dense(c, deg)
        runs = []
        for _ in range(3):
            r, s, h = nbg.nbg_pagerank(c, A, deg, tol=1e-6, itermax=100, type=nbg.FP32)
            runs.append((nbg.nbg_vector_export_dense(c, r), s, h))
        ro, so, dho, _ = oracle.pagerank(rp, ci, d, dtype=np.float32, itermax=100, tol=1e-6)
        assert runs[0][1] == so
        assert rel(runs[0][0], ro) <= 1e-5
        for v, s, h in runs[1:]:
            assert s == runs[0][1] and np.array_equal(v, runs[0][0]) and np.array_equal(h, runs[0][2])
        st = nbg.nbg_get_stats(c)
        assert st["kernels_launched"] > 0
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("n,src,dst", [(1, [], []), (3, [0], [1]), (40, list(range(1, 40)), [0] * 39),
                                       (5000, list(range(1, 5000)), [0] * 4999)])
def test_rb_degenerate(nbg, monkeypatch, n, src, dst):
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    src = np.asarray(src, np.int32)
    dst = np.asarray(dst, np.int32)
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_edges(c, n, src, dst)
        orp, oci, odeg = oracle.build_csr(n, src, dst)
        r, sw, _ = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=5, type=nbg.FP64)
        ro, so, _, _ = oracle.pagerank(orp, oci, odeg, dtype=np.float64, itermax=5)
        assert sw == so and rel(nbg.nbg_vector_export_dense(c, r), ro) <= 1e-10
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("ng", [1, 3, 64])
def test_rb_row_groups(nbg, monkeypatch, ng):
    """Row groups of the pipelined mode (NBG_RB_NG): one group, an uneven count, more groups than
    rows per group allows (clamped) -- PageRank against the oracle and repeated solves bit-identical
    (the monotonic completion counters carry over between launches)."""
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    monkeypatch.setenv("NBG_RB_NG", str(ng))
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 13, 16, 7)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        d = nbg.nbg_vector_export_dense(c, deg)
        runs = []
        for _ in range(3):
            r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=9, type=nbg.FP32)
            runs.append((nbg.nbg_vector_export_dense(c, r), h))
        ro, so, dho, _ = oracle.pagerank(rp, ci, d, dtype=np.float32, itermax=9)
        assert rel(runs[0][0], ro) <= 1e-5
        for v, h in runs[1:]:
            assert np.array_equal(v, runs[0][0]) and np.array_equal(h, runs[0][1])
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_rb_cold_gather_qualifiers_same_bits(nbg, monkeypatch, T):
    """NBG_SPMV_COLD picks the load the cold gathers use (ld.global.cg by default, the read-only path
    with L1 allocation for nc / el; DESIGN.md §7 has the measured sweep): the qualifier is a cache
    hint only, so every variant must return the same bits.  The matrix has more non-empty columns
    than the shared-memory hot cache holds (≈ 43 K fp32 / 21 K fp64 entries), so cold gathers run."""
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    rng = np.random.default_rng(11)
    n, m = 3000, 400000
    lens = _lens(rng, n)
    lens[rng.choice(n, 40, replace=False)] = 4000
    rp, ci = _matrix(rng, n, m, lens)
    assert np.unique(ci).size > 60000
    t = nbg.TYPE_OF[T]
    npT = nbg.NP_OF[t]
    x = rng.random(m).astype(npT)
    res = {}
    for q in ["cg", "nc", "el"]:
        monkeypatch.setenv("NBG_SPMV_COLD", q)
        c = nbg.nbg_init(nbg.NONBLOCKING, 0)
        try:
            A = nbg.nbg_matrix_from_csr(c, n, m, rp, ci, type=t)
            res[q] = nbg.nbg_vector_export_dense(c, nbg.nbg_mxv(c, t, "PLUS", "SECOND", A, nbg.nbg_vector_from_dense(c, t, x)))
        finally:
            nbg.nbg_finalize(c)
    exp = ops.mxv("PLUS", "SECOND", rp, ci, None, x, npT)
    assert rel(res["cg"][lens > 0], exp[lens > 0]) <= (2e-7 if T == "fp32" else 1e-14)
    assert np.array_equal(res["nc"], res["cg"])
    assert np.array_equal(res["el"], res["cg"])


def test_rb_epilogue_cache_hints_same_bits(nbg, monkeypatch, rb_mode):
    """NBG_RB_EPI_HINT puts an L2 cache policy on the epilogue pass's fp32 vector loads / stores
    (default: evict_first input loads): a hint only -- ranks and the delta history
    must equal the hint-free kernel's bit for bit, and the oracle within the north-star tolerance."""
    monkeypatch.setenv("NBG_SPMV_RB", "1")
    res = {}
    rp = ci = d = None
    for hint in ["0", "ef", "efs", "efl", "el", "els", ""]:
        if hint:
            monkeypatch.setenv("NBG_RB_EPI_HINT", hint)
        else:
            monkeypatch.delenv("NBG_RB_EPI_HINT", raising=False)     # the default choice
        c = nbg.nbg_init(nbg.NONBLOCKING, 0)
        try:
            A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 13, 16, 5)
            if rp is None:
                rp, ci = nbg.nbg_matrix_export_csr(c, A)
                d = nbg.nbg_vector_export_dense(c, deg)
            r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=10, dangling=nbg.PR_UNIFORM, type=nbg.FP32)
            res[hint] = (nbg.nbg_vector_export_dense(c, r), s, np.asarray(h))
        finally:
            nbg.nbg_finalize(c)
    ro, so, _, _ = oracle.pagerank(rp, ci, d, dtype=np.float32, itermax=10, uniform=True)
    assert res["0"][1] == so == 10 and rel(res["0"][0], ro) <= 1e-5
    for hint in ["ef", "efs", "efl", "el", "els", ""]:
        assert np.array_equal(res[hint][0], res["0"][0]) and np.array_equal(res[hint][2], res["0"][2])
