"""Matrix Market ingestion (PAPER.md:324 reads GAP-web.mtx).

CPU: the oracle's reader against hand-derived edge lists / CSR (the format's definition).
GPU: nbg_matrix_from_mtx gives the oracle's CSR and out-degree bit for bit on generated files
(general real with duplicates and self-loops, symmetric pattern, comment lines), errors map to
the documented statuses, and PageRank on a loaded graph matches the oracle.
"""
import os

import numpy as np
import pytest

import oracle


def _write(path, text):
    with open(path, "w") as f:
        f.write(text)
    return path


def test_oracle_read_mtx_symmetric_pattern(tmp_path):
    p = _write(tmp_path / "a.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n% comment\n4 4 3\n2 1\n3 2\n4 4\n")
    n, s, d = oracle.read_mtx(p)
    assert n == 4
    # (2,1) -> edges 1->0 and 0->1; (3,2) -> 2->1 and 1->2; (4,4) -> 3->3 (one self-loop)
    assert sorted(zip(s.tolist(), d.tolist())) == sorted([(1, 0), (0, 1), (2, 1), (1, 2), (3, 3)])
    rp, ci, deg = oracle.build_csr(n, s, d)
    assert rp.tolist() == [0, 1, 3, 4, 4]         # AT rows = destinations; the self-loop is dropped
    assert ci.tolist() == [1, 0, 2, 1]
    assert deg.tolist() == [1, 2, 1, 0]


def test_oracle_read_mtx_general_real(tmp_path):
    p = _write(tmp_path / "b.mtx", "%%MatrixMarket matrix coordinate real general\n3 5 4\n1 2 0.5\n1 2 7\n3 5 -1e3\n2 1 2\n")
    n, s, d = oracle.read_mtx(p)
    assert n == 5 and s.tolist() == [0, 0, 2, 1] and d.tolist() == [1, 1, 4, 0]
    rp, ci, deg = oracle.build_csr(n, s, d)
    assert rp.tolist() == [0, 1, 2, 2, 2, 3] and ci.tolist() == [1, 0, 2]   # duplicate (1,2) kept once
    assert deg.tolist() == [1, 1, 1, 0, 0]


def test_oracle_read_mtx_errors(tmp_path):
    with pytest.raises(ValueError):
        oracle.read_mtx(_write(tmp_path / "c.mtx", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"))
    with pytest.raises(IndexError):
        oracle.read_mtx(_write(tmp_path / "d.mtx", "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n"))


def _random_mtx(path, n, m, seed, symmetric=False, field="real"):
    rng = np.random.default_rng(seed)
    i = rng.integers(1, n + 1, m)
    j = rng.integers(1, n + 1, m)
    if symmetric:
        i, j = np.maximum(i, j), np.minimum(i, j)
    lines = [f"%%MatrixMarket matrix coordinate {field} {'symmetric' if symmetric else 'general'}", "% generated", f"{n} {n} {m}"]
    for a, b in zip(i, j):
        lines.append(f"{a} {b}" if field == "pattern" else f"{a} {b} {rng.random():.6f}")
        if rng.random() < 0.01:
            lines.append("% interleaved comment")
    _write(path, "\n".join(lines) + "\n")


@pytest.mark.gpu
@pytest.mark.parametrize("symmetric,field", [(False, "real"), (True, "pattern"), (False, "integer")])
def test_mtx_csr_bit_exact(tmp_path, symmetric, field):
    from paper_2509_14211_b200 import nbg
    p = tmp_path / "g.mtx"
    _random_mtx(p, 3000, 40000, 3, symmetric, field)
    n, s, d = oracle.read_mtx(p)
    orp, oci, odeg = oracle.build_csr(n, s, d)
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_mtx(c, p)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
        assert np.array_equal(nbg.nbg_vector_export_dense(c, deg), odeg)
        r, sweeps, _ = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=10, type=nbg.FP64)
        ro, so, _, _ = oracle.pagerank(orp, oci, odeg, dtype=np.float64, itermax=10)
        rv = nbg.nbg_vector_export_dense(c, r)
        assert sweeps == so and float(np.max(np.abs(rv - ro) / ro)) <= 1e-10
    finally:
        nbg.nbg_finalize(c)


@pytest.mark.gpu
def test_mtx_errors(tmp_path):
    from paper_2509_14211_b200 import nbg
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        cases = [("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", nbg.INVALID_VALUE),
                 ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 1\n", nbg.INVALID_VALUE),
                 ("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n", nbg.INVALID_VALUE),
                 ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n", nbg.INDEX_OUT_OF_BOUNDS),
                 ("not a matrix market file\n", nbg.INVALID_VALUE)]
        for k, (text, st) in enumerate(cases):
            p = _write(tmp_path / f"e{k}.mtx", text)
            with pytest.raises(nbg.NbgError) as ex:
                nbg.nbg_matrix_from_mtx(c, p)
            assert ex.value.status == st, (k, ex.value)
        with pytest.raises(nbg.NbgError) as ex:
            nbg.nbg_matrix_from_mtx(c, tmp_path / "missing.mtx")
        assert ex.value.status == nbg.INVALID_VALUE
    finally:
        nbg.nbg_finalize(c)
