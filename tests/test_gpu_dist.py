"""The row-partitioned (multi-GPU) path on one GPU: a one-rank NCCL communicator (one GPU per
gpurun call; the N > 1 exchange logic is covered by tests/test_dist_gloo.py on the CPU).

* nbg_pagerank_dist over the whole matrix as the rank's block equals nbg_pagerank.
* row blocks (nbg_matrix_row_block) are the CSR row slices, bit for bit.
* the byte-balanced partition covers all rows with monotone cuts.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.mark.parametrize("T", ["fp32", "fp64"])
def test_dist_one_rank_equals_single(nbg, T):
    t = nbg.TYPE_OF[T]
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        nbg.nbg_dist_init(c, 0, 1, nbg.nbg_dist_unique_id())
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 14, 16, 7)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        n = rp.shape[0] - 1
        cuts = nbg.nbg_partition_rows(rp, 1, 20)
        assert cuts[0] == 0 and cuts[-1] == n
        B = nbg.nbg_matrix_row_block(c, A, int(cuts[0]), int(cuts[1]))
        r1, s1, h1 = nbg.nbg_pagerank(c, A, deg, tol=-1.0, itermax=15, type=t)
        r2, s2, h2 = nbg.nbg_pagerank_dist(c, B, deg, cuts, tol=-1.0, itermax=15, type=t)
        v1 = nbg.nbg_vector_export_dense(c, r1)
        v2 = nbg.nbg_vector_export_dense(c, r2)
        assert s1 == s2 == 15
        assert rel(v2, v1) <= (1e-6 if T == "fp32" else 1e-13)
        ro, so, dho, _ = oracle.pagerank(rp, ci, nbg.nbg_vector_export_dense(c, deg), dtype=nbg.NP_OF[t], itermax=15)
        assert rel(v2, ro) <= (1e-5 if T == "fp32" else 1e-10)
    finally:
        nbg.nbg_finalize(c)


def test_row_blocks_are_csr_slices(nbg):
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    try:
        A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 12, 8, 3)
        rp, ci = nbg.nbg_matrix_export_csr(c, A)
        n = rp.shape[0] - 1
        cuts = nbg.nbg_partition_rows(rp, 4, 20)
        assert np.all(np.diff(cuts) >= 0) and cuts[0] == 0 and cuts[-1] == n
        for k in range(4):
            B = nbg.nbg_matrix_row_block(c, A, int(cuts[k]), int(cuts[k + 1]))
            brp, bci = nbg.nbg_matrix_export_csr(c, B)
            assert np.array_equal(brp, rp[cuts[k]:cuts[k + 1] + 1] - rp[cuts[k]])
            assert np.array_equal(bci, ci[rp[cuts[k]]:rp[cuts[k + 1]]])
            nbg.nbg_matrix_free(c, B)
    finally:
        nbg.nbg_finalize(c)
