# v6 SpMV time split: same row structure, (a) real columns, (b) all columns hot (colidx % 32768,
# duplicates kept as separate entries), (c) real columns with the hot cache disabled
import sys, os; sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
def run(label, rp, ci, n, env=None):
    if env:
        for k, v in env.items(): os.environ[k] = v
    c = nbg.nbg_init(nbg.NONBLOCKING, 0)
    A = nbg.nbg_matrix_from_csr(c, n, n, rp, ci, type=nbg.FP32)
    x = nbg.nbg_vector_from_dense(c, nbg.FP32, np.random.rand(n).astype(np.float32))
    nbg.nbg_set_timing(c, 1)
    for _ in range(10):
        m = nbg.nbg_mxv(c, nbg.FP32, "PLUS", "SECOND", A, x)
        nbg.nbg_vector_wait(c, m)
        nbg.nbg_vector_free(c, m)
    nbg.nbg_sync(c)
    ms, cnt = nbg.nbg_get_timing(c, "spmv")
    print(f"{label}: {ms / cnt * 1e3:.1f} us per mxv ({cnt} launches)", flush=True)
    nbg.nbg_finalize(c)
    if env:
        for k in env: del os.environ[k]
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
nbg.nbg_finalize(c)
n = rp.shape[0] - 1
run("real", rp, ci, n)
ci2 = (ci % 32768).astype(np.int32)
run("all hot (col % 32768)", rp, ci2, n)
run("real, hot cache 0 KB", rp, ci, n, {"NBG_SPMV_HOT_KB": "0"})
