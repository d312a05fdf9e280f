import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2509_14211_b200 import nbg
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 10, 8, 1)
x = nbg.nbg_vector_new_const(c, nbg.FP64, 1024, 1.0)
m = nbg.nbg_mxv(c, nbg.FP64, "PLUS", "SECOND", A, x)
print(nbg.nbg_vector_export_dense(c, m)[:10])
rp, ci = nbg.nbg_matrix_export_csr(c, A)
print(np.diff(rp)[:10])
