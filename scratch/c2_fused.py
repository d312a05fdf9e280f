# the config-2 fused chain alone (for an ncu capture of its one kernel): T from argv (fp32 / fp64)
import sys; sys.path.insert(0, ".")
import inputs
from paper_2509_14211_b200 import nbg
import numpy as np
T = nbg.FP64 if sys.argv[1:] == ["fp64"] else nbg.FP32
x, y = inputs.uniform_vectors(1 << 24, 1, np.float64 if T == nbg.FP64 else np.float32)
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
vx, vy = nbg.nbg_vector_from_dense(c, T, x), nbg.nbg_vector_from_dense(c, T, y)
for _ in range(4):
    a = nbg.nbg_apply(c, T, "ADD_C", vy, 1.0); z = nbg.nbg_ewise_mult(c, T, "TIMES", vx, a)
    c1 = nbg.nbg_apply(c, T, "MUL_C", z, 0.5); c2 = nbg.nbg_ewise_add(c, T, "PLUS", c1, vx)
    c3 = nbg.nbg_ewise_mult(c, T, "TIMES", c2, vy); c4 = nbg.nbg_apply(c, T, "ABS_SUB_C", c3, 0.25)
    c5 = nbg.nbg_ewise_add(c, T, "MAX", c4, z); s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", c5)
    for h in (a, z, c1, c2, c3, c4, c5): nbg.nbg_vector_free(c, h)
    print(nbg.nbg_scalar_get(c, s)); nbg.nbg_scalar_free(c, s)
nbg.nbg_finalize(c)
