# which kernels compile in each e2e iteration (new matrix per iteration)
import sys, os, glob, time; sys.path.insert(0, '.')
import torch
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
c = nbg.nbg_init(nbg.NONBLOCKING, 0, torch.cuda.current_stream().cuda_stream)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, int(os.environ.get("SCALE", "16")), 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0] - 1
dump = os.environ["NBG_JIT_DUMP"]
seen = set(glob.glob(dump + "/*.cu"))
for it in range(4):
    s0 = nbg.nbg_get_stats(c)
    t0 = time.perf_counter()
    A2 = nbg.nbg_matrix_from_csr(c, n, n, rp, ci, type=nbg.FP32)
    d2 = nbg.nbg_vector_from_dense(c, nbg.INT32, d)
    for rep in range(2):
        r, s, _ = nbg.nbg_pagerank(c, A2, d2, tol=1e-6, itermax=100)
        nbg.nbg_vector_free(c, r)
    nbg.nbg_sync(c)
    s1 = nbg.nbg_get_stats(c)
    now = set(glob.glob(dump + "/*.cu"))
    print(f"iter {it}: {1e3*(time.perf_counter()-t0):.1f} ms  jit {s1['jit_compiles']-s0['jit_compiles']}  plans_built {s1['plans_built']-s0['plans_built']}  new: {sorted(os.path.basename(x) for x in now - seen)}")
    seen = now
    nbg.nbg_vector_free(c, d2); nbg.nbg_matrix_free(c, A2)
