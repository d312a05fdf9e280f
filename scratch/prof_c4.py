import sys, time; sys.path.insert(0,'.')
import torch
from paper_2509_14211_b200 import nbg
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
torch.cuda.set_device(0)
c = nbg.nbg_init(nbg.NONBLOCKING, 0, torch.cuda.current_stream().cuda_stream)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, scale, 16, 1)
for i in range(3):
    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=1e-6, itermax=100, type=nbg.FP32)
    nbg.nbg_vector_free(c, r)
nbg.nbg_sync(c)
print("sweeps", s, nbg.nbg_get_stats(c))
