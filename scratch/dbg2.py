import sys; sys.path.insert(0,'.')
from paper_2509_14211_b200 import nbg
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 10, 8, 1)
for run in range(3):
    print("=== run", run, file=sys.stderr)
    r, s, h = nbg.nbg_pagerank(c, A, deg, tol=-1, itermax=5, type=nbg.FP32)
    print(nbg.nbg_get_stats(c), file=sys.stderr)
