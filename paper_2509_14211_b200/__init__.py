"""paper_2509_14211_b200 -- B200-native nonblocking GraphBLAS hot path (arxiv 2509.14211).

The product is libnbg.so (C ABI in include/nbg.h; CUDA kernels for sm_100a, NVRTC-generated
fused regions, NCCL for the row-partitioned exchange).  ``paper_2509_14211_b200.nbg`` is the
thin ctypes binding with the same names.  Build in-tree with
``python -m paper_2509_14211_b200.build``.
"""


def load():
    """Import the binding (raises ImportError if libnbg.so is missing -- no fallback)."""
    from . import nbg
    return nbg
