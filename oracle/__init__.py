"""CPU oracle -- TEST INFRASTRUCTURE, not the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with
``paper_2509_14211_b200`` (the CUDA path) and never imports it; the product never imports
this package (``tests/test_boundary.py`` checks both directions).

Contents
--------
``orc.c``   plain C: SplitMix64, R-MAT / Erdos-Renyi edge lists, CSR(AT) + out-degree build,
            plus-second mxv, and the Fig. 6 PageRank sweep in fp32/fp64.
``ops.py``  plain numpy semantics of the GraphBLAS subset the C ABI exposes (apply,
            ewise_mult, ewise_add, mxv, reduce, convert) over full / iso / empty vectors.
``__init__`` a ctypes loader that compiles ``orc.c`` with gcc (``-O2 -ffp-contract=off``).

Pins (what ties this oracle to something other than itself) live in ``tests/test_oracle.py``,
``tests/test_oracle_ops_pins.py`` (every operator branch of ops.py, ``convert``, the fp32 mxv, the
R-MAT level-bit order) and ``tests/test_sparse_oracle.py``; DESIGN.md §4 lists them per function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "orc.c")
_LIB = os.path.join(_HERE, "liborc.so")
_lock = threading.Lock()
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)


_LIB_OMP = os.path.join(_HERE, "liborc_omp.so")


def build(force: bool = False, omp: bool = False) -> str:
    """Compile orc.c -> liborc.so (plain gcc, no FMA contraction, no fast-math).  omp=True builds
    the same source with -fopenmp -> liborc_omp.so (row loop over threads; identical results),
    used only as the all-core CPU baseline of bench.py."""
    out = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math"]
                              + (["-fopenmp"] if omp else []) + ["-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


_lib_omp = None


def _bind(L):
    for nm, fp in (("orc_pagerank_f64", _f64p), ("orc_pagerank_f32", _f32p)):
        f = getattr(L, nm)
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int64, _i64p, _i32p, _i32p, ctypes.c_double, ctypes.c_int,
                      ctypes.c_int, ctypes.c_double, fp, _f64p, _f64p]
    return L


def lib_omp():
    """The OpenMP build (threads from OMP_NUM_THREADS, default: all host cores)."""
    global _lib_omp
    with _lock:
        if _lib_omp is None:
            _lib_omp = _bind(ctypes.CDLL(build(omp=True)))
    return _lib_omp


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            L.orc_sm64.restype = ctypes.c_uint64
            L.orc_sm64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
            L.orc_rmat_edges.restype = None
            L.orc_rmat_edges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, _i32p, _i32p]
            L.orc_er_edges.restype = None
            L.orc_er_edges.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, _i32p, _i32p]
            L.orc_build_csr.restype = ctypes.c_int64
            L.orc_build_csr.argtypes = [ctypes.c_int64, ctypes.c_int64, _i32p, _i32p, _i64p, _i32p, _i32p]
            L.orc_mxv_plus_f64.restype = None
            L.orc_mxv_plus_f64.argtypes = [ctypes.c_int64, _i64p, _i32p, _f64p, _f64p]
            L.orc_mxv_plus_f32.restype = None
            L.orc_mxv_plus_f32.argtypes = [ctypes.c_int64, _i64p, _i32p, _f32p, _f32p]
            for nm, fp in (("orc_pagerank_f64", _f64p), ("orc_pagerank_f32", _f32p)):
                f = getattr(L, nm)
                f.restype = ctypes.c_int
                f.argtypes = [ctypes.c_int64, _i64p, _i32p, _i32p, ctypes.c_double, ctypes.c_int,
                              ctypes.c_int, ctypes.c_double, fp, _f64p, _f64p]
            L.orc_sweep_rows_f32.restype = None
            L.orc_sweep_rows_f32.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i32p, _f32p,
                                             ctypes.c_float, _f32p]
            _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def sm64(key: int, k: int) -> int:
    return int(lib().orc_sm64(key & (2**64 - 1), k & (2**64 - 1)))


def rmat_edges(scale: int, edge_factor: int, seed: int):
    m = edge_factor << scale
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    lib().orc_rmat_edges(scale, m, seed, _p(src, _i32p), _p(dst, _i32p))
    return src, dst


def er_edges(logn: int, mean_deg: int, seed: int):
    m = mean_deg << logn
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    lib().orc_er_edges(logn, m, seed, _p(src, _i32p), _p(dst, _i32p))
    return src, dst


def read_mtx(path):
    """Matrix Market coordinate file -> (n, src, dst) edge list, written from the format's own
    definition (NIST Matrix Market exchange format): header "%%MatrixMarket matrix coordinate
    <field> <symmetry>", '%' comments, size line "M N NNZ", NNZ 1-based lines "i j [value]".
    Entry (i, j) is the edge i -> j; symmetric files contribute (j, i) too for i != j; values are
    ignored.  n = max(M, N).  Plain Python line by line (test infrastructure; small files)."""
    with open(path) as f:
        head = f.readline().split()
        if len(head) < 5 or head[0] != "%%MatrixMarket" or head[1].lower() != "matrix" or head[2].lower() != "coordinate":
            raise ValueError("not a coordinate Matrix Market file")
        field, sym = head[3].lower(), head[4].lower()
        if field not in ("pattern", "real", "integer") or sym not in ("general", "symmetric"):
            raise ValueError("unsupported field / symmetry")
        line = f.readline()
        while line.strip() == "" or line.lstrip().startswith("%"):
            line = f.readline()
        M, N, NZ = (int(v) for v in line.split()[:3])
        src, dst = [], []
        got = 0
        while got < NZ:
            line = f.readline()
            if line == "":
                raise ValueError("file ends early")
            t = line.split()
            if not t or t[0].startswith("%"):
                continue
            i, j = int(t[0]), int(t[1])
            if not (1 <= i <= M and 1 <= j <= N):
                raise IndexError("index out of range")
            src.append(i - 1)
            dst.append(j - 1)
            if sym == "symmetric" and i != j:
                src.append(j - 1)
                dst.append(i - 1)
            got += 1
    return max(M, N), np.array(src, np.int32), np.array(dst, np.int32)


def build_csr(n: int, src: np.ndarray, dst: np.ndarray):
    """-> (rowptr int64[n+1], colidx int32[nnz], deg int32[n]) of AT (edge u->v at AT[v,u])."""
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    m = src.shape[0]
    rowptr = np.zeros(n + 1, np.int64)
    colidx = np.empty(max(m, 1), np.int32)
    deg = np.zeros(n, np.int32)
    nnz = lib().orc_build_csr(n, m, _p(src, _i32p), _p(dst, _i32p), _p(rowptr, _i64p),
                              _p(colidx, _i32p), _p(deg, _i32p))
    if nnz < 0:
        raise MemoryError("orc_build_csr")
    return rowptr, colidx[:nnz].copy(), deg


def mxv_plus(rowptr, colidx, x):
    n = rowptr.shape[0] - 1
    if x.dtype == np.float64:
        m = np.empty(n, np.float64)
        lib().orc_mxv_plus_f64(n, _p(rowptr, _i64p), _p(colidx, _i32p), _p(x, _f64p), _p(m, _f64p))
    else:
        x = np.ascontiguousarray(x, np.float32)
        m = np.empty(n, np.float32)
        lib().orc_mxv_plus_f32(n, _p(rowptr, _i64p), _p(colidx, _i32p), _p(x, _f32p), _p(m, _f32p))
    return m


def pagerank(rowptr, colidx, deg, *, alpha=0.85, dtype=np.float64, uniform=True, itermax=20, tol=-1.0,
             threads=False):
    """Fig. 6 PageRank sweep.  -> (r, sweeps, delta_hist, ds_hist).
    threads=True runs the OpenMP build (same results; bench.py's all-core baseline only)."""
    n = rowptr.shape[0] - 1
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    colidx = np.ascontiguousarray(colidx, np.int32)
    deg = np.ascontiguousarray(deg, np.int32)
    r = np.empty(n, dtype)
    dh = np.zeros(max(itermax, 1), np.float64)
    sh = np.zeros(max(itermax, 1), np.float64)
    L = lib_omp() if threads else lib()
    f = L.orc_pagerank_f64 if dtype == np.float64 else L.orc_pagerank_f32
    fp = _f64p if dtype == np.float64 else _f32p
    sweeps = f(n, _p(rowptr, _i64p), _p(colidx, _i32p), _p(deg, _i32p), float(alpha), int(uniform),
               int(itermax), float(tol), _p(r, fp), _p(dh, _f64p), _p(sh, _f64p))
    if sweeps < 0:
        raise MemoryError("orc_pagerank")
    return r, sweeps, dh[:sweeps].copy(), sh[:sweeps].copy()


def sweep_rows_f32(lo, hi, rowptr, colidx, y, c):
    out = np.empty(hi - lo, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    lib().orc_sweep_rows_f32(lo, hi, _p(rowptr, _i64p), _p(colidx, _i32p), _p(y, _f32p),
                             float(np.float32(c)), _p(out, _f32p))
    return out
