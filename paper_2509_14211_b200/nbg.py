"""Thin ctypes binding of the C ABI (include/nbg.h) -- argument marshalling only.

Every function has the C name, takes the context first, returns the C out-parameters as Python
values and raises ``NbgError`` on a non-zero status.  All computation happens in libnbg.so
(CUDA kernels for sm_100a); there is no Python or CPU fallback: if the library is missing this
module raises at import.

Arrays: a numpy array is passed as NBG_HOST memory, a torch CUDA tensor as NBG_DEVICE memory
(its data pointer).  PyTorch is used only for device memory / streams (plumbing).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(_HERE, "libnbg.so")
if not os.path.exists(LIBPATH):
    raise ImportError(f"libnbg.so not built ({LIBPATH}); run `python -m paper_2509_14211_b200.build`")
lib = ctypes.CDLL(LIBPATH, mode=ctypes.RTLD_GLOBAL)

# ---------------------------------------------------------------- enums (mirror nbg.h)
SUCCESS, NULL_POINTER, INVALID_VALUE, DIMENSION_MISMATCH, DOMAIN_MISMATCH, INDEX_OUT_OF_BOUNDS, \
    INVALID_OBJECT, OUT_OF_MEMORY, NOT_IMPLEMENTED, PANIC = range(10)
STATUS_NAMES = ["SUCCESS", "NULL_POINTER", "INVALID_VALUE", "DIMENSION_MISMATCH", "DOMAIN_MISMATCH",
                "INDEX_OUT_OF_BOUNDS", "INVALID_OBJECT", "OUT_OF_MEMORY", "NOT_IMPLEMENTED", "PANIC"]
BOOL, INT32, INT64, FP32, FP64 = range(5)
BLOCKING, NONBLOCKING = 0, 1
HOST, DEVICE = 0, 1
COPY, BORROW = 0, 1
IDENTITY, AINV, ABS, MINV, ADD_C, MUL_C, AXPB, ABS_SUB_C, RECIP_SCALED, ISZERO = range(10)
PLUS, MINUS, TIMES, DIV, MIN, MAX, FIRST, SECOND, ABSDIFF, MAX_DIVX_C = range(10)
GRAPH_RMAT, GRAPH_ER = 0, 1
FORMAT_FULL, FORMAT_ISO, FORMAT_SPARSE, FORMAT_BITSET, FORMAT_EMPTY = range(5)
FORMAT_NAMES = ["full", "iso", "sparse", "bitset", "empty"]
PR_UNIFORM, PR_DROP = 0, 1
FLAG_DETERMINISTIC = 1
DIST_EXCHANGE_COLLECTIVE, DIST_EXCHANGE_PEER = 0, 1

UNOPS = {n: i for i, n in enumerate(["IDENTITY", "AINV", "ABS", "MINV", "ADD_C", "MUL_C", "AXPB", "ABS_SUB_C",
                                      "RECIP_SCALED", "ISZERO"])}
BINOPS = {n: i for i, n in enumerate(["PLUS", "MINUS", "TIMES", "DIV", "MIN", "MAX", "FIRST", "SECOND", "ABSDIFF",
                                       "MAX_DIVX_C"])}
NP_OF = {BOOL: np.uint8, INT32: np.int32, INT64: np.int64, FP32: np.float32, FP64: np.float64}
TYPE_OF = {"bool": BOOL, "int32": INT32, "int64": INT64, "fp32": FP32, "fp64": FP64}


class NbgError(RuntimeError):
    def __init__(self, status, fn, msg=""):
        self.status = status
        super().__init__(f"{fn} -> {STATUS_NAMES[status] if 0 <= status < 10 else status}: {msg}")


# ---------------------------------------------------------------- structs
class nbg_config(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("flags", ctypes.c_int)]


class nbg_unop(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("c0", ctypes.c_double), ("c1", ctypes.c_double)]


class nbg_binop(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("c0", ctypes.c_double)]


class nbg_semiring(ctypes.Structure):
    _fields_ = [("add", ctypes.c_int), ("mul", ctypes.c_int), ("mul_c0", ctypes.c_double)]


class nbg_graphgen(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("scale", ctypes.c_int), ("edge_factor", ctypes.c_int), ("seed", ctypes.c_uint64)]


class nbg_pr_params(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("tol", ctypes.c_double), ("itermax", ctypes.c_int),
                ("dangling", ctypes.c_int), ("type", ctypes.c_int)]


class nbg_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("waits", "plans_built", "plan_hits", "jit_compiles", "kernels_launched",
                                                "vectors_materialized", "intermediates_elided", "memo_hits",
                                                "side_outputs", "bytes_materialized", "host_plan_ns")] + \
               [("jit_ms", ctypes.c_double), ("structured_regions", ctypes.c_uint64), ("structured_index_loops", ctypes.c_uint64),
                ("jit_disk_hits", ctypes.c_uint64)]


vp = ctypes.c_void_p
i64 = ctypes.c_int64
pvp = ctypes.POINTER(ctypes.c_void_p)

# every exported symbol of nbg.h with its argument types
SIGNATURES = {
    "nbg_init": [pvp, ctypes.POINTER(nbg_config)],
    "nbg_finalize": [vp],
    "nbg_last_error": [vp, ctypes.c_char_p, ctypes.c_size_t],
    "nbg_sync": [vp],
    "nbg_unop_define": [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)],
    "nbg_binop_define": [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)],
    "nbg_get_stats": [vp, ctypes.POINTER(nbg_stats)],
    "nbg_reset_stats": [vp],
    "nbg_set_timing": [vp, ctypes.c_int],
    "nbg_get_timing": [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)],
    "nbg_matrix_from_csr": [vp, pvp, i64, i64, i64, vp, vp, vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int],
    "nbg_matrix_from_edges": [vp, pvp, pvp, i64, i64, vp, vp, ctypes.c_int],
    "nbg_matrix_from_mtx": [vp, pvp, pvp, ctypes.c_char_p],
    "nbg_graph_edges": [vp, ctypes.POINTER(nbg_graphgen), vp, vp, ctypes.c_int],
    "nbg_matrix_from_generator": [vp, pvp, pvp, ctypes.POINTER(nbg_graphgen)],
    "nbg_matrix_nrows": [vp, vp, ctypes.POINTER(i64)],
    "nbg_matrix_ncols": [vp, vp, ctypes.POINTER(i64)],
    "nbg_matrix_nnz": [vp, vp, ctypes.POINTER(i64)],
    "nbg_matrix_export_csr": [vp, vp, vp, vp, ctypes.c_int],
    "nbg_matrix_free": [vp, vp],
    "nbg_matrix_row_block": [vp, pvp, vp, i64, i64],
    "nbg_vector_new": [vp, pvp, ctypes.c_int, i64],
    "nbg_vector_new_const": [vp, pvp, ctypes.c_int, i64, ctypes.c_double],
    "nbg_vector_from_dense": [vp, pvp, ctypes.c_int, i64, vp, ctypes.c_int, ctypes.c_int],
    "nbg_vector_export_dense": [vp, vp, vp, ctypes.c_int],
    "nbg_vector_size": [vp, vp, ctypes.POINTER(i64)],
    "nbg_vector_type": [vp, vp, ctypes.POINTER(ctypes.c_int)],
    "nbg_vector_nvals": [vp, vp, ctypes.POINTER(i64)],
    "nbg_vector_is_materialized": [vp, vp, ctypes.POINTER(ctypes.c_int)],
    "nbg_vector_device_ptr": [vp, vp, pvp],
    "nbg_vector_free": [vp, vp],
    "nbg_vector_from_sparse": [vp, pvp, ctypes.c_int, i64, i64, vp, vp, ctypes.c_int],
    "nbg_vector_export_sparse": [vp, vp, ctypes.POINTER(i64), vp, vp, ctypes.c_int],
    "nbg_vector_format": [vp, vp, ctypes.POINTER(ctypes.c_int)],
    "nbg_vector_estimated_fill": [vp, vp, ctypes.POINTER(ctypes.c_double)],
    "nbg_scalar_new": [vp, pvp, ctypes.c_int, ctypes.c_double],
    "nbg_scalar_get": [vp, vp, ctypes.POINTER(ctypes.c_double)],
    "nbg_scalar_free": [vp, vp],
    "nbg_apply": [vp, pvp, ctypes.c_int, nbg_unop, vp],
    "nbg_apply_bind2nd": [vp, pvp, ctypes.c_int, nbg_binop, vp, vp],
    "nbg_ewise_mult": [vp, pvp, ctypes.c_int, nbg_binop, vp, vp],
    "nbg_ewise_add": [vp, pvp, ctypes.c_int, nbg_binop, vp, vp],
    "nbg_convert": [vp, pvp, ctypes.c_int, vp],
    "nbg_mxv": [vp, pvp, ctypes.c_int, nbg_semiring, vp, vp],
    "nbg_reduce": [vp, pvp, ctypes.c_int, ctypes.c_int, vp],
    "nbg_scalar_apply": [vp, pvp, ctypes.c_int, nbg_unop, vp],
    "nbg_vector_wait": [vp, vp],
    "nbg_scalar_wait": [vp, vp],
    "nbg_wait_all": [vp],
    "nbg_pagerank": [vp, vp, vp, ctypes.POINTER(nbg_pr_params), pvp, ctypes.POINTER(ctypes.c_int), vp],
    "nbg_partition_rows": [vp, i64, ctypes.c_int, i64, vp],
    "nbg_dist_unique_id": [vp],
    "nbg_dist_init": [vp, ctypes.c_int, ctypes.c_int, vp],
    "nbg_vector_allgather": [vp, pvp, vp, vp],
    "nbg_scalar_allreduce": [vp, pvp, vp],
    "nbg_pagerank_dist": [vp, vp, vp, vp, i64, ctypes.POINTER(nbg_pr_params), pvp, ctypes.POINTER(ctypes.c_int), vp],
    "nbg_xacc_encode": [vp, i64, vp],
    "nbg_xacc_decode": [vp, vp],
    "nbg_scalar_export_slot": [vp, vp, vp],
    "nbg_dist_exchange_plan": [vp, ctypes.c_int, i64, vp, vp],
    "nbg_dist_init_loopback": [vp, ctypes.c_int],
    "nbg_dist_set_exchange": [vp, ctypes.c_int],
    "nbg_guard_selftest": [vp],
    "nbg_dist_graph_from_generator": [vp, ctypes.POINTER(nbg_graphgen), i64, pvp, pvp, vp, vp],
    "nbg_vector_allgather_reduce": [vp, pvp, vp, vp, i64, ctypes.c_int, vp, vp],
}
for _n, _a in SIGNATURES.items():
    _f = getattr(lib, _n)
    _f.argtypes = _a
    _f.restype = ctypes.c_int


def _err(ctx, fn, st):
    msg = ""
    if ctx:
        buf = ctypes.create_string_buffer(4096)
        lib.nbg_last_error(ctx, buf, 4096)
        msg = buf.value.decode(errors="replace")
    raise NbgError(st, fn, msg)


def _call(ctx, fn, *args):
    st = getattr(lib, fn)(*args)
    if st != SUCCESS:
        _err(ctx, fn, st)


def _ptr(a):
    """(address, space) of a numpy array (HOST) or a torch CUDA tensor (DEVICE)."""
    if a is None:
        return None, HOST
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, HOST
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), (DEVICE if a.is_cuda else HOST)
    if isinstance(a, int):
        return a, DEVICE
    raise TypeError(type(a))


# ---------------------------------------------------------------- context
def nbg_init(mode=NONBLOCKING, device=0, stream=None, flags=0):
    cfg = nbg_config(mode, device, stream, flags)
    ctx = ctypes.c_void_p()
    _call(None, "nbg_init", ctypes.byref(ctx), ctypes.byref(cfg))
    return ctx


def nbg_finalize(ctx):
    _call(None, "nbg_finalize", ctx)


def nbg_sync(ctx):
    _call(ctx, "nbg_sync", ctx)


def nbg_unop_define(name, expr):
    """Register a user unary operator (CUDA expression over x, c0, c1) -> its code."""
    code = ctypes.c_int()
    _call(None, "nbg_unop_define", name.encode(), expr.encode(), ctypes.byref(code))
    return code.value


def nbg_binop_define(name, expr):
    """Register a user binary operator (CUDA expression over x, y, c0) -> its code."""
    code = ctypes.c_int()
    _call(None, "nbg_binop_define", name.encode(), expr.encode(), ctypes.byref(code))
    return code.value


def nbg_get_stats(ctx):
    s = nbg_stats()
    _call(ctx, "nbg_get_stats", ctx, ctypes.byref(s))
    return {f: getattr(s, f) for f, _ in nbg_stats._fields_}


def nbg_reset_stats(ctx):
    _call(ctx, "nbg_reset_stats", ctx)


def nbg_set_timing(ctx, enable):
    _call(ctx, "nbg_set_timing", ctx, int(enable))


def nbg_get_timing(ctx, cls):
    ms = ctypes.c_double()
    n = i64()
    _call(ctx, "nbg_get_timing", ctx, cls.encode(), ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


# ---------------------------------------------------------------- matrices
def nbg_matrix_from_csr(ctx, nrows, ncols, rowptr, colidx, vals=None, type=FP32, iso=1.0, own=COPY):
    rp, sp = _ptr(rowptr)
    ci, _ = _ptr(colidx)
    va, _ = _ptr(vals)
    nnz = int(colidx.shape[0])
    A = ctypes.c_void_p()
    _call(ctx, "nbg_matrix_from_csr", ctx, ctypes.byref(A), nrows, ncols, nnz, rp, ci, va, type, float(iso), sp, own)
    return A


def nbg_matrix_from_edges(ctx, n, src, dst):
    s, sp = _ptr(src)
    d, _ = _ptr(dst)
    A, deg = ctypes.c_void_p(), ctypes.c_void_p()
    _call(ctx, "nbg_matrix_from_edges", ctx, ctypes.byref(A), ctypes.byref(deg), n, int(src.shape[0]), s, d, sp)
    return A, deg


def nbg_matrix_from_mtx(ctx, path):
    """Matrix Market coordinate file -> (AT, out-degree) (include/nbg.h nbg_matrix_from_mtx)."""
    A, deg = ctypes.c_void_p(), ctypes.c_void_p()
    _call(ctx, "nbg_matrix_from_mtx", ctx, ctypes.byref(A), ctypes.byref(deg), str(path).encode())
    return A, deg


def nbg_graph_edges(ctx, kind, scale, edge_factor, seed, src=None, dst=None):
    g = nbg_graphgen(kind, scale, edge_factor, seed)
    m = edge_factor << scale
    if src is None:
        src = np.empty(m, np.int32)
        dst = np.empty(m, np.int32)
    s, sp = _ptr(src)
    d, _ = _ptr(dst)
    _call(ctx, "nbg_graph_edges", ctx, ctypes.byref(g), s, d, sp)
    return src, dst


def nbg_matrix_from_generator(ctx, kind, scale, edge_factor, seed):
    g = nbg_graphgen(kind, scale, edge_factor, seed)
    A, deg = ctypes.c_void_p(), ctypes.c_void_p()
    _call(ctx, "nbg_matrix_from_generator", ctx, ctypes.byref(A), ctypes.byref(deg), ctypes.byref(g))
    return A, deg


def _i64_out(ctx, fn, h):
    v = i64()
    _call(ctx, fn, ctx, h, ctypes.byref(v))
    return v.value


def nbg_matrix_nrows(ctx, A):
    return _i64_out(ctx, "nbg_matrix_nrows", A)


def nbg_matrix_ncols(ctx, A):
    return _i64_out(ctx, "nbg_matrix_ncols", A)


def nbg_matrix_nnz(ctx, A):
    return _i64_out(ctx, "nbg_matrix_nnz", A)


def nbg_matrix_export_csr(ctx, A):
    n, nnz = nbg_matrix_nrows(ctx, A), nbg_matrix_nnz(ctx, A)
    rp = np.empty(n + 1, np.int64)
    ci = np.empty(max(nnz, 1), np.int32)
    _call(ctx, "nbg_matrix_export_csr", ctx, A, rp.ctypes.data, ci.ctypes.data, HOST)
    return rp, ci[:nnz]


def nbg_matrix_row_block(ctx, A, lo, hi):
    B = ctypes.c_void_p()
    _call(ctx, "nbg_matrix_row_block", ctx, ctypes.byref(B), A, int(lo), int(hi))
    return B


def nbg_matrix_free(ctx, A):
    _call(ctx, "nbg_matrix_free", ctx, A)


# ---------------------------------------------------------------- vectors / scalars
def _out():
    return ctypes.c_void_p()


def nbg_vector_new(ctx, type, n):
    v = _out()
    _call(ctx, "nbg_vector_new", ctx, ctypes.byref(v), type, n)
    return v


def nbg_vector_new_const(ctx, type, n, value):
    v = _out()
    _call(ctx, "nbg_vector_new_const", ctx, ctypes.byref(v), type, n, float(value))
    return v


def nbg_vector_from_dense(ctx, type, data, own=COPY, n=None):
    p, sp = _ptr(data)
    n = int(data.shape[0]) if n is None else n
    v = _out()
    _call(ctx, "nbg_vector_from_dense", ctx, ctypes.byref(v), type, n, p, sp, own)
    return v


def nbg_vector_type(ctx, v):
    t = ctypes.c_int()
    _call(ctx, "nbg_vector_type", ctx, v, ctypes.byref(t))
    return t.value


def nbg_vector_size(ctx, v):
    return _i64_out(ctx, "nbg_vector_size", v)


def nbg_vector_nvals(ctx, v):
    return _i64_out(ctx, "nbg_vector_nvals", v)


def nbg_vector_is_materialized(ctx, v):
    t = ctypes.c_int()
    _call(ctx, "nbg_vector_is_materialized", ctx, v, ctypes.byref(t))
    return bool(t.value)


def nbg_vector_export_dense(ctx, v, out=None):
    if out is None:
        out = np.empty(nbg_vector_size(ctx, v), NP_OF[nbg_vector_type(ctx, v)])
    p, sp = _ptr(out)
    _call(ctx, "nbg_vector_export_dense", ctx, v, p, sp)
    return out


def nbg_vector_device_ptr(ctx, v):
    p = ctypes.c_void_p()
    _call(ctx, "nbg_vector_device_ptr", ctx, v, ctypes.byref(p))
    return p.value


def nbg_vector_free(ctx, v):
    _call(ctx, "nbg_vector_free", ctx, v)


def nbg_vector_from_sparse(ctx, type, n, indices, values):
    """Sparse vector (include/nbg.h nbg_vector_from_sparse): int32 ascending indices + values."""
    nv = int(indices.shape[0])
    ip, sp = _ptr(indices)
    vp_, sp2 = _ptr(values)
    if sp != sp2:
        raise ValueError("indices and values must live in the same space")
    v = _out()
    _call(ctx, "nbg_vector_from_sparse", ctx, ctypes.byref(v), type, int(n), nv, ip, vp_, sp)
    return v


def nbg_vector_export_sparse(ctx, v):
    """-> (indices int32, values) of the present entries, ascending (two-call protocol)."""
    nv = i64(0)
    _call(ctx, "nbg_vector_export_sparse", ctx, v, ctypes.byref(nv), None, None, HOST)
    idx = np.empty(nv.value, np.int32)
    vals = np.empty(nv.value, NP_OF[nbg_vector_type(ctx, v)])
    if nv.value:
        _call(ctx, "nbg_vector_export_sparse", ctx, v, ctypes.byref(nv), idx.ctypes.data, vals.ctypes.data, HOST)
    return idx, vals


def nbg_vector_format(ctx, v):
    t = ctypes.c_int()
    _call(ctx, "nbg_vector_format", ctx, v, ctypes.byref(t))
    return t.value


def nbg_vector_estimated_fill(ctx, v):
    f = ctypes.c_double()
    _call(ctx, "nbg_vector_estimated_fill", ctx, v, ctypes.byref(f))
    return f.value


def nbg_scalar_new(ctx, type, value):
    s = _out()
    _call(ctx, "nbg_scalar_new", ctx, ctypes.byref(s), type, float(value))
    return s


def nbg_scalar_get(ctx, s):
    v = ctypes.c_double()
    _call(ctx, "nbg_scalar_get", ctx, s, ctypes.byref(v))
    return v.value


def nbg_scalar_free(ctx, s):
    _call(ctx, "nbg_scalar_free", ctx, s)


# ---------------------------------------------------------------- operations
def _code(c, table):
    return table[c] if isinstance(c, str) else int(c)


def nbg_apply(ctx, type, op, u, c0=0.0, c1=0.0):
    w = _out()
    _call(ctx, "nbg_apply", ctx, ctypes.byref(w), type, nbg_unop(_code(op, UNOPS), c0, c1), u)
    return w


def nbg_apply_bind2nd(ctx, type, op, u, s, c0=0.0):
    w = _out()
    _call(ctx, "nbg_apply_bind2nd", ctx, ctypes.byref(w), type, nbg_binop(_code(op, BINOPS), c0), u, s)
    return w


def nbg_ewise_mult(ctx, type, op, u, v, c0=0.0):
    w = _out()
    _call(ctx, "nbg_ewise_mult", ctx, ctypes.byref(w), type, nbg_binop(_code(op, BINOPS), c0), u, v)
    return w


def nbg_ewise_add(ctx, type, op, u, v, c0=0.0):
    w = _out()
    _call(ctx, "nbg_ewise_add", ctx, ctypes.byref(w), type, nbg_binop(_code(op, BINOPS), c0), u, v)
    return w


def nbg_convert(ctx, type, u):
    w = _out()
    _call(ctx, "nbg_convert", ctx, ctypes.byref(w), type, u)
    return w


def nbg_mxv(ctx, type, add, mul, A, u, mul_c0=0.0):
    w = _out()
    _call(ctx, "nbg_mxv", ctx, ctypes.byref(w), type, nbg_semiring(_code(add, BINOPS), _code(mul, BINOPS), mul_c0), A, u)
    return w


def nbg_reduce(ctx, type, monoid, u):
    s = _out()
    _call(ctx, "nbg_reduce", ctx, ctypes.byref(s), type, _code(monoid, BINOPS), u)
    return s


def nbg_scalar_apply(ctx, type, op, s, c0=0.0, c1=0.0):
    w = _out()
    _call(ctx, "nbg_scalar_apply", ctx, ctypes.byref(w), type, nbg_unop(_code(op, UNOPS), c0, c1), s)
    return w


def nbg_vector_wait(ctx, v):
    _call(ctx, "nbg_vector_wait", ctx, v)


def nbg_scalar_wait(ctx, s):
    _call(ctx, "nbg_scalar_wait", ctx, s)


def nbg_wait_all(ctx):
    _call(ctx, "nbg_wait_all", ctx)


# ---------------------------------------------------------------- PageRank / distributed
def nbg_pagerank(ctx, AT, deg, alpha=0.85, tol=-1.0, itermax=20, dangling=PR_UNIFORM, type=FP32):
    p = nbg_pr_params(alpha, tol, itermax, dangling, type)
    r = _out()
    sw = ctypes.c_int()
    hist = np.zeros(max(itermax, 1), np.float64)
    _call(ctx, "nbg_pagerank", ctx, AT, deg, ctypes.byref(p), ctypes.byref(r), ctypes.byref(sw), hist.ctypes.data)
    return r, sw.value, hist[:sw.value].copy()


def nbg_partition_rows(rowptr, nparts, bytes_per_row):
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    cuts = np.zeros(nparts + 1, np.int64)
    _call(None, "nbg_partition_rows", rowptr.ctypes.data, int(rowptr.shape[0] - 1), nparts, int(bytes_per_row),
          cuts.ctypes.data)
    return cuts


def nbg_dist_unique_id():
    buf = ctypes.create_string_buffer(128)
    _call(None, "nbg_dist_unique_id", ctypes.cast(buf, ctypes.c_void_p))
    return bytes(buf.raw)


def nbg_dist_init(ctx, rank, nranks, uid: bytes):
    buf = ctypes.create_string_buffer(uid, 128)
    _call(ctx, "nbg_dist_init", ctx, rank, nranks, ctypes.cast(buf, ctypes.c_void_p))


def nbg_vector_allgather(ctx, u, cuts):
    cuts = np.ascontiguousarray(cuts, np.int64)
    w = _out()
    _call(ctx, "nbg_vector_allgather", ctx, ctypes.byref(w), u, cuts.ctypes.data)
    return w


def nbg_scalar_allreduce(ctx, s):
    w = _out()
    _call(ctx, "nbg_scalar_allreduce", ctx, ctypes.byref(w), s)
    return w


def nbg_pagerank_dist(ctx, AT_blk, deg_blk, cuts, ncols_g, alpha=0.85, tol=-1.0, itermax=20, dangling=PR_UNIFORM,
                      type=FP32):
    cuts = np.ascontiguousarray(cuts, np.int64)
    p = nbg_pr_params(alpha, tol, itermax, dangling, type)
    r = _out()
    sw = ctypes.c_int()
    hist = np.zeros(max(itermax, 1), np.float64)
    _call(ctx, "nbg_pagerank_dist", ctx, AT_blk, deg_blk, cuts.ctypes.data, int(ncols_g), ctypes.byref(p),
          ctypes.byref(r), ctypes.byref(sw), hist.ctypes.data)
    return r, sw.value, hist[:sw.value].copy()


def nbg_xacc_encode(terms):
    """Host only: the 16-word exact-accumulator slot of a list of float64 terms."""
    t = np.ascontiguousarray(terms, np.float64)
    slot = np.zeros(16, np.uint64)
    _call(None, "nbg_xacc_encode", t.ctypes.data if t.size else None, int(t.shape[0]), slot.ctypes.data)
    return slot


def nbg_xacc_decode(slot):
    slot = np.ascontiguousarray(slot, np.uint64)
    v = ctypes.c_double()
    _call(None, "nbg_xacc_decode", slot.ctypes.data, ctypes.byref(v))
    return v.value


def nbg_scalar_export_slot(ctx, s):
    slot = np.zeros(16, np.uint64)
    _call(ctx, "nbg_scalar_export_slot", ctx, s, slot.ctypes.data)
    return slot


def nbg_dist_init_loopback(ctxs):
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value if isinstance(c, ctypes.c_void_p) else c for c in ctxs])
    _call(None, "nbg_dist_init_loopback", ctypes.cast(arr, ctypes.c_void_p), len(ctxs))


def nbg_guard_selftest(ctx):
    """include/nbg.h nbg_guard_selftest (NBG_GUARD=1 red-zone check of an intentional overflow)."""
    _call(ctx, "nbg_guard_selftest", ctx)


def nbg_dist_set_exchange(ctx, mode):
    """include/nbg.h nbg_dist_set_exchange: DIST_EXCHANGE_COLLECTIVE (default) or DIST_EXCHANGE_PEER
    (the exchange fused into the producing kernel as peer stores)."""
    _call(ctx, "nbg_dist_set_exchange", ctx, int(mode))


def nbg_dist_exchange_plan(cuts, ncols_g):
    cuts = np.ascontiguousarray(cuts, np.int64)
    P = cuts.shape[0] - 1
    off = np.zeros(P, np.int64)
    cnt = np.zeros(P, np.int64)
    _call(None, "nbg_dist_exchange_plan", cuts.ctypes.data, P, int(ncols_g), off.ctypes.data, cnt.ctypes.data)
    return off, cnt


def nbg_dist_graph_from_generator(ctx, kind, scale, edge_factor, seed, nranks=1, bytes_per_row=20):
    g = nbg_graphgen(kind, scale, edge_factor, seed)
    A = _out()
    d = _out()
    cuts = np.zeros(nranks + 1, np.int64)
    ncg = ctypes.c_int64()
    _call(ctx, "nbg_dist_graph_from_generator", ctx, ctypes.byref(g), int(bytes_per_row), ctypes.byref(A),
          ctypes.byref(d), cuts.ctypes.data, ctypes.byref(ncg))
    return A, d, cuts, ncg.value


def nbg_vector_allgather_reduce(ctx, u_blk, cuts, ncols_g, scalars=()):
    cuts = np.ascontiguousarray(cuts, np.int64)
    w = _out()
    k = len(scalars)
    sin = (ctypes.c_void_p * max(k, 1))(*scalars)
    sout = (ctypes.c_void_p * max(k, 1))()
    _call(ctx, "nbg_vector_allgather_reduce", ctx, ctypes.byref(w), u_blk, cuts.ctypes.data, int(ncols_g), k,
          ctypes.cast(sin, ctypes.c_void_p), ctypes.cast(sout, ctypes.c_void_p))
    return w, [ctypes.c_void_p(sout[i]) for i in range(k)]


def jit_selftest():
    """NVRTC-compile representative generated regions (no GPU needed). -> (fails, log)."""
    f = lib.nbg_debug_jit_selftest
    f.restype = ctypes.c_int
    buf = ctypes.create_string_buffer(1 << 16)
    fails = f(buf, 1 << 16)
    return fails, buf.value.decode(errors="replace")
