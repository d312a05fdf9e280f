"""Plain numpy semantics of the GraphBLAS subset (TEST INFRASTRUCTURE -- see oracle/__init__.py).

Vectors are modelled as ``None`` (an empty vector: no stored entries) or a dense numpy array
(a full vector; an iso vector is the same array with one value repeated).  Every operator is
evaluated element by element in its OUTPUT type T, with its inputs and constants first
converted to T -- the typed-operator reading (reading R1) of GraphBLAS's
``GrB_PLUS_FP32``-style operators.  numpy's float32/float64 ufuncs are single IEEE
round-to-nearest operations, so each line below is one rounding in T.

Passages followed:
  apply             SPEC.md:183-189, Fig. 4 (VectorApply wraps its base)
  ewise_mult        SPEC.md:190-196 (intersection: empty if either side is empty)
  ewise_add         SPEC.md:197-203 (union: op where both present, else the present value)
  mxv               SPEC.md:204-210, Fig. 3 (identity, add, mul); dense output
  reduce            SPEC.md:211-217 (empty -> identity)
  convert
Float PLUS reductions return the exact sum of the terms rounded once to float64
(``math.fsum``): the plain definition of "sum" (reading R4 in DESIGN.md).
"""
from __future__ import annotations

import math

import numpy as np

DT = {"bool": np.bool_, "int32": np.int32, "int64": np.int64, "fp32": np.float32, "fp64": np.float64}


def _is_float(T):
    return np.dtype(T).kind == "f"


def _c(v, T):
    """Constant converted to T (round to nearest for floats, truncation for ints)."""
    if np.dtype(T) == np.bool_:
        return np.bool_(v != 0)
    return np.array(v).astype(T)[()]


def convert(x, T):
    if x is None:
        return None
    if np.dtype(T) == np.bool_:
        return x != 0
    if np.dtype(x.dtype) == np.bool_:
        return x.astype(T)
    if _is_float(T):
        return x.astype(T)        # int/float -> float: round to nearest
    if _is_float(x.dtype):
        with np.errstate(invalid="ignore"):
            return np.trunc(x).astype(T)
    return x.astype(T)


def _compute_type(T):
    # bool outputs are computed in int64 and normalised to 0/1 (reading R1)
    return np.int64 if np.dtype(T) == np.bool_ else T


def _finish(v, T):
    if np.dtype(T) == np.bool_:
        return v != 0
    return np.asarray(v, dtype=T)


def _div(a, b, T):
    if _is_float(T):
        with np.errstate(divide="ignore", invalid="ignore"):
            return a / b
    out = np.zeros_like(a)
    nz = b != 0
    # C-style truncating integer division in exact integer arithmetic; x/0 := 0 (reading R2)
    an, bn = a[nz].astype(np.int64), b[nz].astype(np.int64)
    with np.errstate(all="ignore"):
        # magnitudes as uint64 (|INT64_MIN| = 2^63 exactly), quotient toward zero, then the sign
        mag = np.abs(an).astype(np.uint64) // np.abs(bn).astype(np.uint64)
        neg = (an < 0) != (bn < 0)
        q = np.where(neg, (np.uint64(0) - mag).astype(np.int64), mag.astype(np.int64))
    out[nz] = q.astype(a.dtype)
    return out


def unop(code, x, T, c0=0.0, c1=0.0):
    if x is None:
        return None
    C = _compute_type(T)
    v = convert(x, C)
    k0, k1 = _c(c0, C), _c(c1, C)
    with np.errstate(all="ignore"):
        if code == "IDENTITY":
            r = v
        elif code == "AINV":
            r = -v
        elif code == "ABS":
            r = np.abs(v)
        elif code == "MINV":
            r = _div(np.ones_like(v), v, C)
        elif code == "ADD_C":
            r = v + k0
        elif code == "MUL_C":
            r = v * k0
        elif code == "AXPB":
            r = (k0 * v) + k1           # two roundings in T: fl(fl(c0*x) + c1)
        elif code == "ABS_SUB_C":
            r = np.abs(v - k0)
        elif code == "RECIP_SCALED":
            nz = v != 0
            r = np.zeros_like(v)
            r[nz] = _div(np.full(int(nz.sum()), k0, dtype=C), v[nz], C)
        elif code == "ISZERO":
            r = (v == 0).astype(C)
        else:
            raise ValueError(code)
    return _finish(r, T)


def binop(code, x, y, T, c0=0.0):
    C = _compute_type(T)
    a = convert(x, C)
    b = convert(y, C)
    with np.errstate(all="ignore"):
        if code == "PLUS":
            r = a + b
        elif code == "MINUS":
            r = a - b
        elif code == "TIMES":
            r = a * b
        elif code == "DIV":
            r = _div(a, b, C)
        elif code == "MIN":
            r = np.fmin(a, b)
        elif code == "MAX":
            r = np.fmax(a, b)
        elif code == "FIRST":
            r = a
        elif code == "SECOND":
            r = b
        elif code == "ABSDIFF":
            r = np.abs(a - b)
        elif code == "MAX_DIVX_C":     # Fig. 6: (x, y) -> max(x / damping, y)
            r = np.fmax(_div(a, np.full_like(a, _c(c0, C)), C), b)
        else:
            raise ValueError(code)
    return _finish(r, T)


def ewise_mult(code, u, v, T, c0=0.0):
    if u is None or v is None:
        return None
    return binop(code, u, v, T, c0)


def ewise_add(code, u, v, T, c0=0.0):
    if u is None and v is None:
        return None
    if u is None:
        return convert(v, T)
    if v is None:
        return convert(u, T)
    return binop(code, u, v, T, c0)


def apply_bind2nd(code, u, s, T, c0=0.0):
    if u is None:
        return None
    return binop(code, u, np.full(u.shape[0], s), T, c0)


def _ident(monoid, T):
    """Identity of the monoid in T: 0 for PLUS, +/-inf for float MIN/MAX, the largest / smallest
    value of T for integer MIN/MAX (the value an empty fold yields)."""
    if monoid == "PLUS":
        return _c(0, T)
    if _is_float(T):
        return _c(math.inf if monoid == "MIN" else -math.inf, T)
    if np.dtype(T) == np.bool_:
        return _c(1 if monoid == "MIN" else 0, T)
    info = np.iinfo(np.dtype(T))
    return np.array(info.max if monoid == "MIN" else info.min, dtype=T)[()]


def reduce(monoid, v, T):
    """Fold of the stored values.  PLUS on floats: exact sum rounded once."""
    if v is None or v.shape[0] == 0:
        return _ident(monoid, T)
    if monoid == "PLUS":
        if _is_float(v.dtype) or _is_float(T):
            return _c(math.fsum(float(z) for z in v.astype(np.float64)), T)
        return _c(int(v.astype(np.int64).sum(dtype=np.int64)), T)
    if monoid == "MIN":
        return _c(np.fmin.reduce(v), T)
    if monoid == "MAX":
        return _c(np.fmax.reduce(v), T)
    raise ValueError(monoid)


def mxv(add, mul, rowptr, colidx, vals, x, T, iso=1.0):
    """w[i] = fold_add(identity, mul(A[i,j], x[j]) for stored A[i,j], j ascending) (Fig. 3).

    mul is evaluated in T; PLUS folds of floats accumulate in float64 in ascending j and the
    row result is rounded once to T (reading Q4).  An empty row yields the identity
    (dense output semantics).  vals None => iso-valued matrix with value ``iso``.
    """
    n = rowptr.shape[0] - 1
    C = _compute_type(T)
    out = np.empty(n, dtype=T)
    if x is None:
        out[:] = _ident(add, T)
        return out
    xc = convert(x, C)
    for i in range(n):
        lo, hi = int(rowptr[i]), int(rowptr[i + 1])
        cols = colidx[lo:hi]
        a = (np.full(hi - lo, iso) if vals is None else vals[lo:hi])
        prod = binop(mul, a, xc[cols], C)
        if add == "PLUS":
            if _is_float(C):
                acc = 0.0
                for z in prod:
                    acc += float(z)          # fp64, ascending j
                out[i] = _c(acc, T)
            else:
                out[i] = _c(int(np.asarray(prod, np.int64).sum()), T)
        elif add == "MIN":
            out[i] = _c(np.fmin.reduce(prod), T) if prod.size else _ident("MIN", T)
        elif add == "MAX":
            out[i] = _c(np.fmax.reduce(prod), T) if prod.size else _ident("MAX", T)
        else:
            raise ValueError(add)
    return out
