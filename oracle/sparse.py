"""Sparse-vector semantics of the GraphBLAS subset (TEST INFRASTRUCTURE -- see oracle/__init__.py;
only tests/ may import it).  SURVEY 8(f) NEXT-3.

A vector is ``SV(n, idx, vals)``: length n, strictly ascending int64 indices of the present
entries and their values (numpy dtype = the vector's type).  Values are computed by the dense
oracle (oracle/ops.py) on the gathered values, so every element is the same single rounding in the
output type.  Passages followed:

  representations     PAPER.md:111 (SparseVector / BitSetVector / FullVector)
  apply / bind2nd     SPEC.md:183-189: structure identical to the operand, values op-mapped
  ewise_mult          SPEC.md:190-196: entries at the INTERSECTION of the stored positions
  ewise_add           SPEC.md:197-203: UNION; both present -> op(u, v); one present -> that value
  reduce              SPEC.md:211-217: fold of the stored values, identity if none
  mxv                 SPEC.md:204-210: row i folds mul(A[i,j], x[j]) over stored A[i,j] with x[j]
                      present, ascending j; a row that meets no present x[j] yields the identity
                      (dense output, reading Q4 for the fp64 accumulation)
  estimated fill      PAPER.md:236-240: materialised = nnz / size; ewise_mult = product of the
                      operands' fills; apply = operand; ewise_add = f_u + f_v - f_u f_v (reading N1
                      in DESIGN.md: the average-case metadata estimator, the paper gives no formula)
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import ops


@dataclass
class SV:
    n: int
    idx: np.ndarray      # int64, strictly ascending
    vals: np.ndarray     # values of the present entries


def full(vals):
    """A full vector: every index present."""
    vals = np.asarray(vals)
    return SV(int(vals.shape[0]), np.arange(vals.shape[0], dtype=np.int64), vals)


def sparse(n, idx, vals):
    idx = np.asarray(idx, np.int64)
    assert np.all(np.diff(idx) > 0) and (idx.size == 0 or (idx[0] >= 0 and idx[-1] < n))
    return SV(int(n), idx, np.asarray(vals))


def apply(code, u: SV, T, c0=0.0, c1=0.0) -> SV:
    return SV(u.n, u.idx.copy(), ops.unop(code, u.vals, T, c0, c1))


def bind2nd(code, u: SV, s, T, c0=0.0) -> SV:
    return SV(u.n, u.idx.copy(), ops.binop(code, u.vals, np.full(u.idx.shape[0], s), T, c0))


def ewise_mult(code, u: SV, v: SV, T, c0=0.0) -> SV:
    both, iu, iv = np.intersect1d(u.idx, v.idx, assume_unique=True, return_indices=True)
    return SV(u.n, both.astype(np.int64), ops.binop(code, u.vals[iu], v.vals[iv], T, c0))


def ewise_add(code, u: SV, v: SV, T, c0=0.0) -> SV:
    allidx = np.union1d(u.idx, v.idx).astype(np.int64)
    out = np.empty(allidx.shape[0], dtype=T)
    inu = np.isin(allidx, u.idx)
    inv = np.isin(allidx, v.idx)
    pu = np.minimum(np.searchsorted(u.idx, allidx), max(u.idx.shape[0] - 1, 0))
    pv = np.minimum(np.searchsorted(v.idx, allidx), max(v.idx.shape[0] - 1, 0))
    b = inu & inv
    if b.any():
        out[b] = ops.binop(code, u.vals[pu[b]], v.vals[pv[b]], T, c0)
    ou = inu & ~inv
    if ou.any():
        out[ou] = ops.convert(u.vals[pu[ou]], T)
    ov = inv & ~inu
    if ov.any():
        out[ov] = ops.convert(v.vals[pv[ov]], T)
    return SV(u.n, allidx, out)


def reduce(monoid, u: SV, T):
    return ops.reduce(monoid, u.vals if u.idx.size else None, T)


def mxv(add, mul, rowptr, colidx, vals, x: SV, T, iso=1.0):
    """Dense w (T[nrows]): fold over stored A[i,j] with x[j] present."""
    n = rowptr.shape[0] - 1
    present = np.zeros(x.n, bool)
    present[x.idx] = True
    xd = np.zeros(x.n, dtype=x.vals.dtype)
    xd[x.idx] = x.vals
    C = ops._compute_type(T)
    out = np.empty(n, dtype=T)
    for i in range(n):
        lo, hi = int(rowptr[i]), int(rowptr[i + 1])
        cols = np.asarray(colidx[lo:hi], np.int64)
        keep = present[cols]
        a = np.full(hi - lo, iso) if vals is None else np.asarray(vals[lo:hi])
        terms = ops.binop(mul, a[keep], xd[cols[keep]], C)
        if add == "PLUS":
            if ops._is_float(T):
                acc = 0.0
                for t in terms.astype(np.float64):
                    acc += float(t)           # fp64, ascending j (reading Q4)
                out[i] = ops._c(acc, T)
            else:
                out[i] = ops._c(int(terms.astype(np.int64).sum()), T)
        else:
            ident = (math.inf if add == "MIN" else -math.inf) if ops._is_float(T) else \
                (np.iinfo(np.dtype(T)).max if add == "MIN" else np.iinfo(np.dtype(T)).min)
            r = ops._c(ident, T)
            for t in terms:
                r = np.fmin(r, t) if add == "MIN" else np.fmax(r, t)
            out[i] = ops._c(r, T)
    return out


def fill(u: SV) -> float:
    """Estimated (= actual) fill of a materialised vector: nnz / size."""
    return u.idx.shape[0] / u.n if u.n else 0.0


def fill_mult(fu: float, fv: float) -> float:
    return fu * fv                      # PAPER.md:237 "just the product of the sparsities"


def fill_add(fu: float, fv: float) -> float:
    return fu + fv - fu * fv            # reading N1
