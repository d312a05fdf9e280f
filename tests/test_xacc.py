"""The exact cross-block combine (fixed-point limbs) against the
definition of an exactly rounded sum: math.fsum (correctly rounded exact sum)."""
import ctypes
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def xsum():
    from paper_2509_14211_b200 import nbg
    f = nbg.lib.nbg_debug_xacc_sum
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_void_p, ctypes.c_longlong]

    def run(v):
        v = np.ascontiguousarray(v, np.float64)
        return f(v.ctypes.data, v.shape[0])
    return run


@pytest.mark.parametrize("seed", range(8))
def test_exact_sum_matches_fsum(xsum, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 5000))
    mant = rng.standard_normal(n)
    exps = rng.integers(-60, 60, n)
    v = np.ldexp(mant, exps)
    assert xsum(v) == math.fsum(v)


def test_exact_sum_cancellation_and_order(xsum):
    v = np.array([1e30, 1.0, -1e30, 2.0 ** -100, 3.0])
    assert xsum(v) == math.fsum(v) == 4.0 + 2.0 ** -100
    rng = np.random.default_rng(1)
    w = rng.random(1000) * 1e-3
    assert xsum(w) == xsum(w[::-1]) == xsum(rng.permutation(w)) == math.fsum(w)


def test_exact_sum_ties_to_even(xsum):
    # 1 + 2^-53 is a tie: rounds to even (1.0); adding a tiny sticky bit rounds up
    assert xsum(np.array([1.0, 2.0 ** -53])) == 1.0
    assert xsum(np.array([1.0, 2.0 ** -53, 2.0 ** -120])) == 1.0 + 2.0 ** -52
    assert xsum(np.array([1.0 + 2.0 ** -52, 2.0 ** -53])) == 1.0 + 2.0 ** -51


def test_exact_sum_specials(xsum):
    assert xsum(np.array([])) == 0.0
    assert math.isinf(xsum(np.array([1.0, np.inf])))
    assert math.isnan(xsum(np.array([np.inf, -np.inf])))
    assert math.isnan(xsum(np.array([1.0, np.nan])))
