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


def test_terms_outside_the_exact_window(xsum):
    """Terms of magnitude >= 2^128 or < 2^-160 are outside the exact window: they are summed in
    fp64 (arrival order) and added to the window's correctly rounded value -- no NaN, no loss."""
    big = np.array([1e40, 2e40, -1e40, 3.0])
    assert abs(xsum(big) - math.fsum(big)) <= 4 * np.spacing(2e40)
    assert xsum(np.array([1e300, 1e300])) == 2e300
    tiny = np.full(7, 1e-60)
    assert abs(xsum(tiny) - 7e-60) <= 8 * np.spacing(7e-60)
    # a term straddling 2^-160 keeps its bits above the edge (error < 2^-160)
    assert abs(xsum(np.array([2.0 ** -120, 1.0])) - (1.0 + 2.0 ** -120)) <= 2.0 ** -52
    assert math.isinf(xsum(np.array([1e308, 1e308])))
