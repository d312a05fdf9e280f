"""User-defined operators: definition and NVRTC validation run on the CPU
(no GPU needed); tests/test_gpu_userops.py checks their values, fusion and the persistent cache."""
import pytest


@pytest.fixture(scope="module")
def nbg():
    from paper_2509_14211_b200 import nbg as m
    return m


def test_define_returns_distinct_codes(nbg):
    a = nbg.nbg_unop_define("sq_plus", "x * x + c0")
    b = nbg.nbg_binop_define("scaled_absdiff", "nbg_abs(x - y) * c0")
    c = nbg.nbg_unop_define("sq_plus_again", "x * x + c0")
    assert a >= 1000 and b >= 1000 and len({a, b, c}) == 3


@pytest.mark.parametrize("expr", ["x +* 2", "undefined_fn(x)", "x; asm(\"trap;\")", "(x", "x) + (y", "}"])
def test_invalid_unop_expressions_are_rejected(nbg, expr):
    with pytest.raises(nbg.NbgError) as e:
        nbg.nbg_unop_define("bad", expr)
    assert e.value.status == nbg.INVALID_VALUE


def test_unop_cannot_use_y(nbg):
    with pytest.raises(nbg.NbgError):
        nbg.nbg_unop_define("bad", "x + y")
    assert nbg.nbg_binop_define("ok", "x + y") >= 1000


def test_undefined_code_is_rejected_at_call_time(nbg):
    import ctypes
    # an op descriptor with an unregistered user code fails validation before any device work
    assert nbg.lib.nbg_apply(None, None, 3, nbg.nbg_unop(999999, 0, 0), None) == nbg.NULL_POINTER
