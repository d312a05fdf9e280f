import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


_JIT_DIR = None


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
    # One persistent kernel cache (csrc/jit.cpp, keyed by a hash of the generated
    # source) for the whole session, in a fresh directory: most tests open their own context and
    # would otherwise recompile the same generated kernels with NVRTC.  The cubins are the ones
    # NVRTC produced earlier in this very session; nothing outlives it.
    global _JIT_DIR
    if not os.environ.get("NBG_JIT_CACHE"):
        import tempfile
        _JIT_DIR = tempfile.mkdtemp(prefix="nbg_jit_tests_")
        os.environ["NBG_JIT_CACHE"] = _JIT_DIR


def pytest_unconfigure(config):
    global _JIT_DIR
    if _JIT_DIR:
        import shutil
        shutil.rmtree(_JIT_DIR, ignore_errors=True)
        os.environ.pop("NBG_JIT_CACHE", None)
        _JIT_DIR = None


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
