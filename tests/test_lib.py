"""The C-ABI library loads here (no GPU) and exports exactly what include/sem1d.h declares."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1806_01422_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sem1d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sem[13]d_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes binding"
    assert set(_lib.SIGNATURES) == set(names)


def test_library_identity(lib):
    assert lib.sem1d_version() == 1
    assert lib.sem1d_max_degree() == 32


def test_plan_validation_without_gpu(lib):
    """Plans are host objects: argument checking works without a device."""
    n = 8
    K = np.zeros((n, n)); Dw = np.zeros((n, n)); pat = np.ones(n + 1)
    h = ctypes.c_void_p()
    assert lib.sem1d_plan_create(16, 7, 1, 0.01, K.ctypes.data, Dw.ctypes.data, pat.ctypes.data,
                                 pat.ctypes.data, 1, ctypes.byref(h)) == 0
    assert lib.sem1d_plan_ndof(h) == 16 * 7
    assert lib.sem1d_terminal_work_size(h) >= 1
    assert lib.sem1d_plan_destroy(h) == 0
    for args in [(16, 0, 1, 0.01), (16, 33, 1, 0.01), (0, 7, 1, 0.01), (1, 1, 1, 0.01),
                 (16, 7, 1, -1.0)]:
        rc = lib.sem1d_plan_create(*args, K.ctypes.data, Dw.ctypes.data, pat.ctypes.data,
                                   pat.ctypes.data, 1, ctypes.byref(h))
        assert rc == -1 and _lib.last_error()
    # Dirichlet plans have E*N + 1 nodes
    assert lib.sem1d_plan_create(5, 3, 0, 0.1, K.ctypes.data, Dw.ctypes.data, pat.ctypes.data,
                                 pat.ctypes.data, 2, ctypes.byref(h)) == 0
    assert lib.sem1d_plan_ndof(h) == 16
    lib.sem1d_plan_destroy(h)
    # compute entry points reject NULL plans before touching the device
    assert lib.sem1d_rhs(None, None, None, None, None) == -1


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1806_01422_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\".*?\"\"\"", "", txt, flags=re.S), f


def test_integration_binding_is_the_documented_one():
    """INTEGRATION.md reproduces integration/semopt_b200.py verbatim (the executed drop-in,
    tests/test_gpu_dropin.py), so the document cannot drift from the tested binding."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = open(os.path.join(root, "integration", "semopt_b200.py")).read()
    doc = open(os.path.join(root, "INTEGRATION.md")).read()
    assert code.strip() in doc
