"""CPU: the C-ABI library loads, exports every symbol include/fmmbem_b200.h declares,
and the product path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1506_05957_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmmbem_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fmmbem_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("fmmbem_plan_create", "fmmbem_op_create", "fmmbem_op_apply", "fmmbem_op_gmres",
                 "fmmbem_op_assemble_rhs", "fmmbem_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared_functions()) == set(N.SIGNATURES)
    N.load()  # binds argtypes for every symbol


def test_no_cpu_fallback_without_device():
    if N.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    from paper_1506_05957_b200 import make_icosphere
    from paper_1506_05957_b200.operator import GpuBemOperator

    with pytest.raises(RuntimeError, match="no CUDA device"):
        GpuBemOperator(make_icosphere(1), "laplace_second", n_crit=16)


def test_argument_errors_map_to_valueerror_before_device_work():
    from paper_1506_05957_b200.operator import GpuFmmPlan

    pts = np.random.default_rng(0).uniform(-1, 1, (50, 3))
    with pytest.raises(ValueError):
        GpuFmmPlan(pts, pts, theta=1.5)
    with pytest.raises(ValueError):
        GpuFmmPlan(pts, pts, n_crit=0)
    with pytest.raises(ValueError):
        GpuFmmPlan(np.zeros((0, 3)), pts)
    with pytest.raises(NotImplementedError):
        GpuFmmPlan(pts, pts, policy="treecode")
