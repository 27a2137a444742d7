"""ctypes binding of ``libfmmbem_b200.so`` (declared in ``include/fmmbem_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()``.  There is
no CPU fallback: if the library is missing or no CUDA device is visible, the
first call raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_NAME = "libfmmbem_b200.so"
# FMMBEM_LIB: an alternative build of the same library (A/B kernel experiments, tools/)
LIB_PATH = os.environ.get("FMMBEM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)
_c_int32_p = ctypes.POINTER(ctypes.c_int32)
_c_uint8_p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p

# name: (restype, argtypes)
SIGNATURES = {
    "fmmbem_last_error": (ctypes.c_char_p, []),
    "fmmbem_version": (ctypes.c_int, []),
    "fmmbem_device_count": (ctypes.c_int, [_c_int32_p]),
    "fmmbem_fp64_peak": (ctypes.c_int, [ctypes.c_int, _c_double_p]),
    "fmmbem_plan_create": (ctypes.c_int, [_c_double_p, ctypes.c_int64, _c_double_p, ctypes.c_int64,
                                          ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(_vp)]),
    "fmmbem_plan_destroy": (ctypes.c_int, [_vp]),
    "fmmbem_plan_sizes": (ctypes.c_int, [_vp, _c_int64_p]),
    "fmmbem_plan_tree": (ctypes.c_int, [_vp, ctypes.c_int, _c_int64_p, _c_double_p, _c_double_p,
                                        _c_int32_p, _c_int32_p, _c_int64_p, _c_int64_p, _c_uint8_p]),
    "fmmbem_plan_pairs": (ctypes.c_int, [_vp, ctypes.c_int, _c_int32_p]),
    "fmmbem_plan_evaluate": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            _c_double_p, _c_double_p]),
    "fmmbem_expansion_p2m": (ctypes.c_int, [_c_double_p, ctypes.c_int64, _c_double_p, _c_double_p,
                                            ctypes.c_int, ctypes.c_int, _c_double_p, ctypes.c_int]),
    "fmmbem_expansion_translate": (ctypes.c_int, [ctypes.c_int, _c_double_p, ctypes.c_int,
                                                  ctypes.c_int, _c_double_p, _c_double_p,
                                                  ctypes.c_int]),
    "fmmbem_expansion_evaluate": (ctypes.c_int, [ctypes.c_int, _c_double_p, ctypes.c_int,
                                                 ctypes.c_int, _c_double_p, ctypes.c_int64,
                                                 ctypes.c_int, _c_double_p, _c_double_p,
                                                 ctypes.c_int]),
    "fmmbem_op_create": (ctypes.c_int, [_c_double_p, ctypes.c_int64, _c_double_p, _c_double_p,
                                        _c_double_p, _c_double_p, _c_double_p, _c_double_p,
                                        _c_double_p, _c_double_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(_vp)]),
    "fmmbem_op_destroy": (ctypes.c_int, [_vp]),
    "fmmbem_op_size": (ctypes.c_int, [_vp, _c_int64_p]),
    "fmmbem_op_plan": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "fmmbem_op_apply": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int]),
    "fmmbem_op_apply_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, _vp]),
    "fmmbem_op_dense_apply": (ctypes.c_int, [_vp, _c_double_p, _c_double_p]),
    "fmmbem_op_assemble_rhs": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_int, ctypes.c_int,
                                              _c_double_p]),
    "fmmbem_op_correction": (ctypes.c_int, [_vp, ctypes.c_int, _c_int64_p, _c_int32_p, _c_int64_p,
                                            _c_int64_p, _c_double_p]),
    "fmmbem_op_gmres": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _c_double_p, _c_double_p, _c_int32_p, _c_int32_p,
                                       _c_int32_p, _vp, _vp]),
    "fmmbem_op_gmres_device": (ctypes.c_int, [_vp, _vp, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, _vp, _c_double_p, _c_int32_p,
                                              _c_int32_p, _c_int32_p, _vp, _vp, _vp]),
    "fmmbem_op_set_timing": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int]),
    "fmmbem_op_set_serial": (ctypes.c_int, [_vp, ctypes.c_int]),
    "fmmbem_op_stage_times": (ctypes.c_int, [_vp, _c_double_p, _c_int64_p, ctypes.c_int]),
    "fmmbem_op_counters": (ctypes.c_int, [_vp, _c_int64_p, _c_int64_p, _c_double_p]),
    "fmmbem_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "fmmbem_op_leaf_work": (ctypes.c_int, [_vp, ctypes.c_int, _c_double_p]),
    "fmmbem_op_shard": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _c_int32_p, _c_int32_p,
                                       ctypes.c_char_p]),
    "fmmbem_op_unshard": (ctypes.c_int, [_vp]),
    "fmmbem_op_shard_host": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _c_int32_p, _c_int32_p,
                                            _vp, _vp, _vp]),
}

# int (*)(int32_t k, double residual, int32_t p, void* user)  (fmmbem_gmres_callback)
GMRES_CALLBACK = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
                                  ctypes.c_void_p)

# int (*)(const double* send, double* recv, int64_t count, void* user)  (fmmbem_allgather_fn)
ALLGATHER_CALLBACK = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_void_p)
# int (*)(double* buf, int64_t count, void* user)  (fmmbem_allreduce_fn)
ALLREDUCE_CALLBACK = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                      ctypes.c_void_p)

_lib = None


def load():
    """Load the library once and bind every declared symbol (raises if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_NAME} is not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; "
                "g.build()'` - there is no CPU fallback for this path")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().fmmbem_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_c_double_p)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_int64_p)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_int32_p)


def u8ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_uint8_p)


def f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and out.shape != shape:
        raise ValueError(f"expected shape {shape}, got {out.shape}")
    return out


def host_array(n: int) -> np.ndarray:
    """A new float64 host array for a result the device writes: page-locked (torch's caching
    host allocator: no first-touch page faults, the D2H copy lands in it directly) when a
    CUDA torch is importable, else plain numpy."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    except Exception:
        pass
    return np.empty(n)


def device_count() -> int:
    n = ctypes.c_int32(0)
    check(load().fmmbem_device_count(ctypes.byref(n)))
    return int(n.value)


def fp64_peak_tflops(device: int = 0) -> float:
    v = ctypes.c_double(0.0)
    check(load().fmmbem_fp64_peak(device, ctypes.byref(v)))
    return float(v.value)
