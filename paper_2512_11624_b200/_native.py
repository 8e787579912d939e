"""ctypes binding of libgsvr_b200.so (the C ABI declared in include/gsvr_b200.h).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2512_11624_b200/csrc``).  There is no fallback: if the library or a CUDA
device is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import (InvalidParameterError, NumericalDegeneracyError,
                     TrainingDivergedError)

LIB_PATH = Path(os.environ.get("GSVR_B200_LIB")
                or Path(__file__).resolve().parent / "_lib" / "libgsvr_b200.so")

OK, ERR_INVALID, ERR_NONFINITE, ERR_DEGENERATE, ERR_CUDA = 0, 1, 2, 3, 4
F32, F64 = 0, 1

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f64 = ctypes.c_double

# name -> (restype, argtypes); every pointer is passed as void*.
_SIGNATURES = {
    "gsvr_abi_version": (_i32, []),
    "gsvr_last_error": (ctypes.c_char_p, []),
    "gsvr_last_error_index": (_i64, []),
    "gsvr_last_error_value": (_f64, []),
    "gsvr_field_covariances": (_i32, [_i64, _vp, _vp, _vp, _i32, _vp]),
    "gsvr_field_chain": (_i32, [_i64, _vp, _vp, _vp, _f64, _f64, _vp, _vp, _vp]),
    "gsvr_slice_inputs": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gsvr_slice_chain": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gsvr_render_forward": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp,
                                   _vp, _f64, _vp, _vp]),
    "gsvr_train_step_backward": (_i32, [_i64, _i64, _i64, _i64] + [_vp] * 8 + [_vp, _i32]
                                 + [_vp] * 3 + [_f64] + [_vp] * 9 + [_vp]),
    "gsvr_train_step_backward_host": (_i32, [_i64, _i64, _i64, _i64] + [_vp] * 8 + [_vp, _i32]
                                      + [_vp] * 3 + [_f64] + [_vp] * 9 + [_vp]),
    "gsvr_set_kernel_timing": (_i32, [_i32]),
    "gsvr_kernel_time_ms": (_f64, [_vp]),
    "gsvr_render_batch": (_i32, [_i64, _i64] + [_vp] * 7 + [_i32, _i64] + [_vp] * 3 + [_f64, _vp, _vp]),
    "gsvr_corrected_points": (_i32, [_i64] + [_vp] * 6),
    "gsvr_eval_field": (_i32, [_i64, _i64, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _f64, _vp,
                               _vp]),
    "gsvr_knn_build": (_i32, [_i64, _vp, _vp, _vp]),
    "gsvr_knn_free": (None, [_vp]),
    "gsvr_knn_count": (_i64, [_vp]),
    "gsvr_knn_query": (_i32, [_vp, _i64, _vp, _i64, _vp, _i32, _vp]),
    "gsvr_batch_create": (_i32, [_i64, _i64, _vp, _vp, _vp, _i32, _vp, _vp]),
    "gsvr_batch_free": (None, [_vp]),
    "gsvr_batch_tiles": (_i64, [_vp]),
    "gsvr_batch_perm": (_vp, [_vp]),
    "gsvr_batch_set_observed": (_i32, [_vp, _vp, _vp]),
    "gsvr_batch_refresh": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "gsvr_batch_knn_fallback_rows": (_i64, [_vp]),
    "gsvr_batch_invalidate_seeds": (None, [_vp]),
    "gsvr_batch_bin": (_i32, [_vp, _i64, _i64, _vp, _i32, _vp]),
    "gsvr_batch_neighbors": (_i32, [_vp, _vp, _vp]),
    "gsvr_batch_tile_gaussians": (_i64, [_vp]),
    "gsvr_batch_tile_info": (_i32, [_vp] * 8),
    "gsvr_batch_tile_geometry": (_i32, [_vp] * 5),
    "gsvr_train_tiles": (_i32, [_vp, _i64, _i64] + [_vp] * 8 + [_f64] + [_vp] * 6),
    "gsvr_batch_displacement": (_i32, [_vp] * 7),
    "gsvr_field_adamw_step": (_i32, [_i64] + [_vp] * 7 + [_f64, _f64, _vp] + [_f64] * 7
                              + [_i32, _vp, _vp, _vp, _vp, _vp]),
    "gsvr_field_workspace_bytes": (_i64, []),
    "gsvr_psf_quadrature": (_i32, [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64,
                                   _vp, _vp, _vp]),
    "gsvr_stack_slice_counts": (_i32, [_i32, _vp, _vp, _vp]),
    "gsvr_build_points": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gsvr_init_sample": (_i32, [_i32, _vp, _vp, _f64, _i64, _vp, _vp, _vp, _vp, _i32, _vp]),
    "gsvr_init_source_intensity": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "gsvr_pairwise_sum": (_i32, [_i64, _vp, _vp, _vp]),
    "gsvr_init_weights": (_i32, [_i32, _vp, _vp, _f64, _vp, _vp]),
    "gsvr_cumsum": (_i32, [_i64, _vp, _vp]),
    "gsvr_copy_d2h": (_i32, [_vp, _vp, _i64, _vp]),
    "gsvr_probe_fp32_peak": (_i32, [_vp, _vp]),
    "gsvr_batch_is_planar": (_i32, [_vp]),
    "gsvr_set_kernel_variant": (_i32, [_i32]),
    "gsvr_slice_adamw_step": (_i32, [_i64] + [_vp] * 8 + [_i32, _vp] + [_f64] * 7
                              + [_i32, _i64] + [_vp] * 7),
}

_lib = None


def lib():
    """Load the CUDA library (raises if it is absent: there is no CPU path)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(nvcc, sm_100a). There is no CPU fallback.")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return tuple(_SIGNATURES)


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception classes."""
    if rc == OK:
        return
    L = lib()
    msg = L.gsvr_last_error().decode(errors="replace")
    where = f"{what}: " if what else ""
    if rc == ERR_INVALID:
        raise InvalidParameterError(f"{where}{msg}")
    if rc == ERR_NONFINITE:
        raise TrainingDivergedError(f"{where}{msg}")
    if rc == ERR_DEGENERATE:
        raise NumericalDegeneracyError(f"{where}{msg}")
    raise RuntimeError(f"{where}CUDA failure: {msg}")


def last_index() -> int:
    return int(lib().gsvr_last_error_index())


def last_value() -> float:
    return float(lib().gsvr_last_error_value())
