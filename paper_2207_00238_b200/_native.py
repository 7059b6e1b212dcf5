"""ctypes binding of the C-ABI in include/tframe_fse.h (libtframe_b200.so).

The library is the product: there is no Python or CPU fallback.  Loading
fails loudly when the in-tree build is missing.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# TF_LIB selects a tuning variant built by `build.py --variant` (default: the product library)
LIB_PATH = Path(os.environ.get("TF_LIB") or Path(__file__).resolve().parent / "_lib" / "libtframe_b200.so")
HEADER = Path(__file__).resolve().parent.parent / "include" / "tframe_fse.h"

TF_OK, TF_EINVAL, TF_EIO, TF_EPROTO, TF_ETILING, TF_ECUDA, TF_ENCCL, TF_ENOMEM, TF_EUNSUPPORTED = range(9)
TF_MODE_EXACT, TF_MODE_FAST = 0, 1


class tf_rect(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("w", C.c_int32), ("h", C.c_int32)]


class tf_fse_params(C.Structure):
    _fields_ = [("block", C.c_int32), ("margin", C.c_int32), ("iters", C.c_int32),
                ("gamma", C.c_double), ("rho", C.c_double)]


class tf_run_stats(C.Structure):
    _fields_ = [("plan_us", C.c_int64), ("distribute_us", C.c_int64),
                ("compute_span_us", C.c_int64), ("merge_us", C.c_int64),
                ("total_us", C.c_int64), ("overhead_pixels", C.c_int64),
                ("blocks_reference", C.c_int64), ("blocks_processed", C.c_int64),
                ("kernel_ms", C.c_double), ("flops", C.c_double),
                ("iterations", C.c_int64), ("pixels_evaluated", C.c_int64),
                ("flops_executed", C.c_double), ("blocks_refined", C.c_int64)]


class tf_quality_metrics(C.Structure):
    _fields_ = [("mse", C.c_double), ("psnr", C.c_double), ("mse_missing", C.c_double),
                ("psnr_missing", C.c_double), ("ssim", C.c_double), ("n_missing", C.c_int64)]


_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p
_i = C.c_int

# name -> (restype, argtypes); must cover every function declared in the header
SIGNATURES = {
    "tf_abi_version": (_i, []),
    "tf_create": (_vp, [_i, C.POINTER(C.c_int)]),
    "tf_destroy": (None, [_vp]),
    "tf_last_error": (C.c_char_p, [_vp]),
    "tf_set_mode": (_i, [_vp, _i]),
    "tf_get_mode": (_i, [_vp]),
    "tf_device_count": (_i, [C.POINTER(C.c_int)]),
    "tf_check_fse_params": (_i, [C.POINTER(tf_fse_params)]),
    "tf_fse_params_from_string": (_i, [C.c_char_p, C.POINTER(tf_fse_params)]),
    "tf_fse_params_to_string": (_i, [C.POINTER(tf_fse_params), C.c_char_p, _i]),
    "tf_influence_radius": (_i, [C.POINTER(tf_fse_params)]),
    "tf_plan_proposed": (_i, [_i, _i, _i, C.POINTER(tf_rect)]),
    "tf_expand": (_i, [C.POINTER(tf_rect), _i, _i, _i, C.POINTER(tf_rect)]),
    "tf_interior_boundary": (C.c_longlong, [C.POINTER(tf_rect), _i]),
    "tf_count_blocks": (C.c_int64, [_vp, _i, _i, _i]),
    "tf_fse_extrapolate": (_i, [_vp, _vp, _vp, _i, _i, C.POINTER(tf_fse_params), _vp]),
    "tf_tiled_extrapolate": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, C.POINTER(tf_fse_params),
                                  _vp, C.POINTER(tf_run_stats)]),
    "tf_tiled_extrapolate_device": (_i, [_vp, _i, _vp, _vp, _i, _i, _i, _i, _i,
                                         C.POINTER(tf_fse_params), _i, _i, _vp, _vp,
                                         C.POINTER(tf_run_stats)]),
    "tf_diffusion_extrapolate": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp]),
    "tf_tiled_diffusion": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp, C.POINTER(tf_run_stats)]),
    "tf_fse_kernel_times": (_i, [_vp, _i, C.POINTER(C.c_float), _i]),
    "tf_calibrate": (_i, [_i, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "tf_calibrate_peaks": (_i, [_i, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "tf_kernel_launches": (_i, [_vp, _i, C.POINTER(C.c_int64)]),
    "tf_tiled_extrapolate_rank": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, C.POINTER(tf_fse_params), _i,
                                       _vp, _vp]),
    "tf_selftest_div": (_i, [_i, C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]),
    "tf_comm_unique_id": (_i, [_vp]),
    "tf_comm_init": (_i, [_vp, _i, _i, _vp]),
    "tf_comm_gather": (_i, [_vp, _vp, _vp, C.c_int64, _i, _vp]),
    "tf_comm_gather_cores": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp]),
    "tf_core_layout": (_i, [_i, _i, _i, _i, _i, C.POINTER(tf_rect), _vp, _vp, _vp, _vp]),
    "tf_synth_frame": (_i, [_i, _i, _i, _i, _vp, _vp]),
    "tf_quality_device": (_i, [_vp, _i, _vp, _vp, _vp, _i, _i, _i, _i, _vp, C.POINTER(tf_quality_metrics)]),
    "tf_quality": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, C.POINTER(tf_quality_metrics)]),
    "tf_mse": (_i, [_vp, _vp, _vp, _i, _i, C.POINTER(C.c_double)]),
    "tf_mse_missing": (_i, [_vp, _vp, _vp, _vp, _i, _i, C.POINTER(C.c_double)]),
    "tf_psnr": (_i, [_vp, _vp, _vp, _i, _i, C.POINTER(C.c_double)]),
    "tf_ssim": (_i, [_vp, _vp, _vp, _i, _i, C.POINTER(C.c_double)]),
    "tf_psnr_from_mse": (C.c_double, [C.c_double]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2207_00238_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().tf_last_error(None)
    return msg.decode() if msg else ""


class TframeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[tf status {code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != TF_OK:
        msg = last_error()
        if rc == TF_EINVAL:
            raise ValueError(msg)  # std::invalid_argument
        if rc == TF_ETILING:
            raise TilingError(msg)
        raise TframeError(rc, msg)


class TilingError(RuntimeError):
    """Mirrors tframe::TilingError (error.hpp:11-14): degenerate tiling."""
