"""TEST INFRASTRUCTURE ONLY — CPU oracle bindings.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package, and only as the CHECKER (or the timed CPU
reference arm).  The product (paper_2207_00238_b200) never imports it.

Two oracles:
  * Restatement (liboracle.so, fse_oracle.c): plain-C FSE-lite + tiling with
    per-block instrumentation; always buildable (gcc), travels to the GPU box.
  * Reference (_ref/libtframe_ref.so, ref_shim.cpp): the UNMODIFIED reference
    headers compiled from /root/reference by oracle/Makefile; built here and
    shipped prebuilt to the GPU box (git-ignored, not gpurun-ignored).
Parity pin: tests/test_oracle.py checks the restatement byte-for-byte against
the reference library and against tests/golden/ fixtures the reference made.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libtframe_ref.so"


class orc_params(C.Structure):
    _fields_ = [("block", C.c_int32), ("margin", C.c_int32), ("iters", C.c_int32),
                ("gamma", C.c_double), ("rho", C.c_double)]


class orc_block_stats(C.Structure):
    _fields_ = [("bx", C.c_int32), ("by", C.c_int32), ("M", C.c_int32), ("L", C.c_int32),
                ("iters", C.c_int32), ("pairs", C.c_int32), ("touched", C.c_int32),
                ("unknown", C.c_int32), ("min_gap", C.c_double),
                ("gap_iter", C.c_int32), ("pad", C.c_int32)]


_orc = None
_ref = None


def _u8(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.uint8:
        a = (a != 0).astype(np.uint8) if a.dtype == bool else a.astype(np.uint8)
    return a


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_LIB.exists():
            raise RuntimeError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_LIB))
        L.orc_plan_proposed.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_expand.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_fse_lite.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(orc_params),
                                   C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_tiled.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.POINTER(orc_params), C.c_void_p, C.c_void_p]
        L.orc_check_params.argtypes = [C.POINTER(orc_params)]
        L.orc_diffusion.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_tiled_diffusion.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_int, C.c_void_p]
        _orc = L
    return _orc


def have_ref() -> bool:
    return REF_LIB.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(str(REF_LIB))
        L.ref_last_error.restype = C.c_char_p
        L.ref_plan_proposed.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.ref_interior_boundary.argtypes = [C.c_int, C.c_int, C.c_int]
        L.ref_interior_boundary.restype = C.c_longlong
        L.ref_expand.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.ref_fse_lite.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_double, C.c_double, C.c_void_p, C.POINTER(C.c_int64)]
        L.ref_fse_lite_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int64,
                                         C.POINTER(C.c_int64)]
        L.ref_registry.argtypes = [C.c_char_p, C.c_char_p] + [C.POINTER(C.c_int)] * 3 + \
            [C.POINTER(C.c_double)] * 2 + [C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_run_local.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_void_p,
                                    C.POINTER(C.c_int64)]
        L.ref_tiled_allcores.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_int, C.c_int, C.c_void_p]
        L.ref_tiled_allcores_part.argtypes = L.ref_tiled_allcores.argtypes[:-1] + [C.c_int, C.c_int, C.c_void_p]
        L.ref_synth_frame.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_diffusion.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.ref_run_local_diffusion.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_int, C.c_int, C.c_void_p]
        L.ref_gen_scatter_mask.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint32, C.c_void_p]
        L.ref_make_scene.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_void_p]
        L.ref_psnr.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.ref_psnr.restype = C.c_double
        L.ref_ssim.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.ref_ssim.restype = C.c_double
        L.ref_mse.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.ref_mse.restype = C.c_double
        L.ref_mse_missing.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                      C.POINTER(C.c_double)]
        _ref = L
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}")
        self.code = code


# ------------------------------------------------------------------ restatement
def plan_proposed(W, H, N):
    out = np.zeros((max(N, 1), 4), np.int32)
    rc = orc().orc_plan_proposed(W, H, N, out.ctypes.data)
    if rc:
        raise OracleError(rc)
    return out[:N]


def expand(core, d, W, H):
    c = np.asarray(core, np.int32)
    h = np.zeros(4, np.int32)
    rc = orc().orc_expand(c.ctypes.data, d, W, H, h.ctypes.data)
    if rc:
        raise OracleError(rc)
    return h


def fse_lite(img, known, block, margin, iters, gamma, rho, with_stats=False):
    """Restated fse_lite_extrapolate (extrapolate.hpp:263).  Returns out, or
    (out, stats structured array) with per-block I_b, P_b, T_b, U_b, min gap."""
    img = _u8(img)
    kn = _u8(known)
    h, w = img.shape
    out = np.empty_like(img)
    p = orc_params(block, margin, iters, gamma, rho)
    nb = C.c_int64(0)
    cap = ((w + block - 1) // block) * ((h + block - 1) // block) if with_stats else 0
    st = (orc_block_stats * max(cap, 1))()
    rc = orc().orc_fse_lite(img.ctypes.data, kn.ctypes.data, w, h, C.byref(p), out.ctypes.data,
                            C.cast(st, C.c_void_p) if with_stats else None, cap, C.byref(nb))
    if rc:
        raise OracleError(rc)
    if not with_stats:
        return out
    arr = np.ctypeslib.as_array(st)[: nb.value].copy()
    return out, arr


def tiled(img, known, tiles, overlap, block, margin, iters, gamma, rho):
    """Restated run_master: returns (out, processed blocks per (frame, tile))."""
    img = _u8(img)
    kn = _u8(known)
    if img.ndim == 2:
        frames, (H, W) = 1, img.shape
    else:
        frames, H, W = img.shape
    out = np.empty_like(img)
    bpt = np.zeros(frames * tiles, np.int64)
    p = orc_params(block, margin, iters, gamma, rho)
    rc = orc().orc_tiled(img.ctypes.data, kn.ctypes.data, W, H, frames, tiles, overlap, C.byref(p),
                         out.ctypes.data, bpt.ctypes.data)
    if rc:
        raise OracleError(rc)
    return out, bpt


# ------------------------------------------------------------------ reference
def diffusion(img, known, iters):
    """C restatement of diffusion_extrapolate (extrapolate.hpp:41-84)."""
    img, known = _u8(img), _u8(known)
    h, w = img.shape
    out = np.empty_like(img)
    rc = orc().orc_diffusion(img.ctypes.data, known.ctypes.data, w, h, iters, out.ctypes.data)
    if rc:
        raise OracleError(rc)
    return out


def tiled_diffusion(img, known, tiles, overlap, iters):
    """run_master with the diffusion extrapolator (C restatement); img (frames, H, W) or (H, W)."""
    img, known = _u8(img), _u8(known)
    frames = img.shape[0] if img.ndim == 3 else 1
    H, W = img.shape[-2:]
    out = img.copy()
    rc = orc().orc_tiled_diffusion(img.ctypes.data, known.ctypes.data, W, H, frames, tiles, overlap,
                                   iters, out.ctypes.data)
    if rc:
        raise OracleError(rc)
    return out


def ref_diffusion(img, known, iters):
    """The compiled reference's diffusion_extrapolate."""
    img, known = _u8(img), _u8(known)
    h, w = img.shape
    out = np.empty_like(img)
    rc = ref().ref_diffusion(img.ctypes.data, known.ctypes.data, w, h, iters, out.ctypes.data)
    if rc:
        raise OracleError(rc, ref_error())
    return out


def ref_run_local_diffusion(img, known, tiles, overlap, iters, workers=1):
    """The reference's run_local with algo "diffusion"."""
    img, known = _u8(img), _u8(known)
    H, W = img.shape
    out = np.empty_like(img)
    rc = ref().ref_run_local_diffusion(img.ctypes.data, known.ctypes.data, W, H, tiles, overlap, iters,
                                       workers, out.ctypes.data)
    if rc:
        raise OracleError(rc, ref_error())
    return out


def ref_error() -> str:
    return ref().ref_last_error().decode()


def ref_plan_proposed(W, H, N):
    out = np.zeros((max(N, 1), 4), np.int32)
    rc = ref().ref_plan_proposed(W, H, N, out.ctypes.data)
    if rc:
        raise OracleError(rc, ref_error())
    return out[:N]


def ref_expand(core, d, W, H):
    c = np.asarray(core, np.int32)
    h = np.zeros(4, np.int32)
    rc = ref().ref_expand(c.ctypes.data, d, W, H, h.ctypes.data)
    if rc:
        raise OracleError(rc, ref_error())
    return h


def ref_fse_lite(img, known, block, margin, iters, gamma, rho, count_blocks=False):
    img = _u8(img)
    kn = _u8(known)
    h, w = img.shape
    out = np.empty_like(img)
    nb = C.c_int64(0)
    rc = ref().ref_fse_lite(img.ctypes.data, kn.ctypes.data, w, h, block, margin, iters, gamma, rho,
                            out.ctypes.data, C.byref(nb) if count_blocks else None)
    if rc:
        raise OracleError(rc, ref_error())
    return (out, nb.value) if count_blocks else out


def ref_run_local(img, known, tiles, overlap, block, margin, iters, gamma, rho, workers):
    img = _u8(img)
    kn = _u8(known)
    H, W = img.shape
    out = np.empty_like(img)
    us = C.c_int64(0)
    rc = ref().ref_run_local(img.ctypes.data, kn.ctypes.data, W, H, tiles, overlap, block, margin,
                             iters, gamma, rho, workers, out.ctypes.data, C.byref(us))
    if rc:
        raise OracleError(rc, ref_error())
    return out, us.value


def ref_synth_frame(config, frame, W, H):
    """The versioned input generator (paper_2207_00238_b200/csrc/synth_gen.hpp) compiled into
    the reference shim: the same bytes as the product's tf_synth_frame, without loading it."""
    img = np.empty((H, W), np.uint8)
    kn = np.empty((H, W), np.uint8)
    if ref().ref_synth_frame(int(config), int(frame), int(W), int(H), img.ctypes.data, kn.ctypes.data):
        raise OracleError(1, "ref_synth_frame: bad arguments")
    return img, kn


def ref_tiled_allcores(img, known, tiles, overlap, block, margin, iters, gamma, rho,
                       threads=None, band_blocks=1, out=None, part=0, n_parts=1):
    img = _u8(img)
    kn = _u8(known)
    if img.ndim == 2:
        frames, (H, W) = 1, img.shape
    else:
        frames, H, W = img.shape
    if out is None:
        out = img.copy()
    threads = threads or os.cpu_count() or 1
    rc = ref().ref_tiled_allcores_part(img.ctypes.data, kn.ctypes.data, W, H, frames, tiles, overlap,
                                       block, margin, iters, gamma, rho, threads, band_blocks,
                                       part, n_parts, out.ctypes.data)
    if rc:
        raise OracleError(rc, ref_error())
    return out


def ref_registry(name, params=""):
    b, m, i = C.c_int(0), C.c_int(0), C.c_int(0)
    g, r = C.c_double(0), C.c_double(0)
    infl = C.c_int(0)
    buf = C.create_string_buffer(256)
    rc = ref().ref_registry(name.encode(), params.encode(), C.byref(b), C.byref(m), C.byref(i),
                            C.byref(g), C.byref(r), C.byref(infl), buf, 256)
    if rc:
        raise OracleError(rc, ref_error())
    return dict(block=b.value, margin=m.value, iters=i.value, gamma=g.value, rho=r.value,
                influence=infl.value, params_string=buf.value.decode())


def ref_gen_scatter_mask(w, h, fraction, block, seed):
    out = np.empty((h, w), np.uint8)
    rc = ref().ref_gen_scatter_mask(w, h, fraction, block, seed, out.ctypes.data)
    if rc:
        raise OracleError(rc, ref_error())
    return out


def ref_make_scene(w, h, seed):
    out = np.empty((h, w), np.uint8)
    ref().ref_make_scene(w, h, seed, out.ctypes.data)
    return out


def ref_psnr(a, b):
    a, b = _u8(a), _u8(b)
    return ref().ref_psnr(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0])


def psnr(a, b) -> float:
    """metrics.hpp:327-335 (restated; used where the reference lib is absent)."""
    d = a.astype(np.float64) - b.astype(np.float64)
    mse = float(np.mean(d * d))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(255.0 * 255.0 / mse)


def ref_interior_boundary(W, H, N) -> int:
    """tiling.hpp:231 on plan_proposed(W, H, N), via the compiled reference."""
    return int(ref().ref_interior_boundary(W, H, N))


# ---- metrics (metrics.hpp:12-88): C restatement and the compiled reference
def _orc_metrics():
    L = orc()
    if not getattr(L, "_metrics_bound", False):
        L.orc_mse.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.orc_mse.restype = C.c_double
        L.orc_mse_missing.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                      C.POINTER(C.c_double)]
        L.orc_psnr_from_mse.argtypes = [C.c_double]
        L.orc_psnr_from_mse.restype = C.c_double
        L.orc_ssim.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.orc_ssim.restype = C.c_double
        L._metrics_bound = True
    return L


def mse(a, b) -> float:
    a, b = _u8(a), _u8(b)
    return _orc_metrics().orc_mse(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0])


def mse_missing(a, b, known) -> float:
    a, b, k = _u8(a), _u8(b), _u8((np.asarray(known) != 0).astype(np.uint8))
    v = C.c_double()
    rc = _orc_metrics().orc_mse_missing(a.ctypes.data, b.ctypes.data, k.ctypes.data, a.shape[1],
                                        a.shape[0], C.byref(v))
    if rc:
        raise OracleError(rc, "mse_missing: mask has no unknown pixels")
    return v.value


def psnr_from_mse(m) -> float:
    return _orc_metrics().orc_psnr_from_mse(float(m))


def orc_psnr(a, b) -> float:
    return psnr_from_mse(mse(a, b))


def ssim(a, b) -> float:
    a, b = _u8(a), _u8(b)
    return _orc_metrics().orc_ssim(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0])


def ref_mse(a, b) -> float:
    a, b = _u8(a), _u8(b)
    return ref().ref_mse(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0])


def ref_mse_missing(a, b, known) -> float:
    a, b, k = _u8(a), _u8(b), _u8((np.asarray(known) != 0).astype(np.uint8))
    v = C.c_double()
    rc = ref().ref_mse_missing(a.ctypes.data, b.ctypes.data, k.ctypes.data, a.shape[1], a.shape[0],
                               C.byref(v))
    if rc:
        raise OracleError(rc, ref_error())
    return v.value


def ref_ssim(a, b) -> float:
    a, b = _u8(a), _u8(b)
    return ref().ref_ssim(a.ctypes.data, b.ctypes.data, a.shape[1], a.shape[0])
