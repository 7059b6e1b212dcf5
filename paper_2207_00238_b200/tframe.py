"""Host-side mirror of the reference's extrapolator and tiling interface.

Same names, argument meaning and error behaviour as tframe (the reference,
/root/reference/proj/include/tframe), backed by the sm_100a C-ABI library:

    reference                                   here
    ------------------------------------------  ---------------------------------
    Rect, TileLayout (tiling.hpp:16-54)          Rect, TileLayout
    plan_proposed / plan (tiling.hpp:99,301)     plan_proposed / plan
    interior_boundary (tiling.hpp:231)           interior_boundary
    ExpandedTile, expand (overlap.hpp:16-34)     ExpandedTile, expand
    FseLiteParams (extrapolate.hpp:86)           FseLiteParams
    check_fse_params (extrapolate.hpp:102)       check_fse_params
    Extrapolator (extrapolate.hpp:22-36)         Extrapolator
    FseLiteExtrapolator (extrapolate.hpp:390)    FseLiteExtrapolator (GPU)
    fse_lite_extrapolate (extrapolate.hpp:263)   fse_lite_extrapolate (GPU)
    registry_lookup (extrapolate.hpp:418)        registry_lookup
    MasterConfig, RunStats (runtime.hpp:25-41)   MasterConfig, RunStats
    run_master / run_local (runtime.hpp:75,142)  run_master / run_local (GPUs)

Images are numpy uint8 arrays of shape (H, W) (or (F, H, W) for batches);
masks have the same shape, nonzero = known (image.hpp:53 PixelMask).
std::invalid_argument maps to ValueError, TilingError to TilingError.
"""
from __future__ import annotations

import ctypes as C
import threading
from abc import ABC, abstractmethod
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import TilingError, check, lib

__all__ = [
    "Rect", "TileLayout", "ExpandedTile", "plan_proposed", "plan", "interior_boundary", "expand",
    "FseLiteParams", "check_fse_params", "Extrapolator", "FseLiteExtrapolator",
    "fse_lite_extrapolate", "registry_lookup", "MasterConfig", "RunStats", "run_master",
    "run_local", "Context", "count_blocks", "synth_frame", "TilingError",
]


# ---------------------------------------------------------------- tiling
@dataclass(frozen=True)
class Rect:
    x: int = 0
    y: int = 0
    w: int = 0
    h: int = 0

    def area(self) -> int:
        return self.w * self.h

    def contains(self, px: int, py: int) -> bool:
        return self.x <= px < self.x + self.w and self.y <= py < self.y + self.h

    def _c(self) -> N.tf_rect:
        return N.tf_rect(self.x, self.y, self.w, self.h)


@dataclass
class TileLayout:
    image_w: int
    image_h: int
    tiles: list[Rect]
    strategy: str = "proposed"
    n: int = 0


def plan_proposed(W: int, H: int, N_: int) -> TileLayout:
    """tiling.hpp:99-111: rows of compact, nearly equal tiles (paper Alg. 1)."""
    n = max(int(N_), 0)
    arr = (N.tf_rect * max(n, 1))()
    check(lib().tf_plan_proposed(int(W), int(H), int(N_), arr))
    return TileLayout(W, H, [Rect(r.x, r.y, r.w, r.h) for r in arr[:n]], "proposed", n)


def plan(strategy: str, W: int, H: int, N_: int) -> TileLayout:
    """tiling.hpp:301-308.  Only the proposed strategy is on the hot path; the
    vertical/optimal planners are paper baselines (out of scope)."""
    if strategy != "proposed":
        raise NotImplementedError(f"strategy '{strategy}' is not part of the B200 hot path")
    return plan_proposed(W, H, N_)


def interior_boundary(layout: TileLayout) -> int:
    """tiling.hpp:231-250."""
    arr = (N.tf_rect * max(len(layout.tiles), 1))(*[t._c() for t in layout.tiles])
    return int(lib().tf_interior_boundary(arr, len(layout.tiles)))


@dataclass(frozen=True)
class ExpandedTile:
    core: Rect
    halo: Rect
    d: int = 0

    def overhead_pixels(self) -> int:
        return self.halo.area() - self.core.area()


def expand(tile: Rect, d: int, image_w: int, image_h: int) -> ExpandedTile:
    """overlap.hpp:25-34: core grown by d on each side, clamped to the image."""
    core = tile._c()
    halo = N.tf_rect()
    check(lib().tf_expand(C.byref(core), int(d), int(image_w), int(image_h), C.byref(halo)))
    return ExpandedTile(tile, Rect(halo.x, halo.y, halo.w, halo.h), int(d))


# ---------------------------------------------------------------- parameters
@dataclass
class FseLiteParams:
    """extrapolate.hpp:86-92."""
    block_size: int = 4
    support_margin: int = 8
    model_iterations: int = 100
    compensation: float = 0.5  # gamma
    weight_decay: float = 0.8  # rho

    def _c(self) -> N.tf_fse_params:
        return N.tf_fse_params(int(self.block_size), int(self.support_margin),
                               int(self.model_iterations), float(self.compensation),
                               float(self.weight_decay))


def check_fse_params(p: FseLiteParams) -> None:
    """extrapolate.hpp:102-110; raises ValueError (std::invalid_argument)."""
    c = p._c()
    check(lib().tf_check_fse_params(C.byref(c)))


def _params_from_string(s: str) -> FseLiteParams:
    c = N.tf_fse_params()
    check(lib().tf_fse_params_from_string(s.encode(), C.byref(c)))
    return FseLiteParams(c.block, c.margin, c.iters, c.gamma, c.rho)


# ---------------------------------------------------------------- context
class Context:
    """Owns a tf_ctx: per-GPU streams, device buffers, NCCL communicators."""

    def __init__(self, n_gpus: int = 1, device_ids: list[int] | None = None, mode: str = "exact"):
        ids = (C.c_int * n_gpus)(*device_ids) if device_ids else None
        h = lib().tf_create(int(n_gpus), ids)
        if not h:
            raise N.TframeError(N.TF_ECUDA, N.last_error())
        self._h = h
        self.n_gpus = n_gpus
        self.set_mode(mode)

    @property
    def handle(self) -> int:
        return self._h

    def set_mode(self, mode: str) -> None:
        m = {"exact": N.TF_MODE_EXACT, "fast": N.TF_MODE_FAST}[mode]
        check(lib().tf_set_mode(self._h, m))
        self.mode = mode

    def reload_tuning(self) -> None:
        """Re-read the TF_* tuning environment (read once per context, include/tframe_fse.h)."""
        check(lib().tf_set_mode(self._h, {"exact": N.TF_MODE_EXACT, "fast": N.TF_MODE_FAST}[self.mode]))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().tf_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    # -- host-buffer path (Extrapolator / run_master equivalents)
    def tiled(self, image: np.ndarray, mask: np.ndarray, tiles: int, overlap: int,
              params: FseLiteParams, out: np.ndarray | None = None) -> tuple[np.ndarray, "RunStats"]:
        img = np.ascontiguousarray(image, dtype=np.uint8)
        kn = np.ascontiguousarray(mask)
        if kn.dtype != np.uint8:
            kn = (kn != 0).astype(np.uint8)
        if img.shape != kn.shape:
            raise ValueError("run_master: image/mask dimension mismatch")
        if img.ndim == 2:
            frames, (H, W) = 1, img.shape
        elif img.ndim == 3:
            frames, H, W = img.shape
        else:
            raise ValueError("image must be (H, W) or (F, H, W)")
        if out is None:
            out = np.empty_like(img)
        st = N.tf_run_stats()
        p = params._c()
        check(lib().tf_tiled_extrapolate(self._h, img.ctypes.data, kn.ctypes.data, W, H, frames,
                                         int(tiles), int(overlap), C.byref(p), out.ctypes.data,
                                         C.byref(st)))
        return out, RunStats._from_c(st)

    def tiled_diffusion(self, image: np.ndarray, mask: np.ndarray, tiles: int, overlap: int,
                        iters: int) -> tuple[np.ndarray, "RunStats"]:
        """run_master with algo "diffusion" (runtime.hpp:75-139)."""
        img = np.ascontiguousarray(image, dtype=np.uint8)
        kn = np.ascontiguousarray(mask)
        if kn.dtype != np.uint8:
            kn = (kn != 0).astype(np.uint8)
        if img.shape != kn.shape:
            raise ValueError("run_master: image/mask dimension mismatch")
        frames, H, W = (1, *img.shape) if img.ndim == 2 else img.shape
        out = np.empty_like(img)
        st = N.tf_run_stats()
        check(lib().tf_tiled_diffusion(self._h, img.ctypes.data, kn.ctypes.data, W, H, frames,
                                       int(tiles), int(overlap), int(iters), out.ctypes.data,
                                       C.byref(st)))
        return out, RunStats._from_c(st)

    # -- quality metrics (metrics.hpp:12-90) on the GPU
    def quality(self, a: np.ndarray, b: np.ndarray, mask: np.ndarray | None = None,
                ssim: bool = True) -> list[dict]:
        """Per frame of (H, W) or (F, H, W) u8 images: mse, psnr, mse_missing,
        psnr_missing, ssim, n_missing (tf_quality in include/tframe_fse.h)."""
        A = np.ascontiguousarray(a, dtype=np.uint8)
        B = np.ascontiguousarray(b, dtype=np.uint8)
        if A.shape != B.shape:
            raise ValueError("mse: dimension mismatch")
        frames, H, W = (1, *A.shape) if A.ndim == 2 else A.shape
        kn = None
        if mask is not None:
            kn = np.ascontiguousarray(mask)
            if kn.dtype != np.uint8:
                kn = (kn != 0).astype(np.uint8)
            if kn.shape != A.shape:
                raise ValueError("mse_missing: dimension mismatch")
        out = (N.tf_quality_metrics * frames)()
        check(lib().tf_quality(self._h, A.ctypes.data, B.ctypes.data,
                               kn.ctypes.data if kn is not None else None, W, H, frames,
                               int(bool(ssim)), out))
        return [{f: getattr(q, f) for f, _ in N.tf_quality_metrics._fields_} for q in out]

    def quality_device(self, d_a: int, d_b: int, d_known: int | None, W: int, H: int,
                       frames: int = 1, ssim: bool = True, stream: int = 0, gpu: int = 0) -> list[dict]:
        out = (N.tf_quality_metrics * frames)()
        check(lib().tf_quality_device(self._h, gpu, d_a, d_b, d_known or None, W, H, frames,
                                      int(bool(ssim)), stream or None, out))
        return [{f: getattr(q, f) for f, _ in N.tf_quality_metrics._fields_} for q in out]

    # -- device path (inputs already in HBM; torch tensors or raw pointers)
    def tiled_device(self, d_img: int, d_known: int, d_out: int, W: int, H: int, frames: int,
                     tiles: int, overlap: int, params: FseLiteParams, stream: int = 0,
                     part: int = 0, n_parts: int = 1, gpu: int = 0,
                     want_stats: bool = False) -> "RunStats | None":
        p = params._c()
        st = N.tf_run_stats() if want_stats else None
        check(lib().tf_tiled_extrapolate_device(
            self._h, gpu, d_img, d_known, W, H, frames, tiles, overlap, C.byref(p), part, n_parts,
            d_out, stream or None, C.byref(st) if st is not None else None))
        return RunStats._from_c(st) if st is not None else None


_default_ctx: dict[tuple, Context] = {}
_ctx_lock = threading.Lock()


def default_context(device: int = 0, mode: str = "exact") -> Context:
    key = (device, mode)
    with _ctx_lock:
        if key not in _default_ctx:
            _default_ctx[key] = Context(1, [device], mode)
        return _default_ctx[key]


# ---------------------------------------------------------------- metrics (metrics.hpp)
def _single(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    A = np.ascontiguousarray(a, dtype=np.uint8)
    B = np.ascontiguousarray(b, dtype=np.uint8)
    if A.ndim != 2 or A.shape != B.shape:
        raise ValueError("dimension mismatch")
    return A, B


def mse(a: np.ndarray, b: np.ndarray, device: int = 0) -> float:
    """metrics.hpp:12-24 on the GPU (bit-identical)."""
    A, B = _single(a, b)
    v = C.c_double()
    check(lib().tf_mse(default_context(device).handle, A.ctypes.data, B.ctypes.data, A.shape[1],
                       A.shape[0], C.byref(v)))
    return v.value


def mse_missing(a: np.ndarray, b: np.ndarray, mask: np.ndarray, device: int = 0) -> float:
    """metrics.hpp:27-45: MSE over the pixels the mask marks unknown (ValueError if none)."""
    A, B = _single(a, b)
    kn = np.ascontiguousarray((np.asarray(mask) != 0).astype(np.uint8))
    if kn.shape != A.shape:
        raise ValueError("mse_missing: dimension mismatch")
    v = C.c_double()
    check(lib().tf_mse_missing(default_context(device).handle, A.ctypes.data, B.ctypes.data,
                               kn.ctypes.data, A.shape[1], A.shape[0], C.byref(v)))
    return v.value


def psnr_from_mse(mse_value: float) -> float:
    return lib().tf_psnr_from_mse(float(mse_value))


def psnr(a: np.ndarray, b: np.ndarray, device: int = 0) -> float:
    """metrics.hpp:52-55 on the GPU (bit-identical); +inf for identical images."""
    A, B = _single(a, b)
    v = C.c_double()
    check(lib().tf_psnr(default_context(device).handle, A.ctypes.data, B.ctypes.data, A.shape[1],
                        A.shape[0], C.byref(v)))
    return v.value


def ssim(a: np.ndarray, b: np.ndarray, device: int = 0) -> float:
    """metrics.hpp:58-88 on the GPU (window values bit-identical, mean within 1e-12 rel.)."""
    A, B = _single(a, b)
    v = C.c_double()
    check(lib().tf_ssim(default_context(device).handle, A.ctypes.data, B.ctypes.data, A.shape[1],
                        A.shape[0], C.byref(v)))
    return v.value


# ---------------------------------------------------------------- extrapolators
class Extrapolator(ABC):
    """extrapolate.hpp:20-36: preserve known pixels exactly, assign every
    unknown pixel, be deterministic; output dims equal input dims."""

    @abstractmethod
    def name(self) -> str: ...

    @abstractmethod
    def influence_radius(self) -> int | None: ...

    @abstractmethod
    def extrapolate(self, image: np.ndarray, mask: np.ndarray) -> np.ndarray: ...

    @abstractmethod
    def params_string(self) -> str: ...


class FseLiteExtrapolator(Extrapolator):
    """extrapolate.hpp:390-414, computed on a B200."""

    def __init__(self, params: FseLiteParams | None = None, device: int = 0, mode: str = "exact"):
        self._params = params or FseLiteParams()
        check_fse_params(self._params)
        self._device = device
        self._mode = mode

    def name(self) -> str:
        return "fse-lite"

    def influence_radius(self) -> int:
        return self._params.block_size + self._params.support_margin

    def params(self) -> FseLiteParams:
        return self._params

    def params_string(self) -> str:
        c = self._params._c()
        buf = C.create_string_buffer(256)
        check(lib().tf_fse_params_to_string(C.byref(c), buf, 256))
        return buf.value.decode()

    def extrapolate(self, image: np.ndarray, mask: np.ndarray) -> np.ndarray:
        img = np.asarray(image)
        if img.ndim != 2:
            raise ValueError("extrapolate expects one (H, W) image")
        if np.asarray(mask).shape != img.shape:
            raise ValueError("fse_lite_extrapolate: image/mask dimension mismatch")
        out, _ = default_context(self._device, self._mode).tiled(img, mask, 1, 0, self._params)
        return out


class DiffusionExtrapolator(Extrapolator):
    """extrapolate.hpp:371-386 (diffusion_extrapolate, :41-84), computed on a B200:
    byte-identical to the reference."""

    def __init__(self, iterations: int = 32, device: int = 0):
        if iterations < 1:
            raise ValueError("diffusion_extrapolate: iterations must be >= 1")
        self._iters = int(iterations)
        self._device = device

    def name(self) -> str:
        return "diffusion"

    def influence_radius(self) -> int:
        return self._iters

    def params_string(self) -> str:
        return f"iters={self._iters}"

    def extrapolate(self, image: np.ndarray, mask: np.ndarray) -> np.ndarray:
        img = np.ascontiguousarray(image, dtype=np.uint8)
        kn = np.ascontiguousarray(mask)
        if kn.dtype != np.uint8:
            kn = (kn != 0).astype(np.uint8)
        if img.ndim != 2:
            raise ValueError("extrapolate expects one (H, W) image")
        if kn.shape != img.shape:
            raise ValueError("diffusion_extrapolate: image/mask dimension mismatch")
        out = np.empty_like(img)
        ctx = default_context(self._device)
        check(lib().tf_diffusion_extrapolate(ctx.handle, img.ctypes.data, kn.ctypes.data, img.shape[1],
                                             img.shape[0], self._iters, out.ctypes.data))
        return out


def _parse_params(s: str) -> dict:
    """detail::parse_params (extrapolate.hpp:344-356)."""
    out = {}
    for item in s.split(","):
        if not item:
            continue
        if "=" not in item:
            raise ValueError(f"bad parameter item '{item}', expected key=value")
        k, v = item.split("=", 1)
        out[k] = v
    return out


def _stoi(v: str) -> int:
    """std::stoi: optional whitespace and sign, then digits; trailing text ignored."""
    import re
    m = re.match(r"\s*([+-]?\d+)", v)
    if not m:
        raise ValueError("stoi")
    x = int(m.group(1))
    if not -2**31 <= x < 2**31:
        raise OverflowError("stoi")
    return x


def fse_lite_extrapolate(image: np.ndarray, mask: np.ndarray,
                         params: FseLiteParams | None = None, mode: str = "exact",
                         device: int = 0) -> np.ndarray:
    """extrapolate.hpp:263 on the GPU."""
    return FseLiteExtrapolator(params, device, mode).extrapolate(image, mask)


def registry_lookup(name: str, params: str = "", device: int = 0, mode: str = "exact") -> Extrapolator:
    """extrapolate.hpp:418-437: "fse-lite" (the hot path) and "diffusion" (§8(f)2)."""
    if name == "fse-lite":
        return FseLiteExtrapolator(_params_from_string(params), device, mode)
    if name == "diffusion":
        kv = _parse_params(params)
        return DiffusionExtrapolator(_stoi(kv["iters"]) if "iters" in kv else 32, device)
    raise ValueError(f"unknown algorithm '{name}', available: diffusion, fse-lite")


# ---------------------------------------------------------------- master
@dataclass
class MasterConfig:
    """runtime.hpp:35-41."""
    tiles: int = 1
    overlap: int = 32
    strategy: str = "proposed"
    algo: str = "fse-lite"
    algo_params: str = ""


@dataclass
class RunStats:
    """runtime.hpp:25-33 plus the device counters of tf_run_stats."""
    plan_us: int = 0
    distribute_us: int = 0
    compute_span_us: int = 0
    merge_us: int = 0
    total_us: int = 0
    overhead_pixels: int = 0
    blocks_reference: int = 0
    blocks_processed: int = 0
    kernel_ms: float = 0.0
    flops: float = 0.0
    iterations: int = 0
    pixels_evaluated: int = 0
    flops_executed: float = 0.0
    blocks_refined: int = 0
    tiles: list = field(default_factory=list)

    @classmethod
    def _from_c(cls, s: N.tf_run_stats) -> "RunStats":
        return cls(s.plan_us, s.distribute_us, s.compute_span_us, s.merge_us, s.total_us,
                   s.overhead_pixels, s.blocks_reference, s.blocks_processed, s.kernel_ms,
                   s.flops, s.iterations, s.pixels_evaluated, s.flops_executed, s.blocks_refined)


def run_master(image: np.ndarray, mask: np.ndarray, config: MasterConfig,
               context: Context | None = None) -> tuple[np.ndarray, RunStats]:
    """runtime.hpp:75-139 on the context's GPUs: plan -> expand -> FSE per halo
    -> crop -> merge.  The output is independent of the GPU count."""
    algo = registry_lookup(config.algo, config.algo_params)  # raises for unknown names
    if config.strategy != "proposed":
        raise NotImplementedError(f"strategy '{config.strategy}' is not part of the B200 hot path")
    ctx = context or default_context()
    if isinstance(algo, DiffusionExtrapolator):
        return ctx.tiled_diffusion(image, mask, config.tiles, config.overlap, algo.influence_radius())
    return ctx.tiled(image, mask, config.tiles, config.overlap, algo.params())


def run_local(image: np.ndarray, mask: np.ndarray, config: MasterConfig,
              n_gpus: int = 1) -> tuple[np.ndarray, RunStats]:
    """runtime.hpp:142-155: a full tiled job on an in-process pool (here: GPUs)."""
    ctx = Context(n_gpus)
    try:
        return run_master(image, mask, config, ctx)
    finally:
        ctx.close()


# ---------------------------------------------------------------- helpers
def count_blocks(mask: np.ndarray, block: int) -> int:
    """Blocks fse_lite_extrapolate processes (extrapolate.hpp:278-289)."""
    kn = np.ascontiguousarray(mask)
    if kn.dtype != np.uint8:
        kn = (kn != 0).astype(np.uint8)
    h, w = kn.shape
    return int(lib().tf_count_blocks(kn.ctypes.data, w, h, int(block)))


def synth_frame(config: int, frame: int, W: int, H: int) -> tuple[np.ndarray, np.ndarray]:
    """Versioned synthetic (image, known-mask) for BASELINE config 1..5."""
    img = np.empty((H, W), np.uint8)
    kn = np.empty((H, W), np.uint8)
    check(lib().tf_synth_frame(int(config), int(frame), int(W), int(H), img.ctypes.data,
                               kn.ctypes.data))
    return img, kn
