"""BASELINE.json configs 1..5 as workload descriptors.

The "64x64 DFT" named for configs 1/4/5 is not expressible in the reference:
its DFT size is the clamped support window (extrapolate.hpp:119-122, 291-299),
so every config runs with DFT = window (44x44 / 32x32 / 16x16 / 44x44 / 48x48).
Config 4 uses overlap d = 16 (B-aligned, >= margin): the tiled output is then
independent of the tile count and equal to the whole-image output.
"""
from __future__ import annotations

from dataclasses import dataclass

from .tframe import FseLiteParams


@dataclass(frozen=True)
class Workload:
    config: int
    W: int
    H: int
    frames: int
    tiles: int
    overlap: int
    params: FseLiteParams
    note: str

    @property
    def name(self) -> str:
        return f"c{self.config}"

    @property
    def pixels(self) -> int:
        return self.W * self.H * self.frames

    def describe(self) -> str:
        p = self.params
        return (f"c{self.config}: {self.frames}x{self.W}x{self.H} u8, tiles={self.tiles} d={self.overlap}, "
                f"B={p.block_size} margin={p.support_margin} ({p.block_size + 2 * p.support_margin}^2 "
                f"window = DFT) I={p.model_iterations} rho={p.weight_decay} gamma={p.compensation}")


CONFIGS: dict[int, Workload] = {
    1: Workload(1, 512, 512, 1, 1, 0, FseLiteParams(16, 14, 100, 0.5, 0.8),
                "single tile, single process (CPU-runnable)"),
    2: Workload(2, 1920, 1080, 1, 4, 12, FseLiteParams(8, 12, 200, 0.5, 0.8),
                "4 tiles, overlap = border = 12"),
    3: Workload(3, 3840, 2160, 1, 8, 6, FseLiteParams(4, 6, 50, 0.5, 0.7),
                "i.i.d. pixel loss; 8 tiles, d = margin = 6"),
    4: Workload(4, 7680, 4320, 1, 8, 16, FseLiteParams(16, 14, 200, 0.5, 0.8),
                "cells + scratches; 8 tiles, d = 16 (B-aligned)"),
    5: Workload(5, 1920, 1080, 64, 1, 0, FseLiteParams(16, 16, 150, 0.5, 0.8),
                "64-frame batch, one tile per frame"),
}


def workload(config: int, frames: int | None = None, tiles: int | None = None) -> Workload:
    w = CONFIGS[config]
    return Workload(w.config, w.W, w.H, frames if frames is not None else w.frames,
                    tiles if tiles is not None else w.tiles, w.overlap, w.params, w.note)
