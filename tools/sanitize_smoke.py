"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck):
EXACT + FAST on crops of configs 1-5 (half, pair, wide, GEN, CTA, warp kernels), the
streamed host path (row bands), the device path, diffusion and the quality metrics."""
import os
import sys

sys.path.insert(0, '.')
import numpy as np

from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload

crops = {1: (128, 96), 2: (200, 150), 3: (160, 120), 4: (240, 200), 5: (256, 160)}
for mode in ("exact", "fast"):
    ctx = T.Context(1, [0], mode)
    for c, (W, H) in crops.items():
        wl = workload(c, frames=2 if c == 5 else 1)
        imgs, kns = zip(*[T.synth_frame(c, f, W, H) for f in range(wl.frames)])
        img = np.stack(imgs) if wl.frames > 1 else imgs[0]
        kn = np.stack(kns) if wl.frames > 1 else kns[0]
        for nb in ("1", "3"):
            os.environ["TF_STREAM_BANDS"] = nb
            ctx.reload_tuning()
            out, st = ctx.tiled(img, kn, min(wl.tiles, 4), wl.overlap, wl.params)
            print(f"{mode} c{c} bands={nb}: blocks {st.blocks_processed}", flush=True)
    # small symmetric windows with cell losses: argmax ties -> the FAST near-tie guard and
    # its EXACT refinement launch run
    rng = np.random.default_rng(5)
    for trial in range(4):
        cells = rng.random((20, 30)) > 0.3
        kn = np.repeat(np.repeat(cells, 2, 0), 2, 1).astype(np.uint8)
        img = rng.integers(0, 256, kn.shape, dtype=np.uint8)
        out, st = ctx.tiled(img, kn, 2, 4, T.FseLiteParams(2, 2, 30, 0.5, 0.7))
        print(f"{mode} tie case {trial}: blocks {st.blocks_processed} refined {st.blocks_refined}", flush=True)
    if mode == "fast":
        a, k = T.synth_frame(2, 0, 100, 80)
        q = ctx.quality(np.stack([a, a]), np.stack([out[0] if out.ndim == 3 else a, a]), None)
        d, _ = ctx.tiled_diffusion(a, k, 2, 4, 10)
        print("metrics + diffusion ok", flush=True)
    ctx.close()
