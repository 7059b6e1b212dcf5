"""Timing probe over BASELINE configs: FSE kernel ms and Mpixel/s through the C-ABI."""
import sys, time
sys.path.insert(0, '.')
import os
os.environ.setdefault('TF_STREAM_BANDS', '1')  # one-shot host path: kernel_ms = the FSE launch itself
import numpy as np
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload

mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
cfgs = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 5]
c5_frames = int(sys.argv[3]) if len(sys.argv) > 3 else 16  # config 5 is a 64-frame batch
ctx = T.Context(1, [0], mode)
for c in cfgs:
    wl = workload(c, frames=c5_frames if c == 5 else None)
    imgs, kns = zip(*[T.synth_frame(c, f, wl.W, wl.H) for f in range(wl.frames)])
    img = np.stack(imgs) if wl.frames > 1 else imgs[0]
    kn = np.stack(kns) if wl.frames > 1 else kns[0]
    best = None
    for rep in range(3):
        out, st = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        best = st if best is None or st.kernel_ms < best.kernel_ms else best
    print(f"c{c} {mode}: frames={wl.frames} kernel {best.kernel_ms:8.3f} ms blocks {best.blocks_processed:7d}"
          f" -> {wl.pixels/best.kernel_ms/1e3:9.1f} Mpix/s kernel-only, refined {best.blocks_refined}", flush=True)
