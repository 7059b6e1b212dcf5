"""Quick timing probe: FSE kernel time for a BASELINE config through the C-ABI."""
import sys, time
sys.path.insert(0, '.')
import os
os.environ.setdefault('TF_STREAM_BANDS', '1')  # one-shot host path: kernel_ms = the FSE launch itself
import numpy as np
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import CONFIGS

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
wl = CONFIGS[cfg]
imgs, kns = zip(*[T.synth_frame(cfg, f, wl.W, wl.H) for f in range(wl.frames)])
img = np.stack(imgs) if wl.frames > 1 else imgs[0]
kn = np.stack(kns) if wl.frames > 1 else kns[0]
ctx = T.Context(1, [0], mode)
for rep in range(3):
    t = time.perf_counter()
    out, st = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    dt = time.perf_counter() - t
    print(f"c{cfg} {mode}: wall {dt*1e3:.2f} ms kernel {st.kernel_ms:.3f} ms blocks ref {st.blocks_reference} gpu {st.blocks_processed}"
          f" -> {wl.pixels/st.kernel_ms/1e3:.1f} Mpix/s kernel-only", flush=True)
