"""Diffusion extrapolator timing: full frames, K sweeps, tiled like config 2 (kernel ms)."""
import sys
import time
sys.path.insert(0, '.')
from paper_2207_00238_b200 import tframe as T
import oracle as O

ctx = T.Context(1, [0])
for (W, H, tiles, d, k) in ((1920, 1080, 1, 0, 32), (1920, 1080, 4, 32, 32), (3840, 2160, 8, 64, 64)):
    img, kn = T.synth_frame(2, 0, W, H)
    best = None
    for _ in range(3):
        out, st = ctx.tiled_diffusion(img, kn, tiles, d, k)
        best = st if best is None or st.kernel_ms < best.kernel_ms else best
    t0 = time.time()
    ref = O.tiled_diffusion(img, kn, tiles, d, k)
    cpu = time.time() - t0
    print(f"{W}x{H} tiles={tiles} d={d} K={k}: kernel {best.kernel_ms:.3f} ms "
          f"({W * H / best.kernel_ms / 1e3:.0f} Mpix/s), total {best.total_us / 1e3:.2f} ms; "
          f"C oracle 1 thread {cpu * 1e3:.0f} ms; equal {bool((out == ref).all())}", flush=True)
