"""FAST vs EXACT on one config frame: differing pixels and the kernel time (tuning check)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = workload(c, frames=1)
img, kn = T.synth_frame(c, 0, wl.W, wl.H)
outs = {}
for mode in ("exact", "fast"):
    ctx = T.Context(1, [0], mode)
    best = None
    for _ in range(3):
        out, st = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        best = st if best is None or st.kernel_ms < best.kernel_ms else best
    outs[mode] = out
    print(f"c{c} {mode}: kernel {best.kernel_ms:.3f} ms, refined {best.blocks_refined}", flush=True)
    ctx.close()
print("pixels differing FAST vs EXACT:", int((outs["exact"] != outs["fast"]).sum()))
