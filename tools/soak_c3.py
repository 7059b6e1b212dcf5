"""Parity soak on the headline config: FAST vs EXACT on full c3 frames 1..8 of the generator
(differing pixels and refined blocks per frame)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload
wl = workload(3, frames=1)
ex, fa = T.Context(1, [0], "exact"), T.Context(1, [0], "fast")
tot = 0
for f in range(1, 9):
    img, kn = T.synth_frame(3, f, wl.W, wl.H)
    a, _ = ex.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    b, st = fa.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    d = int((a != b).sum()); tot += d
    print(f"c3 frame {f}: differing pixels {d}, refined {st.blocks_refined}", flush=True)
print("total differing", tot)
