"""FAST vs EXACT agreement on full config frames: within-1 fraction, max |d|, dPSNR."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import CONFIGS
import oracle as O

cfgs = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 3]
ex_ctx, fa_ctx = T.Context(1, [0], "exact"), T.Context(1, [0], "fast")
for c in cfgs:
    wl = CONFIGS[c]
    img, kn = T.synth_frame(c, 0, wl.W, wl.H)
    ex, _ = ex_ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    fa, _ = fa_ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    unk = kn == 0
    d = np.abs(ex.astype(int) - fa.astype(int))[unk]
    print(f"c{c}: unknown {d.size} differ {(d > 0).sum()} within1 {(d <= 1).mean():.6f} max {d.max()} "
          f"dPSNR {abs(O.psnr(img, ex) - O.psnr(img, fa)):.5f} dB", flush=True)
