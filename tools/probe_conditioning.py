"""FAST vs EXACT disagreement as a function of the support window's known fraction (config
5 by default): which blocks would have to run EXACT for FAST to meet the tolerance."""
import os
import sys

sys.path.insert(0, '.')
os.environ.setdefault('TF_STREAM_BANDS', '1')
os.environ.setdefault('TF_HYBRID', '0')  # raw FAST: what the hybrid would have to fix
import numpy as np

from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = workload(cfg, frames=frames)
p = wl.params
B, m = p.block_size, p.support_margin
ex_ctx, fa_ctx = T.Context(1, [0], "exact"), T.Context(1, [0], "fast")
rows = []
tot_unk = tot_bad = 0
for f in range(frames):
    img, kn = T.synth_frame(cfg, f, wl.W, wl.H)
    ex, _ = ex_ctx.tiled(img, kn, wl.tiles, wl.overlap, p)
    fa, _ = fa_ctx.tiled(img, kn, wl.tiles, wl.overlap, p)
    d = np.abs(ex.astype(int) - fa.astype(int))
    k = (kn != 0).astype(np.int64)
    ii = np.pad(k, ((1, 0), (1, 0))).cumsum(0).cumsum(1)  # integral image (single tile: halo = frame)
    H, W = kn.shape
    for by in range(0, H, B):
        for bx in range(0, W, B):
            bw, bh = min(B, W - bx), min(B, H - by)
            blk_unk = (k[by:by + bh, bx:bx + bw] == 0)
            if not blk_unk.any():
                continue
            x0, y0, x1, y1 = max(0, bx - m), max(0, by - m), min(W, bx + bw + m), min(H, by + bh + m)
            known = ii[y1, x1] - ii[y0, x1] - ii[y1, x0] + ii[y0, x0]
            frac = known / ((x1 - x0) * (y1 - y0))
            db = d[by:by + bh, bx:bx + bw][blk_unk]
            rows.append((frac, int(blk_unk.sum()), int((db > 1).sum()), int(db.max())))
    tot_unk += int((kn == 0).sum())
    tot_bad += int((d[kn == 0] > 1).sum())
rows = np.array(rows)
print(f"c{cfg} frames={frames}: blocks {len(rows)}, unknown px {tot_unk}, |d|>1 px {tot_bad} "
      f"-> within1 {1 - tot_bad / tot_unk:.6f}")
for thr in (0.0, 0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5, 0.6):
    sel = rows[:, 0] < thr
    bad_left = tot_bad - rows[sel, 2].sum()
    print(f"  EXACT for window known fraction < {thr:.2f}: {sel.sum():6d} blocks ({sel.mean() * 100:5.1f} %), "
          f"within1 after {1 - bad_left / tot_unk:.6f}")
