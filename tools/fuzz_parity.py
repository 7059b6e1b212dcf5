"""Randomised parity sweep (not a unit test): N random cases over image shape, block size,
margin, iterations, gamma, rho, tiles, overlap, frames and mask pattern.  EXACT through the
GPU must equal the C oracle byte for byte; FAST's agreement with EXACT is aggregated.
    python tools/fuzz_parity.py [N=300] [seed=1]"""
import os
import sys

sys.path.insert(0, '.')
import numpy as np

import oracle as O
from paper_2207_00238_b200 import tframe as T

def run(n, seed, ex_ctx=None, fa_ctx=None, verbose=True):
  rng = np.random.default_rng(seed)
  ex_ctx = ex_ctx or T.Context(1, [0], "exact")
  fa_ctx = fa_ctx or T.Context(1, [0], "fast")
  bad, unk_tot, within_tot, kinds, worst = 0, 0, 0, {}, []
  for case in range(n):
      B = int(rng.choice([2, 3, 4, 5, 8, 16]))
      margin = int(rng.choice([0, 1, 2, 4, 6, 8, 12, 14, 16]))
      span = B + 2 * margin
      if span > 64:
          margin = (64 - B) // 2
      iters = int(rng.integers(1, 80))
      gamma = float(rng.uniform(0.1, 1.0))
      rho = float(rng.uniform(0.5, 0.95))
      W, H = int(rng.integers(8, 260)), int(rng.integers(8, 200))
      frames = int(rng.integers(1, 3))
      tiles = int(rng.integers(1, 7))
      overlap = int(rng.integers(0, 20))
      img = rng.integers(0, 256, (frames, H, W), dtype=np.uint8)
      yy, xx = np.mgrid[0:H, 0:W]
      img = np.clip(img // 4 + (96 + 60 * np.sin(xx / rng.uniform(3, 20)) * np.cos(yy / rng.uniform(3, 20))).astype(np.uint8), 0, 255).astype(np.uint8)
      kind = int(rng.integers(0, 4))
      if kind == 0:
          kn = (rng.random((frames, H, W)) > rng.uniform(0.05, 0.5)).astype(np.uint8)
      elif kind == 1:
          c = int(rng.choice([4, 8, 16]))
          cells = rng.random((frames, (H + c - 1) // c, (W + c - 1) // c)) > rng.uniform(0.1, 0.4)
          kn = np.repeat(np.repeat(cells, c, 1), c, 2)[:, :H, :W].astype(np.uint8)
      elif kind == 2:
          kn = np.ones((frames, H, W), np.uint8)
          for f in range(frames):
              for _ in range(int(rng.integers(1, 4))):
                  cy, cx, r = rng.integers(0, H), rng.integers(0, W), rng.integers(3, 40)
                  kn[f][(yy - cy) ** 2 + (xx - cx) ** 2 < r * r] = 0
      else:
          kn = (rng.random((frames, H, W)) > 0.97).astype(np.uint8)  # almost nothing known
      if frames == 1:
          img, kn = img[0], kn[0]
      p = T.FseLiteParams(B, margin, iters, gamma, rho)
      try:
          want, bpt = O.tiled(img, kn, tiles, overlap, B, margin, iters, gamma, rho)
      except O.OracleError:
          continue  # degenerate tiling: the GPU path must raise too
      ex, st = ex_ctx.tiled(img, kn, tiles, overlap, p)
      fa, _ = fa_ctx.tiled(img, kn, tiles, overlap, p)
      ok = np.array_equal(ex, want) and st.blocks_reference == int(bpt.sum())
      if not ok:
          bad += 1
          print(f"MISMATCH case {case}: W={W} H={H} f={frames} B={B} m={margin} I={iters} tiles={tiles} d={overlap} "
                f"kind={kind} diff={(ex != want).sum()} blocks {st.blocks_reference}/{int(bpt.sum())}", flush=True)
      u = kn == 0
      d = np.abs(ex.astype(int) - fa.astype(int))[u]
      if d.size:
          worst.append(((d <= 1).mean(), int(d.size), dict(W=W, H=H, f=frames, B=B, m=margin, I=iters,
                                                            g=round(gamma, 2), r=round(rho, 2), t=tiles,
                                                            d=overlap, kind=kind, unk=round(float(u.mean()), 2))))
      unk_tot += d.size
      within_tot += int((d <= 1).sum())
      k = kinds.setdefault(kind, [0, 0])
      k[0] += d.size
      k[1] += int((d <= 1).sum())
  if verbose:
    print(f"{n} cases: EXACT mismatches {bad}; FAST within +-1 of EXACT {within_tot / max(unk_tot, 1):.6f} "
          f"over {unk_tot} px; by mask kind " + ", ".join(f"{k}: {v[1] / max(v[0], 1):.5f}" for k, v in sorted(kinds.items())))
    worst.sort(key=lambda w: w[0])
    for w in worst[:15]:
      print(f"  within1 {w[0]:.4f} over {w[1]:6d} px: {w[2]}")
  return bad, within_tot / max(unk_tot, 1)


if __name__ == "__main__":
  run(int(sys.argv[1]) if len(sys.argv) > 1 else 300, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
