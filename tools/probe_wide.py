"""FAST wide kernel (windows 40..64) vs the CTA kernel (TF_NO_WIDE=1): kernel time and parity
against EXACT on full BASELINE frames (configs 1, 4, 5)."""
import os, sys
sys.path.insert(0, '.')
import os
os.environ.setdefault('TF_STREAM_BANDS', '1')  # one-shot host path: kernel_ms = the FSE launch itself
import numpy as np
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload
import oracle as O

cfgs = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 4, 5]
ex_ctx = T.Context(1, [0], "exact")
fa_ctx = T.Context(1, [0], "fast")
for c in cfgs:
    wl = workload(c, frames=4 if c == 5 else None)
    imgs, kns = zip(*[T.synth_frame(c, f, wl.W, wl.H) for f in range(wl.frames)])
    img = np.stack(imgs) if wl.frames > 1 else imgs[0]
    kn = np.stack(kns) if wl.frames > 1 else kns[0]
    ex, st_e = ex_ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    res = {}
    for tag, env in (("cta", {"TF_NO_WIDE": "1"}), ("wm0", {"TF_WIDE_WM": "0"}), ("wm1", {"TF_WIDE_WM": "1"}), ("wm2", {"TF_WIDE_WM": "2"})):
        for k in ("TF_NO_WIDE", "TF_WIDE_WM"):
            os.environ.pop(k, None)
        os.environ.update(env)
        best = None
        for rep in range(3):
            fa, st = fa_ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
            best = st if best is None or st.kernel_ms < best.kernel_ms else best
        unk = kn == 0
        d = np.abs(ex.astype(int) - fa.astype(int))[unk]
        pe = np.mean([O.psnr(i, e) for i, e in zip(np.reshape(img, (-1,) + img.shape[-2:]), np.reshape(ex, (-1,) + ex.shape[-2:]))])
        pf = np.mean([O.psnr(i, e) for i, e in zip(np.reshape(img, (-1,) + img.shape[-2:]), np.reshape(fa, (-1,) + fa.shape[-2:]))])
        print(f"c{c} {tag:4s}: frames={wl.frames} kernel {best.kernel_ms:8.3f} ms (exact {st_e.kernel_ms:8.3f}) blocks {best.blocks_processed}"
              f" within1 {np.mean(d <= 1):.6f} n(d>0) {(d > 0).sum()} max {d.max()} dPSNR {abs(pe - pf):.5f}"
              f" known_kept {np.array_equal(fa[~unk], img[~unk])}", flush=True)
