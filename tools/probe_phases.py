"""Phase timing (clock64 per block: staging / DFT / loop / evaluate) for a config.
Needs a TF_PHASE_TIMING variant:  python -m paper_2207_00238_b200.build --variant phase TF_PHASE_TIMING
    TF_LIB=.../variants/phase.so TF_PHASE_DUMP=1 python tools/probe_phases.py 2 exact"""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2207_00238_b200 import tframe as T  # noqa: E402
from paper_2207_00238_b200.configs import workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
if cfg == 0:  # one isolated c2-sized block (32x32 window): pure per-iteration latency
    import numpy as np
    from dataclasses import replace
    wl = replace(workload(2), W=64, H=64, frames=1, tiles=1, overlap=0)
    a = np.random.default_rng(0).integers(0, 256, (64, 64), dtype=np.uint8)
    b = np.ones((64, 64), np.uint8)
    b[24:32, 24:32] = 0
    imgs, kns = [a], [b]
else:
    wl = workload(cfg, frames=4 if cfg == 5 else None)
    imgs, kns = zip(*[T.synth_frame(cfg, f, wl.W, wl.H) for f in range(wl.frames)])
img = torch.stack([torch.from_numpy(a) for a in imgs]).cuda()
kn = torch.stack([torch.from_numpy(a) for a in kns]).cuda()
out = torch.empty_like(img)
ctx = T.Context(1, [0], mode)
for _ in range(2):
    st = ctx.tiled_device(img.data_ptr(), kn.data_ptr(), out.data_ptr(), wl.W, wl.H, wl.frames, wl.tiles,
                          wl.overlap, wl.params, want_stats=True)
print(f"c{cfg} {mode}: kernel {st.kernel_ms:.3f} ms, blocks {st.blocks_processed}, iterations {st.iterations}")
