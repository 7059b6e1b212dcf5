"""Per-iteration latency of blocks in isolation (1 block) and at 1 / 4 blocks per SM:
FSE kernel time difference between I=300 and I=100 on 8x8 holes (32x32 windows)."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2207_00238_b200 import tframe as T  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
ctx = T.Context(1, [0], mode)
rng = np.random.default_rng(0)
for nblk in (1, 148, 592):
    side = int(np.ceil(np.sqrt(nblk)))
    W = H = 40 * side
    img = rng.integers(0, 256, (H, W), dtype=np.uint8)
    kn = np.ones((H, W), np.uint8)
    cnt = 0
    for by in range(side):
        for bx in range(side):
            if cnt < nblk:
                kn[by * 40 + 16:by * 40 + 24, bx * 40 + 16:bx * 40 + 24] = 0
                cnt += 1
    res = {}
    for I in (100, 300):
        p = T.FseLiteParams(8, 12, I, 0.5, 0.8)
        best = 1e9
        for _ in range(3):
            _, st = ctx.tiled(img, kn, 1, 0, p)
            best = min(best, st.kernel_ms)
        res[I] = best
    per_it = (res[300] - res[100]) / 200 * 1e3
    print(f"{mode} blocks={nblk}: I=100 {res[100]:.3f} ms, I=300 {res[300]:.3f} ms -> {per_it:.3f} us/iteration "
          f"({per_it * 1.965e3:.0f} cycles @1.965GHz)", flush=True)
