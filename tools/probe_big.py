import sys, os, time
sys.path.insert(0, '.')
os.environ['TF_VERBOSE'] = '1'
import numpy as np
import oracle as O
from paper_2207_00238_b200 import tframe as T
for mode in ("exact", "fast"):
    c = T.Context(1, [0], mode)
    for (B, m, I, W, H) in [(8, 12, 12000, 48, 40), (32, 32, 25, 160, 128), (64, 64, 100, 640, 480)]:
        img, kn = T.synth_frame(1, 3, W, H)
        t = time.time(); got, st = c.tiled(img, kn, 1, 0, T.FseLiteParams(B, m, I, 0.5, 0.8)); dt = time.time() - t
        print(mode, B, m, I, W, H, "blocks", st.blocks_processed, "kernel_ms", round(st.kernel_ms, 2), "wall", round(dt, 2), flush=True)
