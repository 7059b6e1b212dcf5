"""e2e probe: the host-buffer C-ABI call (tf_tiled_extrapolate with pinned buffers; streamed row
bands on one GPU) vs torch H2D + device call + D2H, for a BASELINE config in FAST mode."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_2207_00238_b200 import _native as N
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
frames = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = workload(cfg, frames=frames)
imgs, kns = zip(*[T.synth_frame(cfg, f, wl.W, wl.H) for f in range(wl.frames)])
img = np.stack(imgs)
kn = np.stack(kns)
n = img.size
h_img = torch.from_numpy(img.reshape(-1)).pin_memory()
h_kn = torch.from_numpy(kn.reshape(-1)).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
ctx = T.Context(1, [0], mode)
L = N.lib()
p = wl.params._c()


def host_call():
    N.check(L.tf_tiled_extrapolate(ctx.handle, h_img.data_ptr(), h_kn.data_ptr(), wl.W, wl.H, wl.frames,
                                   wl.tiles, wl.overlap, C.byref(p), h_out.data_ptr(), None))


d_img = h_img.cuda()
d_kn = h_kn.cuda()
d_out = torch.empty_like(d_img)
s = torch.cuda.Stream()  # a real stream: NULL would mean the context's own stream


def torch_call():
    with torch.cuda.stream(s):
        d_img.copy_(h_img, non_blocking=True)
        d_kn.copy_(h_kn, non_blocking=True)
        N.check(L.tf_tiled_extrapolate_device(ctx.handle, 0, d_img.data_ptr(), d_kn.data_ptr(), wl.W, wl.H,
                                              wl.frames, wl.tiles, wl.overlap, C.byref(p), 0, 1,
                                              d_out.data_ptr(), s.cuda_stream, None))
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()


def timeit(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3


ref = None
for nb in ("1", "2", "4", "8", "16"):
    os.environ["TF_STREAM_BANDS"] = nb
    ctx.reload_tuning()
    ms = timeit(host_call)
    out = h_out.numpy().copy()
    ref = out if ref is None else ref
    print(f"c{cfg} {mode} frames={wl.frames} host API bands={nb:2s}: {ms:.3f} ms/call -> "
          f"{n / ms / 1e3:.1f} Mpix/s  equal={np.array_equal(out, ref)}", flush=True)
os.environ.pop("TF_STREAM_BANDS", None)
ctx.reload_tuning()
ms = timeit(torch_call)
print(f"c{cfg} {mode} torch H2D + device call + D2H: {ms:.3f} ms/call -> {n / ms / 1e3:.1f} Mpix/s "
      f"equal={np.array_equal(h_out.numpy(), ref)}", flush=True)
