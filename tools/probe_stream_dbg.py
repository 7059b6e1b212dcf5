import ctypes as C, os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2207_00238_b200 import _native as N
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload
wl = workload(2)
img, kn = T.synth_frame(2, 0, wl.W, wl.H)
h_img = torch.from_numpy(img.reshape(-1)).pin_memory(); h_kn = torch.from_numpy(kn.reshape(-1)).pin_memory()
h_out = torch.empty_like(h_img).pin_memory()
ctx = T.Context(1, [0], "fast"); L = N.lib(); p = wl.params._c()
st = N.tf_run_stats()
for nb in sys.argv[1].split(","):
    os.environ["TF_STREAM_BANDS"] = nb
    for i in range(8):
        t = time.perf_counter()
        N.check(L.tf_tiled_extrapolate(ctx.handle, h_img.data_ptr(), h_kn.data_ptr(), wl.W, wl.H, 1, wl.tiles, wl.overlap, C.byref(p), h_out.data_ptr(), C.byref(st)))
        dt = (time.perf_counter() - t) * 1e3
    print(f"bands {nb}: wall {dt:.3f} ms plan {st.plan_us} us total {st.total_us} us kernel {st.kernel_ms:.3f} ms", flush=True)
