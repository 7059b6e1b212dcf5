import ctypes as C, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2207_00238_b200 import _native as N
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import workload
L = N.lib()
for cfg in (2, 3):
  for mode in ("exact", "fast"):
    wl = workload(cfg)
    img, kn = T.synth_frame(cfg, 0, wl.W, wl.H)
    ctx = T.Context(1, [0], mode)
    p = wl.params._c()
    outs = []
    for nb in ("1", "1", "4"):
        os.environ["TF_STREAM_BANDS"] = nb
        o, _ = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        outs.append(o.copy())
    d_img = torch.from_numpy(img.reshape(-1)).cuda(); d_kn = torch.from_numpy(kn.reshape(-1)).cuda(); d_out = torch.empty_like(d_img)
    s = torch.cuda.current_stream()
    for rep in range(2):
        N.check(L.tf_tiled_extrapolate_device(ctx.handle, 0, d_img.data_ptr(), d_kn.data_ptr(), wl.W, wl.H, 1, wl.tiles, wl.overlap, C.byref(p), 0, 1, d_out.data_ptr(), s.cuda_stream, None))
        torch.cuda.synchronize()
        outs.append(d_out.cpu().numpy().reshape(wl.H, wl.W))
    print(cfg, mode, [int((o != outs[0]).sum()) for o in outs], flush=True)
    ctx.close()
