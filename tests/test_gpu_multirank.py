"""GPU tests of the one-process-per-GPU path on one device, and of the scratch-ordering fixes.

* tf_comm_init(nranks = 1) + tf_tiled_extrapolate_device + tf_comm_gather_cores repeated
  (the rank loop of INTEGRATION.md §4; the device path's graph is captured on call 2 and
  replayed afterwards) reproduce the one-shot output every time.
* tf_tiled_extrapolate_rank (host buffers: halo H2D, FSE, core gather, root D2H) equals
  tf_tiled_extrapolate, with and without a communicator.
* LPT ownership (tf_core_layout) composes: every part run on its own buffer and the cores
  assembled by owner equal the single-part run (runtime.hpp:102-130).
* Device calls on different streams back to back (shared per-GPU scratch) stay correct.
* The streamed host path with concurrent bands on the big-window kernel (per-band scratch
  slots sized from a band-independent bound) equals the one-shot path and the oracle.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2207_00238_b200 import _native as N
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import CONFIGS, workload

pytestmark = pytest.mark.gpu


def _comm_ctx(mode):
    ctx = T.Context(1, [0], mode)
    uid = (C.c_uint8 * 128)()
    N.check(N.lib().tf_comm_unique_id(uid))
    N.check(N.lib().tf_comm_init(ctx.handle, 1, 0, uid))
    return ctx


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_one_rank_nccl_device_call_and_gather_repeated(mode):
    import torch
    wl = CONFIGS[2]
    W, H, F = 480, 270, 2
    imgs, kns = zip(*[T.synth_frame(2, f, W, H) for f in range(F)])
    img_np, kn_np = np.stack(imgs), np.stack(kns)
    one = T.Context(1, [0], mode)
    want, _ = one.tiled(img_np, kn_np, wl.tiles, wl.overlap, wl.params)
    one.close()
    ctx = _comm_ctx(mode)
    try:
        img = torch.from_numpy(img_np).cuda()
        kn = torch.from_numpy(kn_np).cuda()
        out = torch.zeros_like(img)
        p = wl.params._c()
        s = torch.cuda.current_stream().cuda_stream
        for it in range(5):
            out.zero_()
            N.check(N.lib().tf_tiled_extrapolate_device(ctx.handle, 0, img.data_ptr(), kn.data_ptr(), W, H, F,
                                                        wl.tiles, wl.overlap, C.byref(p), 0, 1,
                                                        out.data_ptr(), s, None))
            N.check(N.lib().tf_comm_gather_cores(ctx.handle, out.data_ptr(), W, H, F, wl.tiles, 0, s))
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            assert np.array_equal(got, want), f"call {it}: {(got != want).sum()} px differ"
        # the host-buffer rank call through the same communicator
        res = np.zeros_like(img_np)
        io = (C.c_int64 * 2)()
        N.check(N.lib().tf_tiled_extrapolate_rank(ctx.handle, img_np.ctypes.data, kn_np.ctypes.data, W, H, F,
                                                  wl.tiles, wl.overlap, C.byref(p), 0, res.ctypes.data, io))
        assert np.array_equal(res, want)
        assert io[1] == img_np.size and io[0] >= 2 * img_np.size  # halos cover the frame (+ aprons)
    finally:
        ctx.close()


@pytest.mark.parametrize("cfg", [2, 3])
def test_rank_call_without_comm_equals_host_call(cfg):
    wl = workload(cfg)
    W, H = (960, 540)
    img, kn = T.synth_frame(cfg, 0, W, H)
    ctx = T.Context(1, [0], "exact")
    try:
        want, _ = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        out = np.zeros_like(img)
        p = wl.params._c()
        for _ in range(2):
            N.check(N.lib().tf_tiled_extrapolate_rank(ctx.handle, img.ctypes.data, kn.ctypes.data, W, H, 1,
                                                      wl.tiles, wl.overlap, C.byref(p), 0, out.ctypes.data, None))
            assert np.array_equal(out, want)
        q = wl.params
        ref = O.tiled(img, kn, wl.tiles, wl.overlap, q.block_size, q.support_margin, q.model_iterations,
                      q.compensation, q.weight_decay)[0]
        assert np.array_equal(want, ref)
    finally:
        ctx.close()


@pytest.mark.parametrize("n_parts", [2, 3, 5])
def test_lpt_parts_on_separate_buffers_assemble_the_frame(n_parts):
    """Each part computed into its own buffer (as on its own GPU), cores taken by owner."""
    import torch
    wl = CONFIGS[3]
    W, H, F, tiles = 700, 410, 2, 7  # unequal core areas: LPT differs from round robin
    imgs, kns = zip(*[T.synth_frame(3, f, W, H) for f in range(F)])
    img_np, kn_np = np.stack(imgs), np.stack(kns)
    ctx = T.Context(1, [0], "exact")
    try:
        want, _ = ctx.tiled(img_np, kn_np, tiles, wl.overlap, wl.params)
        n = F * tiles
        cores = (N.tf_rect * n)()
        fr = np.zeros(n, np.int32)
        own = np.zeros(n, np.int32)
        N.check(N.lib().tf_core_layout(W, H, F, tiles, n_parts, cores, fr.ctypes.data, own.ctypes.data,
                                       None, None))
        assert len(set(own.tolist())) == min(n_parts, n)
        img = torch.from_numpy(img_np).cuda()
        kn = torch.from_numpy(kn_np).cuda()
        got = np.zeros_like(img_np)
        for part in range(n_parts):
            out = torch.zeros_like(img)
            st = ctx.tiled_device(img.data_ptr(), kn.data_ptr(), out.data_ptr(), W, H, F, tiles, wl.overlap,
                                  wl.params, part=part, n_parts=n_parts, want_stats=True)
            o = out.cpu().numpy()
            for t in np.where(own == part)[0]:
                c = cores[t]
                got[fr[t], c.y:c.y + c.h, c.x:c.x + c.w] = o[fr[t], c.y:c.y + c.h, c.x:c.x + c.w]
            assert st.blocks_processed <= st.blocks_reference
        assert np.array_equal(got, want)
    finally:
        ctx.close()


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_device_calls_on_two_streams_back_to_back(mode):
    """Per-GPU scratch is shared by all calls: a call on stream s2 right after a long call
    on s1 (no host sync between) must wait for it (work-done event)."""
    import torch
    ctx = T.Context(1, [0], mode)
    try:
        a_img, a_kn = T.synth_frame(3, 0, 1920, 1080)
        b_img, b_kn = T.synth_frame(2, 0, 640, 360)
        wa, wb = CONFIGS[3], CONFIGS[2]
        want_a, _ = ctx.tiled(a_img, a_kn, wa.tiles, wa.overlap, wa.params)
        want_b, _ = ctx.tiled(b_img, b_kn, wb.tiles, wb.overlap, wb.params)
        dai, dak = torch.from_numpy(a_img).cuda(), torch.from_numpy(a_kn).cuda()
        dbi, dbk = torch.from_numpy(b_img).cuda(), torch.from_numpy(b_kn).cuda()
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        for _ in range(3):
            oa, ob = torch.zeros_like(dai), torch.zeros_like(dbi)
            torch.cuda.synchronize()
            ctx.tiled_device(dai.data_ptr(), dak.data_ptr(), oa.data_ptr(), 1920, 1080, 1, wa.tiles, wa.overlap,
                             wa.params, stream=s1.cuda_stream)
            ctx.tiled_device(dbi.data_ptr(), dbk.data_ptr(), ob.data_ptr(), 640, 360, 1, wb.tiles, wb.overlap,
                             wb.params, stream=s2.cuda_stream)
            torch.cuda.synchronize()
            assert np.array_equal(oa.cpu().numpy(), want_a)
            assert np.array_equal(ob.cpu().numpy(), want_b)
    finally:
        ctx.close()


def test_streamed_bands_on_the_big_window_kernel(tune_env):
    """640x1080, B = 64, margin = 64 (192x192 windows, big-window kernel) in 2 concurrent
    bands with different candidate counts: byte-identical to one shot and to the oracle."""
    W, H, B, m, I = 640, 1080, 64, 64, 6
    img, _ = T.synth_frame(1, 7, W, H)
    kn = np.ones((H, W), np.uint8)
    rng = np.random.default_rng(3)
    for (x, y) in rng.integers(0, [W - 8, H - 8], size=(60, 2)):
        kn[y:y + 6, x:x + 6] = 0
    kn[:400, :] = 1
    kn[100:104, 100:104] = 0  # band 0: few candidates, band 1: many
    p = T.FseLiteParams(B, m, I, 0.5, 0.8)
    want = O.fse_lite(img, kn, B, m, I, 0.5, 0.8)
    for mode in ("exact", "fast"):
        ctx = T.Context(1, [0], mode)
        try:
            tune_env([ctx], TF_STREAM_BANDS=1)
            one, _ = ctx.tiled(img, kn, 1, 0, p)
            tune_env([ctx], TF_STREAM_BANDS=2)
            for _ in range(3):
                got, _ = ctx.tiled(img, kn, 1, 0, p)
                assert np.array_equal(got, one), f"{mode}: {(got != one).sum()} px differ"
            assert np.array_equal(one, want)
        finally:
            ctx.close()
