"""GPU parity: the sm_100a FSE path (through the C-ABI) against the CPU oracle.

EXACT mode must be byte-identical to the oracle (which is itself pinned
byte-for-byte to the compiled reference, tests/test_oracle.py).  FAST mode
must meet the north-star tolerance: >= 99.9% of reconstructed (unknown)
pixels within +-1 and |dPSNR vs truth| <= 0.05 dB.
"""
import numpy as np
import pytest

import oracle as O
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu

FAST_WITHIN1 = 0.999   # fraction of unknown pixels within +-1 (north star)
FAST_DPSNR_DB = 0.05   # |PSNR(fast, truth) - PSNR(exact, truth)| bound (north star)


@pytest.fixture(scope="module")
def ctx():
    c = T.Context(1, [0], "exact")
    yield c
    c.close()


@pytest.fixture(scope="module")
def fctx():
    c = T.Context(1, [0], "fast")
    yield c
    c.close()


def _params(b, m, i, g, r):
    return T.FseLiteParams(b, m, i, g, r)


def test_random_small_cases_exact(ctx):
    rng = np.random.default_rng(1234)
    for trial in range(40):
        w, h = int(rng.integers(6, 90)), int(rng.integers(6, 90))
        B, m, I = int(rng.integers(2, 17)), int(rng.integers(0, 20)), int(rng.integers(1, 80))
        g, r = float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.2, 0.95))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        kn = (rng.random((h, w)) > rng.uniform(0.05, 0.7)).astype(np.uint8)
        want = O.fse_lite(img, kn, B, m, I, g, r)
        got, st = ctx.tiled(img, kn, 1, 0, _params(B, m, I, g, r))
        assert np.array_equal(got, want), f"trial {trial}: {w}x{h} B={B} m={m} I={I}: {(got != want).sum()} px differ"
        assert st.blocks_reference == T.count_blocks(kn, B)


def test_all_known_identity(ctx):
    img = np.random.default_rng(2).integers(0, 256, (16, 16), dtype=np.uint8)
    out, st = ctx.tiled(img, np.ones_like(img), 1, 0, T.FseLiteParams())
    assert np.array_equal(out, img)
    assert st.blocks_processed == 0


def test_all_unknown_window_gives_128(ctx):
    img = np.full((40, 40), 77, np.uint8)
    kn = np.ones_like(img)
    kn[:, :] = 0  # no known pixel anywhere -> 128 (extrapolate.hpp:320-333)
    out, _ = ctx.tiled(img, kn, 1, 0, T.FseLiteParams(4, 2, 10, 0.5, 0.8))
    assert (out == 128).all()
    want = O.fse_lite(img, kn, 4, 2, 10, 0.5, 0.8)
    assert np.array_equal(out, want)


def test_constant_image_holes(ctx):
    # test_extrapolate.cpp:86-92 (KAT): constant 183 scene, scattered holes
    img = np.full((24, 24), 183, np.uint8)
    rng = np.random.default_rng(5)
    kn = (rng.random((24, 24)) > 0.25).astype(np.uint8)
    out, _ = ctx.tiled(img, kn, 1, 0, T.FseLiteParams())
    assert (out == 183).all()


@pytest.mark.parametrize("cfg,W,H,frames,tiles", [
    (1, 512, 512, 1, 1),
    (2, 480, 270, 1, 4),
    (3, 400, 224, 1, 8),
    (4, 512, 288, 1, 8),
    (5, 384, 216, 2, 1),
])
def test_config_params_exact_vs_oracle(ctx, cfg, W, H, frames, tiles):
    wl = CONFIGS[cfg]
    p = wl.params
    imgs, kns = [], []
    for f in range(frames):
        a, b = T.synth_frame(cfg, f, W, H)
        imgs.append(a)
        kns.append(b)
    img = np.stack(imgs) if frames > 1 else imgs[0]
    kn = np.stack(kns) if frames > 1 else kns[0]
    want, bpt = O.tiled(img, kn, tiles, wl.overlap, p.block_size, p.support_margin,
                        p.model_iterations, p.compensation, p.weight_decay)
    got, st = ctx.tiled(img, kn, tiles, wl.overlap, p)
    diff = int((got != want).sum())
    assert diff == 0, f"c{cfg}: {diff} pixels differ"
    assert st.blocks_reference == int(bpt.sum())  # block enumeration bit-exact


def test_fast_mode_within_tolerance(ctx, fctx):
    for cfg in (1, 2, 4, 5):
        wl = CONFIGS[cfg]
        W, H = (512, 512) if cfg == 1 else (480, 270)
        img, kn = T.synth_frame(cfg, 0, W, H)
        ex, _ = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        fa, _ = fctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        unk = kn == 0
        d = np.abs(ex.astype(int) - fa.astype(int))[unk]
        assert (d <= 1).mean() >= FAST_WITHIN1
        assert abs(O.psnr(img, ex) - O.psnr(img, fa)) <= FAST_DPSNR_DB
        assert np.array_equal(ex[~unk], img[~unk])


@pytest.mark.parametrize("no_gen", [False, True])
def test_fast_mode_border_windows(ctx, fctx, no_gen, tune_env):
    """Small, odd-sized frames: most windows are clamped by the halo (M, L not powers of two),
    which the FAST path runs through the GEN half-spectrum warp kernel, or (TF_NO_GEN=1)
    through the half-spectrum CTA kernel."""
    if no_gen:
        tune_env([fctx], TF_NO_GEN=1)
    ds = []
    for cfg in (2, 3):
        wl = CONFIGS[cfg]
        for (W, H), tiles in (((37, 29), 1), ((61, 44), 2), ((100, 57), 3), ((45, 90), 4)):
            img, kn = T.synth_frame(cfg, 3, W, H)
            ex, st_e = ctx.tiled(img, kn, tiles, wl.overlap, wl.params)
            fa, st_f = fctx.tiled(img, kn, tiles, wl.overlap, wl.params)
            unk = kn == 0
            ds.append(np.abs(ex.astype(int) - fa.astype(int))[unk])
            assert np.array_equal(fa[~unk], img[~unk])
            assert st_e.blocks_processed == st_f.blocks_processed
    d = np.concatenate(ds)
    assert d.size > 1000
    assert (d <= 1).mean() >= FAST_WITHIN1, f"max|d|={d.max()} n(|d|>1)={(d > 1).sum()} of {d.size}"


def test_hoisted_reciprocal_division_is_exact():
    import ctypes as C
    from paper_2207_00238_b200 import _native as N
    bad = C.c_int64(-1)
    N.check(N.lib().tf_selftest_div(0, 1 << 24, 12345, C.byref(bad)))
    assert bad.value == 0


# Config 5's clustered losses (disks of radius 32-128 px) leave 48x48 windows with almost no
# known pixel, where the greedy selection is ill-conditioned and any FMA contraction changes
# later argmax picks (round 1, pure FAST on 4 frames: 0.99753 within +-1, max |d| 187).  The
# FAST hybrid (default) runs blocks whose window known fraction is below 0.05 on the EXACT
# kernel, and the near-tie guard re-runs blocks whose selection meets an argmax near-tie.
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_fast_mode_full_config_frame_within_tolerance(ctx, fctx, cfg):
    """FAST mode (FMA, Hermitian half-spectrum warp / wide kernels) on a full BASELINE frame:
    >= 99.9% of reconstructed pixels within +-1 of EXACT (== reference) and
    |PSNR(fast) - PSNR(exact)| <= 0.05 dB against the ground truth; argmax divergences
    show up as the residual disagreements and are reported in the assertion message."""
    wl = CONFIGS[cfg]
    img, kn = T.synth_frame(cfg, 0, wl.W, wl.H)
    ex, st_e = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    fa, st_f = fctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    unk = kn == 0
    d = np.abs(ex.astype(int) - fa.astype(int))[unk]
    within1 = float((d <= 1).mean())
    dpsnr = abs(O.psnr(img, ex) - O.psnr(img, fa))
    msg = f"c{cfg}: within1={within1:.5f} max|d|={d.max()} n(|d|>1)={(d > 1).sum()} dPSNR={dpsnr:.4f} dB"
    assert within1 >= FAST_WITHIN1, msg
    assert dpsnr <= FAST_DPSNR_DB, msg
    assert np.array_equal(fa[~unk], img[~unk])
    assert st_e.blocks_processed == st_f.blocks_processed


def test_c5_full_64_frame_batch(ctx, fctx):
    """Config 5 as specified: the 64-frame batch in one call.  FAST within the north-star
    tolerance on EVERY frame; EXACT byte-identical to the compiled reference on frames 0 and
    63 (the stated subset: the CPU reference needs ~2 s per frame on all host threads)."""
    wl = CONFIGS[5]
    assert wl.frames == 64
    imgs, kns = zip(*[T.synth_frame(5, f, wl.W, wl.H) for f in range(wl.frames)])
    img, kn = np.stack(imgs), np.stack(kns)
    ex, st_e = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    fa, st_f = fctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    assert st_e.blocks_processed == st_f.blocks_processed == st_e.blocks_reference
    for f in range(wl.frames):
        unk = kn[f] == 0
        d = np.abs(ex[f].astype(int) - fa[f].astype(int))[unk]
        within1 = float((d <= 1).mean())
        dpsnr = abs(O.psnr(img[f], ex[f]) - O.psnr(img[f], fa[f]))
        assert within1 >= FAST_WITHIN1 and dpsnr <= FAST_DPSNR_DB, (f, within1, dpsnr)
    if O.have_ref():
        p = wl.params
        for f in (0, 63):
            want = O.ref_tiled_allcores(img[f], kn[f], wl.tiles, wl.overlap, p.block_size, p.support_margin,
                                        p.model_iterations, p.compensation, p.weight_decay, band_blocks=4)
            assert np.array_equal(ex[f], want), f


def test_exact_mode_full_c2_frame_equals_oracle(ctx):
    """Byte-identical on a full 1920x1080 config-2 frame (4 tiles, d=12) vs the C oracle."""
    wl = CONFIGS[2]
    img, kn = T.synth_frame(2, 1, wl.W, wl.H)
    p = wl.params
    want, bpt = O.tiled(img, kn, wl.tiles, wl.overlap, p.block_size, p.support_margin,
                        p.model_iterations, p.compensation, p.weight_decay)
    got, st = ctx.tiled(img, kn, wl.tiles, wl.overlap, p)
    assert int((got != want).sum()) == 0
    assert st.blocks_reference == int(bpt.sum())


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_partitioned_runs_compose_to_the_full_run(ctx, fctx, mode):
    """One-process-per-GPU path on one device: the parts t % n_parts == part, run one after
    another in place, reproduce the single-part output byte-for-byte (runtime.hpp:102)."""
    import torch
    c = ctx if mode == "exact" else fctx
    wl = CONFIGS[2]
    frames, W, H, tiles = 2, 480, 270, 4
    imgs, kns = zip(*[T.synth_frame(2, f, W, H) for f in range(frames)])
    img = torch.from_numpy(np.stack(imgs)).cuda()
    kn = torch.from_numpy(np.stack(kns)).cuda()
    full = img.clone()
    c.tiled_device(full.data_ptr(), kn.data_ptr(), full.data_ptr(), W, H, frames, tiles,
                   wl.overlap, wl.params)
    for n_parts in (2, 3):
        out = img.clone()
        for part in range(n_parts):
            c.tiled_device(out.data_ptr(), kn.data_ptr(), out.data_ptr(), W, H, frames, tiles,
                           wl.overlap, wl.params, part=part, n_parts=n_parts)
        torch.cuda.synchronize()
        assert torch.equal(out, full), n_parts
    if mode == "exact":
        want, _ = O.tiled(np.stack(imgs), np.stack(kns), tiles, wl.overlap, wl.params.block_size,
                          wl.params.support_margin, wl.params.model_iterations,
                          wl.params.compensation, wl.params.weight_decay)
        assert np.array_equal(full.cpu().numpy(), want)


def test_diffusion_random_cases_equal_oracle():
    """Diffusion extrapolator (§8(f)2) on the GPU == the C restatement (== the reference)."""
    rng = np.random.default_rng(11)
    for _ in range(12):
        h, w = (int(v) for v in rng.integers(1, 90, 2))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        kn = (rng.random((h, w)) > rng.random()).astype(np.uint8)
        k = int(rng.integers(1, 40))
        got = T.DiffusionExtrapolator(k).extrapolate(img, kn)
        assert np.array_equal(got, O.diffusion(img, kn, k)), (h, w, k)
    with pytest.raises(ValueError, match="iterations must be >= 1"):
        T.DiffusionExtrapolator(0)


@pytest.mark.parametrize("tiles,overlap,iters,frames", [(1, 0, 32, 1), (4, 32, 32, 2), (8, 6, 17, 1)])
def test_diffusion_tiled_equals_oracle(tiles, overlap, iters, frames):
    wl = CONFIGS[2]
    W, H = 480, 270
    imgs, kns = zip(*[T.synth_frame(2, f, W, H) for f in range(frames)])
    img = np.stack(imgs) if frames > 1 else imgs[0]
    kn = np.stack(kns) if frames > 1 else kns[0]
    got, _ = T.run_master(img, kn, T.MasterConfig(tiles=tiles, overlap=overlap, algo="diffusion",
                                                   algo_params=f"iters={iters}"))
    want = O.tiled_diffusion(img, kn, tiles, overlap, iters)
    assert np.array_equal(got, want)
    del wl


@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_exact_mode_full_config_frame_equals_reference(ctx, cfg):
    """Full BASELINE frames (c1 512x512, c3 3840x2160 with 8 tiles, one c5 1920x1080 frame) byte-identical to the
    compiled reference run on all host cores (bit-exact band split)."""
    if not O.have_ref():
        pytest.skip("compiled reference not available")
    wl = CONFIGS[cfg]
    img, kn = T.synth_frame(cfg, 0, wl.W, wl.H)
    p = wl.params
    want = O.ref_tiled_allcores(img, kn, wl.tiles, wl.overlap, p.block_size, p.support_margin,
                                p.model_iterations, p.compensation, p.weight_decay)
    got, _ = ctx.tiled(img, kn, wl.tiles, wl.overlap, p)
    assert int((got != want).sum()) == 0


@pytest.mark.parametrize("cfg,frames", [(2, 1), (3, 1), (5, 3), (1, 1)])
def test_streamed_host_path_equals_one_shot(ctx, fctx, cfg, frames, tune_env):
    """The single-GPU host path streams row bands (H2D / FSE / D2H overlap over streams); its
    output and block counts must equal the one-shot path (TF_STREAM_BANDS=1) for any band
    count, in both modes, including multi-frame batches."""
    from paper_2207_00238_b200.configs import workload
    wl = workload(cfg, frames=frames)
    W, H = (wl.W, wl.H) if cfg != 3 else (960, 540)
    imgs, kns = zip(*[T.synth_frame(cfg, f, W, H) for f in range(frames)])
    img = np.stack(imgs) if frames > 1 else imgs[0]
    kn = np.stack(kns) if frames > 1 else kns[0]
    for c in (ctx, fctx):
        tune_env([c], TF_STREAM_BANDS=1)
        want, st1 = c.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        for nb in ("2", "5", "8", "16"):
            tune_env([c], TF_STREAM_BANDS=nb)
            got, st = c.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
            assert np.array_equal(got, want), f"c{cfg} {c.mode} bands={nb}: {(got != want).sum()} pixels differ"
            assert st.blocks_processed == st1.blocks_processed
            assert st.blocks_reference == st1.blocks_reference


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_fast_kernels_with_empty_windows_and_odd_block_counts(ctx, fctx, cfg):
    """FAST half / pair / wide kernels next to large holes: windows without a known pixel
    give 128 (extrapolate.hpp:320-333), a half-warp whose block stops while its partner runs
    (pair kernel) and odd block counts (idle half) behave; KAT: all-unknown frame -> 128."""
    wl = CONFIGS[cfg]
    p = wl.params
    span = p.block_size + 2 * p.support_margin
    W, H = 4 * span + 7, 3 * span + 5
    img, kn = T.synth_frame(cfg, 1, W, H)
    kn = kn.copy()
    kn[span // 2: span // 2 + 2 * span, span: span + 2 * span] = 0  # hole wider than a window
    for tiles in (1, 2, 3):
        ex, st_e = ctx.tiled(img, kn, tiles, wl.overlap, p)
        fa, st_f = fctx.tiled(img, kn, tiles, wl.overlap, p)
        assert st_e.blocks_processed == st_f.blocks_processed
        unk = kn == 0
        assert np.array_equal(fa[~unk], img[~unk])
        want = O.tiled(img, kn, tiles, wl.overlap, p.block_size, p.support_margin, p.model_iterations,
                       p.compensation, p.weight_decay)[0]
        assert np.array_equal(ex, want)
        d = np.abs(ex.astype(int) - fa.astype(int))[unk]
        assert (d <= 1).mean() >= FAST_WITHIN1, f"tiles={tiles}: max|d|={d.max()}"
        assert np.array_equal(ex == 128, fa == 128) or (d <= 1).mean() >= FAST_WITHIN1
    z = np.zeros_like(kn)
    fa, _ = fctx.tiled(img, z, 2, wl.overlap, p)
    assert (fa == 128).all()


def test_fast_hybrid_routes_ill_conditioned_blocks(ctx, fctx, tune_env):
    """Config 5 frames: with the hybrid off (TF_HYBRID=0) FAST leaves the tolerance; with it on
    the blocks it routes to the EXACT kernel are counted in blocks_processed and the output
    meets the tolerance; EXACT mode ignores the setting."""
    wl = CONFIGS[5]
    imgs, kns = zip(*[T.synth_frame(5, f, wl.W, wl.H) for f in range(2)])
    img, kn = np.stack(imgs), np.stack(kns)
    ex, st_e = ctx.tiled(img, kn, 1, wl.overlap, wl.params)
    unk = kn == 0
    tune_env([fctx, ctx], TF_HYBRID=0, TF_NO_TIE_GUARD=1)
    fa0, _ = fctx.tiled(img, kn, 1, wl.overlap, wl.params)
    tune_env([fctx, ctx], TF_HYBRID=0.05, TF_NO_TIE_GUARD=None)
    fa1, st_f = fctx.tiled(img, kn, 1, wl.overlap, wl.params)
    ex1, _ = ctx.tiled(img, kn, 1, wl.overlap, wl.params)
    assert np.array_equal(ex, ex1)
    assert st_f.blocks_processed == st_e.blocks_processed
    w0 = (np.abs(ex.astype(int) - fa0.astype(int))[unk] <= 1).mean()
    w1 = (np.abs(ex.astype(int) - fa1.astype(int))[unk] <= 1).mean()
    assert w1 >= FAST_WITHIN1 > w0, (w0, w1)


def test_device_path_graph_replay_tracks_inputs_and_shapes(fctx):
    """Repeated identical device-path calls are captured once and replayed as a CUDA graph:
    new contents of the same buffers must be picked up, and a call of another shape (or the
    host path) in between must not leave a stale graph behind."""
    import torch
    wl = CONFIGS[2]
    W, H = 480, 270
    frames = [T.synth_frame(2, f, W, H) for f in range(4)]
    d_img = torch.empty(H * W, dtype=torch.uint8, device="cuda")
    d_kn = torch.empty_like(d_img)
    d_out = torch.empty_like(d_img)
    s = torch.cuda.Stream()

    def dev_call(img, kn, tiles=wl.tiles):
        d_img.copy_(torch.from_numpy(img.reshape(-1)))
        d_kn.copy_(torch.from_numpy(kn.reshape(-1)))
        torch.cuda.synchronize()
        fctx.tiled_device(d_img.data_ptr(), d_kn.data_ptr(), d_out.data_ptr(), W, H, 1, tiles, wl.overlap,
                          wl.params, stream=s.cuda_stream)
        s.synchronize()
        return d_out.cpu().numpy().reshape(H, W)

    for rep in range(3):
        for img, kn in frames:  # repeated identical calls on new data (graph replays)
            want, _ = fctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
            for _ in range(3):
                got = dev_call(img, kn)
                assert np.array_equal(got, want)
        img, kn = frames[0]
        want3, _ = fctx.tiled(img, kn, 3, wl.overlap, wl.params)
        assert np.array_equal(dev_call(img, kn, tiles=3), want3)  # another shape in between


def test_host_path_graph_replay_tracks_inputs(fctx, ctx):
    """Repeated identical host-buffer calls (pinned buffers) are captured once and replayed:
    the replays must read the current contents of the same host buffers, and calls of other
    shapes / the device path in between must not leave a stale graph."""
    import torch
    wl = CONFIGS[2]
    W, H = 960, 540
    frames = [T.synth_frame(2, f, W, H) for f in range(3)]
    h_img = torch.empty(H * W, dtype=torch.uint8).pin_memory()
    h_kn = torch.empty_like(h_img).pin_memory()
    h_out = torch.empty_like(h_img).pin_memory()
    import ctypes as C
    from paper_2207_00238_b200 import _native as N
    p = wl.params._c()

    def host_call(c, img, kn, tiles=wl.tiles):
        h_img.numpy()[:] = img.reshape(-1)
        h_kn.numpy()[:] = kn.reshape(-1)
        N.check(N.lib().tf_tiled_extrapolate(c.handle, h_img.data_ptr(), h_kn.data_ptr(), W, H, 1, tiles,
                                             wl.overlap, C.byref(p), h_out.data_ptr(), None))
        return h_out.numpy().reshape(H, W).copy()

    for rep in range(2):
        for img, kn in frames:
            want = O.tiled(img, kn, wl.tiles, wl.overlap, p.block, p.margin, p.iters, p.gamma, p.rho)[0]
            got = [host_call(ctx, img, kn) for _ in range(3)]  # EXACT: byte-identical every replay
            for g in got:
                assert np.array_equal(g, want)
            fa = [host_call(fctx, img, kn) for _ in range(3)]
            assert all(np.array_equal(f, fa[0]) for f in fa)
        img, kn = frames[0]
        want3 = O.tiled(img, kn, 3, wl.overlap, p.block, p.margin, p.iters, p.gamma, p.rho)[0]
        assert np.array_equal(host_call(ctx, img, kn, tiles=3), want3)


GOLD = __import__("pathlib").Path(__file__).resolve().parent / "golden"
GOLD_FSE = sorted(p.name for p in GOLD.glob("*.npz") if p.name != "tiling.npz")


@pytest.mark.parametrize("name", GOLD_FSE)
def test_gpu_reproduces_reference_golden_fixtures(ctx, fctx, name):
    """The committed fixtures the reference itself produced (tests/golden/make_golden.py):
    EXACT byte-identical, FAST within the north-star tolerance, block counts equal."""
    d = np.load(GOLD / name)
    b, m, i = (int(v) for v in d["params"])
    g, r = (float(v) for v in d["fparams"])
    p = T.FseLiteParams(b, m, i, g, r)
    tiles, overlap = int(d["tiles"]), int(d["overlap"])
    got, st = ctx.tiled(d["img"], d["known"], tiles, overlap, p)
    assert np.array_equal(got, d["out"]), f"{name}: {(got != d['out']).sum()} px differ"
    if tiles == 1 and overlap == 0:
        assert st.blocks_reference == int(d["nblocks"])  # FseLiteTrace block count
    fa, _ = fctx.tiled(d["img"], d["known"], tiles, overlap, p)
    unk = d["known"] == 0
    if unk.any():
        dd = np.abs(fa.astype(int) - d["out"].astype(int))[unk]
        assert (dd <= 1).mean() >= FAST_WITHIN1, name
    assert np.array_equal(fa[~unk], d["img"][~unk])


def test_device_path_refuses_a_caller_capture(fctx):
    """Called while the caller captures its stream into a CUDA graph, the device path raises
    ValueError without touching the stream: the caller's capture stays valid, and the next
    plain call still matches the direct result (repeats replay the library's own graph)."""
    import torch
    wl = CONFIGS[2]
    W, H = 320, 180
    img, kn = T.synth_frame(2, 5, W, H)
    want, _ = fctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
    d_img = torch.from_numpy(img.reshape(-1)).cuda()
    d_kn = torch.from_numpy(kn.reshape(-1)).cuda()
    d_out = torch.empty_like(d_img)
    s = torch.cuda.Stream()
    call = lambda: fctx.tiled_device(d_img.data_ptr(), d_kn.data_ptr(), d_out.data_ptr(), W, H, 1, wl.tiles,
                                     wl.overlap, wl.params, stream=s.cuda_stream)
    with torch.cuda.stream(s):
        call()
    torch.cuda.synchronize()
    x = torch.zeros(16, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        x += 1
        with pytest.raises(ValueError, match="capturing"):
            call()
    g.replay()
    torch.cuda.synchronize()
    assert float(x[0]) == 1.0
    d_out.zero_()
    with torch.cuda.stream(s):
        call()
        call()
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().reshape(H, W), want)


def test_big_window_kernel_forced_on_small_cases(ctx, fctx, tune_env):
    """The global-scratch big-window kernel, forced onto ordinary launches (TF_FORCE_BIG=1):
    byte-identical to the oracle in both modes (it computes with EXACT arithmetic)."""
    tune_env([ctx, fctx], TF_FORCE_BIG=1)
    rng = np.random.default_rng(77)
    for trial in range(16):
        w, h = int(rng.integers(6, 80)), int(rng.integers(6, 80))
        B, m, I = int(rng.integers(2, 17)), int(rng.integers(0, 20)), int(rng.integers(1, 60))
        g, r = float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.2, 0.95))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        kn = (rng.random((h, w)) > rng.uniform(0.05, 0.7)).astype(np.uint8)
        tiles = int(rng.integers(1, 4))
        p = _params(B, m, I, g, r)
        try:
            want, bpt = O.tiled(img, kn, tiles, 3, B, m, I, g, r)
        except O.OracleError:
            continue
        for c in (ctx, fctx):
            got, st = c.tiled(img, kn, tiles, 3, p)
            assert np.array_equal(got, want), f"trial {trial} {c.mode}: {(got != want).sum()} px differ"
            assert st.blocks_reference == int(bpt.sum())


@pytest.mark.parametrize("B,m,I,W,H", [(32, 32, 25, 160, 128),    # 96x96 windows: 9216 bins
                                       (64, 64, 60, 320, 256),    # 192x192 windows: 36864 bins
                                       (8, 12, 12000, 48, 40)])   # 32x32 windows, 12000-entry logs
def test_big_windows_and_long_logs_equal_oracle(ctx, fctx, B, m, I, W, H):
    """Support windows and selection logs past the shared-memory kernels' capacity (formerly
    TF_EUNSUPPORTED) run on the big-window kernel: byte-identical to the oracle in both modes."""
    img, kn = T.synth_frame(1, 3, W, H)
    want = O.fse_lite(img, kn, B, m, I, 0.5, 0.8)
    for c in (ctx, fctx):
        got, st = c.tiled(img, kn, 1, 0, _params(B, m, I, 0.5, 0.8))
        assert np.array_equal(got, want), f"{c.mode}: {(got != want).sum()} px differ"
        assert st.blocks_processed == st.blocks_reference == T.count_blocks(kn, B)


def test_degenerate_shapes_equal_oracle(ctx, fctx):
    """1x1, single-row and single-column images, blocks larger than the image, margin 0:
    EXACT byte-identical to the oracle, FAST within +-1 of it on every pixel."""
    rng = np.random.default_rng(9)
    shapes = [(1, 1), (1, 7), (7, 1), (2, 2), (3, 5), (5, 3), (1, 40), (40, 1)]
    for (w, h) in shapes:
        for (B, m) in [(2, 0), (4, 8), (16, 3)]:
            img = rng.integers(0, 256, (h, w), dtype=np.uint8)
            kn = (rng.random((h, w)) > 0.5).astype(np.uint8)
            want = O.fse_lite(img, kn, B, m, 20, 0.5, 0.8)
            got, st = ctx.tiled(img, kn, 1, 0, _params(B, m, 20, 0.5, 0.8))
            assert np.array_equal(got, want), f"{w}x{h} B={B} m={m}"
            assert st.blocks_reference == T.count_blocks(kn, B)
            fgot, _ = fctx.tiled(img, kn, 1, 0, _params(B, m, 20, 0.5, 0.8))
            assert np.abs(fgot.astype(int) - want.astype(int)).max() <= 1, f"fast {w}x{h} B={B} m={m}"


@pytest.mark.parametrize("b,m", [(2, 7), (4, 6), (8, 4)])
def test_pair_kernel_variants_against_exact_and_oracle(ctx, fctx, b, m):
    """FAST on full 16x16 windows runs the pair kernel: its ACC variant (the model accumulated
    at the core pixels, no selection log) for blocks of at most 16 pixels (B = 2, 4), the log
    variant above (B = 8).  Each is held to the north-star tolerance against the oracle; the
    statistics build (device call with stats) must write the same bytes as the plain one; the
    near-tie band hands blocks to the EXACT kernel, so a mirror-symmetric mask -- exact
    argmax ties in the reference -- still reproduces EXACT byte for byte."""
    import torch
    W, H, I = 200, 136, 30
    img, kn = T.synth_frame(3, 11, W, H)  # i.i.d. pixel loss, p = 0.2
    p = T.FseLiteParams(b, m, I, 0.5, 0.7)
    want = O.tiled(img, kn, 2, m, b, m, I, 0.5, 0.7)[0]
    ex, _ = ctx.tiled(img, kn, 2, m, p)
    assert np.array_equal(ex, want)
    fa, st = fctx.tiled(img, kn, 2, m, p)
    unk = kn == 0
    d = np.abs(fa.astype(int) - want.astype(int))[unk]
    assert (d <= 1).mean() >= FAST_WITHIN1, f"B={b}: {(d > 1).sum()} of {d.size} pixels off by more than 1"
    assert np.array_equal(fa[~unk], img[~unk])
    # statistics build of the same kernels
    d_img = torch.from_numpy(img.reshape(-1)).cuda()
    d_kn = torch.from_numpy(kn.reshape(-1)).cuda()
    d_out = torch.empty_like(d_img)
    rs = fctx.tiled_device(d_img.data_ptr(), d_kn.data_ptr(), d_out.data_ptr(), W, H, 1, 2, m, p,
                           want_stats=True)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().reshape(H, W), fa)
    assert rs.blocks_processed == st.blocks_processed
    # structured ties: a mask symmetric about both axes on a symmetric image
    yy, xx = np.mgrid[0:64, 0:64]
    simg = (128 + 60 * np.cos(2 * np.pi * (xx - 31.5) / 16) * np.cos(2 * np.pi * (yy - 31.5) / 8)).astype(np.uint8)
    skn = np.ones((64, 64), np.uint8)
    skn[24:40, 24:40] = 0
    skn[28:36, 28:36] = 1
    swant = O.fse_lite(simg, skn, b, m, I, 0.5, 0.7)
    sex, _ = ctx.tiled(simg, skn, 1, 0, p)
    assert np.array_equal(sex, swant)
    sfa, sst = fctx.tiled(simg, skn, 1, 0, p)
    sd = np.abs(sfa.astype(int) - swant.astype(int))[skn == 0]
    assert (sd <= 1).mean() >= FAST_WITHIN1, f"symmetric case B={b}: {(sd > 1).sum()} of {sd.size} off, refined {sst.blocks_refined}"
