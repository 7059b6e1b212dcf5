"""Quality metrics (reference metrics.hpp:12-90).

CPU: the C restatement (oracle/) equals the compiled reference bit for bit.
GPU: tf_quality / tf_mse / tf_psnr / tf_mse_missing / tf_ssim against the restatement:
MSE, PSNR and MSE-over-missing bit-identical; SSIM exact when the frame has <= 2 windows
(the per-window values are bit-identical, only the mean's summation order differs) and
within SSIM_REL of the reference's sequential sum otherwise."""
import math

import numpy as np
import pytest

import oracle as O

SSIM_REL = 1e-12

SHAPES = [(8, 8), (9, 8), (8, 9), (13, 11), (64, 48), (97, 61), (128, 128), (250, 37)]


def _pair(rng, h, w, noise=20):
    a = rng.integers(0, 256, (h, w), dtype=np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-noise, noise + 1, (h, w)), 0, 255).astype(np.uint8)
    k = (rng.random((h, w)) > 0.3).astype(np.uint8)
    return a, b, k


def test_restated_metrics_equal_reference():
    if not O.have_ref():
        pytest.skip("compiled reference not available")
    rng = np.random.default_rng(7)
    for h, w in SHAPES:
        a, b, k = _pair(rng, h, w)
        assert O.mse(a, b) == O.ref_mse(a, b)
        assert O.orc_psnr(a, b) == O.ref_psnr(a, b)
        assert O.mse_missing(a, b, k) == O.ref_mse_missing(a, b, k)
        assert O.ssim(a, b) == O.ref_ssim(a, b)
    a, b, _ = _pair(rng, 16, 16)
    assert O.orc_psnr(a, a) == math.inf == O.ref_psnr(a, a)
    with pytest.raises(O.OracleError):
        O.ref_mse_missing(a, b, np.ones_like(a))
    with pytest.raises(O.OracleError):
        O.mse_missing(a, b, np.ones_like(a))
    assert math.isnan(O.ssim(a[:7], b[:7]))


@pytest.mark.gpu
def test_gpu_metrics_match_restatement():
    from paper_2207_00238_b200 import tframe as T
    rng = np.random.default_rng(11)
    for h, w in SHAPES:
        a, b, k = _pair(rng, h, w)
        assert T.mse(a, b) == O.mse(a, b)
        assert T.psnr(a, b) == O.orc_psnr(a, b)
        assert T.mse_missing(a, b, k) == O.mse_missing(a, b, k)
        s_gpu, s_ref = T.ssim(a, b), O.ssim(a, b)
        if (h - 7) * (w - 7) <= 2:
            assert s_gpu == s_ref
        else:
            assert abs(s_gpu - s_ref) <= SSIM_REL * abs(s_ref)
    a, b, _ = _pair(rng, 20, 20)
    assert T.psnr(a, a) == math.inf
    with pytest.raises(ValueError, match="mse_missing: mask has no unknown pixels"):
        T.mse_missing(a, b, np.ones_like(a))
    with pytest.raises(ValueError, match="ssim: image smaller than the 8x8 window"):
        T.ssim(a[:7], b[:7])


@pytest.mark.gpu
def test_gpu_quality_batch_and_full_frame():
    """A batch of frames (scalar and 16-byte paths) and a full 3840x2160 frame of an FSE
    reconstruction against the restatement."""
    from paper_2207_00238_b200 import tframe as T
    ctx = T.Context(1, [0], "fast")
    try:
        rng = np.random.default_rng(3)
        for (h, w) in ((45, 67), (64, 64)):  # w*h % 16 != 0 -> byte path; == 0 -> 16-byte path
            fr = [_pair(rng, h, w) for _ in range(5)]
            A = np.stack([f[0] for f in fr]); B = np.stack([f[1] for f in fr]); K = np.stack([f[2] for f in fr])
            q = ctx.quality(A, B, K)
            for i, (a, b, k) in enumerate(fr):
                assert q[i]["mse"] == O.mse(a, b)
                assert q[i]["psnr"] == O.orc_psnr(a, b)
                assert q[i]["mse_missing"] == O.mse_missing(a, b, k)
                assert q[i]["n_missing"] == int((k == 0).sum())
                assert abs(q[i]["ssim"] - O.ssim(a, b)) <= SSIM_REL * abs(O.ssim(a, b))
        img, kn = T.synth_frame(3, 0, 3840, 2160)
        from paper_2207_00238_b200.configs import CONFIGS
        wl = CONFIGS[3]
        out, _ = ctx.tiled(img, kn, wl.tiles, wl.overlap, wl.params)
        q = ctx.quality(img, out, kn)[0]
        assert q["mse"] == O.mse(img, out)
        assert q["psnr"] == O.orc_psnr(img, out)
        assert q["mse_missing"] == O.mse_missing(img, out, kn)
        s = O.ssim(img, out)
        assert abs(q["ssim"] - s) <= SSIM_REL * abs(s)
        nq = ctx.quality(img, out, None, ssim=False)[0]
        assert nq["mse"] == q["mse"] and math.isnan(nq["ssim"]) and nq["n_missing"] == 0
    finally:
        ctx.close()
