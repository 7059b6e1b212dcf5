"""The CPU oracle is pinned before it is trusted (CPU-only tests).

* the plain-C restatement (oracle/fse_oracle.c) reproduces the golden
  fixtures the reference produced (tests/golden/make_golden.py);
* where the compiled reference (oracle/_ref) is present it is also compared
  live, byte-for-byte, on seeded random cases, and the reference's own KATs
  (test_extrapolate.cpp) are re-checked through it.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
FSE_FIXTURES = sorted(p.name for p in GOLD.glob("*.npz") if p.name != "tiling.npz")
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")


def load(name):
    d = np.load(GOLD / name)
    b, m, i = (int(v) for v in d["params"])
    g, r = (float(v) for v in d["fparams"])
    return d, (b, m, i, g, r)


def test_fixture_set_present():
    assert len(FSE_FIXTURES) >= 10
    assert (GOLD / "tiling.npz").exists()


@pytest.mark.parametrize("name", FSE_FIXTURES)
def test_restatement_reproduces_golden(name):
    d, p = load(name)
    tiles, overlap = int(d["tiles"]), int(d["overlap"])
    if tiles == 1 and overlap == 0:
        out, st = O.fse_lite(d["img"], d["known"], *p, with_stats=True)
        assert len(st) == int(d["nblocks"])  # FseLiteTrace block count
    else:
        out, _ = O.tiled(d["img"], d["known"], tiles, overlap, *p)
    assert np.array_equal(out, d["out"]), f"{name}: {(out != d['out']).sum()} px differ"


def test_golden_kats_hold():
    # test_extrapolate.cpp:80-113 properties, on the reference's own outputs
    d, _ = load("kat_all_known.npz")
    assert np.array_equal(d["out"], d["img"])
    d, _ = load("kat_constant.npz")
    assert (d["out"] == 183).all()
    d, _ = load("kat_sinusoid.npz")
    hole = d["known"] == 0
    assert np.abs(d["out"][hole].astype(int) - d["img"][hole].astype(int)).max() <= 2


@needs_ref
def test_restatement_equals_reference_random():
    rng = np.random.default_rng(7)
    for trial in range(40):
        w, h = int(rng.integers(4, 72)), int(rng.integers(4, 72))
        B, m, I = int(rng.integers(2, 12)), int(rng.integers(0, 14)), int(rng.integers(1, 64))
        g, r = float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.2, 0.95))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8) if trial % 2 else O.ref_make_scene(w, h, trial)
        kn = (rng.random((h, w)) > rng.uniform(0.05, 0.8)).astype(np.uint8)
        a, nb = O.ref_fse_lite(img, kn, B, m, I, g, r, count_blocks=True)
        b, st = O.fse_lite(img, kn, B, m, I, g, r, with_stats=True)
        assert np.array_equal(a, b), f"trial {trial}"
        assert nb == len(st)


@needs_ref
def test_restatement_equals_reference_tiled():
    img = O.ref_make_scene(150, 90, 3)
    kn = O.ref_gen_scatter_mask(150, 90, 0.3, 5, 9)
    for tiles, d in ((1, 0), (3, 5), (6, 12), (7, 0)):
        a, _ = O.ref_run_local(img, kn, tiles, d, 6, 7, 30, 0.5, 0.8, workers=2)
        b, _ = O.tiled(img, kn, tiles, d, 6, 7, 30, 0.5, 0.8)
        assert np.array_equal(a, b), (tiles, d)


@needs_ref
def test_allcores_band_split_is_bit_exact():
    # the CPU baseline's all-cores split must equal the as-shipped run_local
    img = O.ref_make_scene(200, 120, 5)
    kn = O.ref_gen_scatter_mask(200, 120, 0.25, 8, 6)
    a, _ = O.ref_run_local(img, kn, 4, 12, 8, 12, 20, 0.5, 0.8, workers=4)
    for bb in (1, 2, 5):
        b = O.ref_tiled_allcores(img, kn, 4, 12, 8, 12, 20, 0.5, 0.8, threads=3, band_blocks=bb)
        assert np.array_equal(a, b), bb


@needs_ref
def test_reference_energy_non_increasing():
    # test_extrapolate.cpp:115-127 through the compiled reference's trace hook
    import ctypes as C
    rng = np.random.default_rng(31)
    img = rng.integers(0, 256, (20, 20), dtype=np.uint8)
    kn = O.ref_gen_scatter_mask(20, 20, 0.3, 2, 7)
    buf = np.zeros(100000)
    n = C.c_int64(0)
    rc = O.ref().ref_fse_lite_trace(img.ctypes.data, kn.ctypes.data, 20, 20, 4, 8, 40, 0.5, 0.8,
                                    buf.ctypes.data, buf.size, C.byref(n))
    assert rc == 0
    k, blocks = 0, 0
    while k < n.value:
        cnt = int(buf[k])
        e = buf[k + 1:k + 1 + cnt]
        assert (np.diff(e) <= 1e-9).all()
        k += 1 + cnt
        blocks += 1
    assert blocks > 0


@needs_ref
def test_restatement_block_stats_consistent():
    # instrumentation used for the F_b flop count: I_b <= I, T_b <= 2 I_b, P_b <= I_b
    img = O.ref_make_scene(64, 48, 2)
    kn = O.ref_gen_scatter_mask(64, 48, 0.3, 4, 3)
    _, st = O.fse_lite(img, kn, 8, 8, 25, 0.5, 0.8, with_stats=True)
    assert (st["iters"] <= 25).all()
    assert (st["pairs"] <= st["iters"]).all()
    assert (st["touched"] <= st["iters"] + st["pairs"]).all()
    assert (st["min_gap"] >= 0).all()


def test_diffusion_restatement_equals_compiled_reference():
    """oracle/fse_oracle.c orc_diffusion / orc_tiled_diffusion == the reference's
    diffusion_extrapolate / run_local(algo="diffusion") byte-for-byte."""
    if not O.have_ref():
        pytest.skip("compiled reference not available")
    rng = np.random.default_rng(7)
    for _ in range(40):
        h, w = (int(v) for v in rng.integers(1, 48, 2))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        kn = (rng.random((h, w)) > rng.random()).astype(np.uint8)
        k = int(rng.integers(1, 50))
        assert np.array_equal(O.diffusion(img, kn, k), O.ref_diffusion(img, kn, k))
    img = rng.integers(0, 256, (130, 170), dtype=np.uint8)
    kn = (rng.random((130, 170)) > 0.3).astype(np.uint8)
    for tiles, d, k in ((1, 0, 32), (4, 32, 32), (6, 8, 20), (3, 40, 5)):
        assert np.array_equal(O.tiled_diffusion(img, kn, tiles, d, k),
                              O.ref_run_local_diffusion(img, kn, tiles, d, k, 2))


@needs_ref
@pytest.mark.parametrize("cfg,W,H", [(1, 512, 512), (2, 640, 360), (3, 960, 540), (4, 800, 450), (5, 480, 270)])
def test_reference_shim_generator_equals_product_generator(cfg, W, H):
    """bench.py's reference arm builds its inputs with ref_synth_frame (synth_gen.hpp compiled
    into oracle/_ref) so that it never loads the product library; the bytes must equal the
    product's tf_synth_frame (the same header-only source)."""
    from paper_2207_00238_b200 import tframe as T
    for frame in (0, 3):
        a = O.ref_synth_frame(cfg, frame, W, H)
        b = T.synth_frame(cfg, frame, W, H)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@needs_ref
def test_allcores_part_split_composes():
    """The bounded-sample split of the reference arm (tiles t % n == part) covers every core."""
    img, kn = O.ref_synth_frame(3, 0, 320, 200)
    args = (8, 6, 4, 6, 20, 0.5, 0.7)
    whole = O.ref_tiled_allcores(img, kn, *args, threads=4)
    out = img.copy()
    for part in range(3):
        O.ref_tiled_allcores(img, kn, *args, threads=4, out=out, part=part, n_parts=3)
    assert np.array_equal(out, whole)
