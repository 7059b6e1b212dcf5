"""Host-side tiling, halo expansion, parameters and block enumeration of the
product library (C-ABI, no GPU needed) against the reference.

Bit-exactness bar (north star): the partitioner and the mask/block
enumeration must match the reference bit for bit.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2207_00238_b200 import tframe as T

GOLD = Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")


def rects(layout):
    return np.array([[t.x, t.y, t.w, t.h] for t in layout.tiles], np.int32).reshape(-1, 4)


def test_golden_layout_1024x480x22():
    # test_tiling.cpp:10-30 and :109-113
    lay = T.plan_proposed(1024, 480, 22)
    r = rects(lay)
    assert len(r) == 22
    rows = [(0, 178, 8), (178, 157, 7), (335, 145, 7)]
    i = 0
    for y, h, n in rows:
        for _ in range(n):
            assert r[i][1] == y and r[i][3] == h
            i += 1
    assert (r[:8, 2] == 128).all()
    assert list(r[8:15, 2]) == [147, 147, 146, 146, 146, 146, 146]
    assert T.interior_boundary(lay) == 5106


def test_single_tile_and_grid():
    assert T.plan_proposed(100, 100, 1).tiles == [T.Rect(0, 0, 100, 100)]
    assert all((t.w, t.h) == (300, 200) for t in T.plan_proposed(600, 400, 4).tiles)


def test_portrait_is_transposed_and_row_major():
    port = rects(T.plan_proposed(480, 1024, 22))
    land = rects(T.plan_proposed(1024, 480, 22))
    want = {(y, x, h, w) for x, y, w, h in land}
    assert {tuple(r) for r in port} == want
    keys = [(r[1], r[0]) for r in port]
    assert keys == sorted(keys)


def test_expand_golden_halos():
    # test_overlap.cpp:22-31
    assert T.expand(T.Rect(0, 0, 128, 178), 32, 1024, 480).halo == T.Rect(0, 0, 160, 210)
    assert T.expand(T.Rect(128, 178, 147, 157), 32, 1024, 480).halo == T.Rect(96, 146, 211, 221)
    z = T.expand(T.Rect(10, 20, 5, 6), 0, 100, 100)
    assert z.halo == z.core
    with pytest.raises(ValueError):
        T.expand(T.Rect(0, 0, 10, 10), -1, 100, 100)
    with pytest.raises(ValueError):
        T.expand(T.Rect(95, 0, 10, 10), 1, 100, 100)


def test_tiling_fixtures_from_reference():
    g = np.load(GOLD / "tiling.npz")
    for name in [k for k in g.files if not k.endswith("_ib")]:
        a = g[name]
        W, H, N, d = (int(v) for v in a[0])
        cores, halos = a[1:1 + N], a[1 + N:]
        lay = T.plan_proposed(W, H, N)
        assert np.array_equal(rects(lay), cores), name
        got_h = np.array([[e.halo.x, e.halo.y, e.halo.w, e.halo.h]
                          for e in (T.expand(t, d, W, H) for t in lay.tiles)], np.int32)
        assert np.array_equal(got_h, halos), name
        assert T.interior_boundary(lay) == int(g[name + "_ib"][0]), name


def test_appendix_c_config_grid_offsets():
    # config 2 right column halos start at x=948 (grid offset 4 for B=8)
    lay = T.plan_proposed(1920, 1080, 4)
    halos = [T.expand(t, 12, 1920, 1080).halo for t in lay.tiles]
    assert [h.x for h in halos] == [0, 948, 0, 948]
    assert [h.y for h in halos] == [0, 0, 528, 528]
    assert all((h.w, h.h) == (972, 552) for h in halos)


def _fuzz_cases(seed, n):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        w, h = int(rng.integers(1, 160)), int(rng.integers(1, 160))
        yield w, h, int(rng.integers(1, min(w * h, 48) + 1))


def test_fuzz_plan_against_restated_oracle():
    for w, h, n in _fuzz_cases(11, 3000):
        try:
            want = O.plan_proposed(w, h, n)
            werr = None
        except O.OracleError as e:
            want, werr = None, e.code
        try:
            got = rects(T.plan_proposed(w, h, n))
            gerr = None
        except T.TilingError:
            got, gerr = None, 4
        assert gerr == werr, (w, h, n)
        if want is not None:
            assert np.array_equal(got, want), (w, h, n)


@needs_ref
def test_fuzz_plan_and_expand_against_reference():
    rng = np.random.default_rng(5)
    for w, h, n in _fuzz_cases(13, 1500):
        try:
            want = O.ref_plan_proposed(w, h, n)
        except O.OracleError as e:
            assert e.code == 4
            with pytest.raises(T.TilingError):
                T.plan_proposed(w, h, n)
            continue
        lay = T.plan_proposed(w, h, n)
        assert np.array_equal(rects(lay), want), (w, h, n)
        d = int(rng.integers(0, 40))
        for t, c in zip(lay.tiles, want):
            e = T.expand(t, d, w, h).halo
            assert [e.x, e.y, e.w, e.h] == list(O.ref_expand(c, d, w, h))


def test_invalid_plan_arguments():
    with pytest.raises(ValueError):
        T.plan_proposed(0, 10, 1)
    with pytest.raises(T.TilingError):
        T.plan_proposed(3, 3, 10)  # more tiles than pixels


def test_count_blocks_matches_oracle_enumeration():
    rng = np.random.default_rng(3)
    for trial in range(30):
        w, h, B = int(rng.integers(1, 90)), int(rng.integers(1, 90)), int(rng.integers(2, 17))
        kn = (rng.random((h, w)) > rng.uniform(0.0, 0.3)).astype(np.uint8)
        img = np.zeros((h, w), np.uint8)
        _, st = O.fse_lite(img, kn, B, 0, 1, 0.5, 0.8, with_stats=True)
        assert T.count_blocks(kn, B) == len(st)


# ---------------------------------------------------------------- parameters
PARAM_STRINGS = ["", "block=8,iters=20,gamma=0.25,rho=0.5", "block=16,margin=14,iters=100",
                 "margin=0", "iters=1,gamma=1", "block=2,margin=3", ",,block=5,,"]
BAD_STRINGS = ["gamma=2.0", "rho=1", "block=1", "iters=0", "margin=-1", "garbage", "block=x"]


def test_registry_defaults_and_parsing():
    fse = T.registry_lookup("fse-lite")
    assert fse.name() == "fse-lite"
    assert fse.params().block_size == 4 and fse.influence_radius() == 12
    p = T.registry_lookup("fse-lite", "block=8,iters=20,gamma=0.25,rho=0.5").params()
    assert (p.block_size, p.support_margin, p.model_iterations, p.compensation, p.weight_decay) == (8, 16, 20, 0.25, 0.5)
    with pytest.raises(ValueError, match="diffusion, fse-lite"):
        T.registry_lookup("bogus")
    for s in BAD_STRINGS:
        with pytest.raises(ValueError):
            T.registry_lookup("fse-lite", s)


@needs_ref
def test_registry_matches_reference():
    for s in PARAM_STRINGS:
        r = O.ref_registry("fse-lite", s)
        e = T.registry_lookup("fse-lite", s)
        p = e.params()
        assert (p.block_size, p.support_margin, p.model_iterations, p.compensation, p.weight_decay) == \
            (r["block"], r["margin"], r["iters"], r["gamma"], r["rho"]), s
        assert e.params_string() == r["params_string"]
        assert e.influence_radius() == r["influence"]
    for s in BAD_STRINGS:
        with pytest.raises(O.OracleError):
            O.ref_registry("fse-lite", s)


def test_check_params_messages():
    with pytest.raises(ValueError, match="block_size must be >= 2"):
        T.check_fse_params(T.FseLiteParams(1))
    with pytest.raises(ValueError, match="compensation"):
        T.check_fse_params(T.FseLiteParams(4, 8, 10, 0.0))
    with pytest.raises(ValueError, match="weight_decay"):
        T.check_fse_params(T.FseLiteParams(4, 8, 10, 0.5, 1.0))


def test_registry_diffusion_matches_reference():
    """registry_lookup("diffusion", params) (extrapolate.hpp:418-424): default 32 sweeps,
    params_string / influence radius, key=value parsing errors as the reference."""
    e = T.registry_lookup("diffusion")
    assert e.name() == "diffusion" and e.influence_radius() == 32 and e.params_string() == "iters=32"
    e = T.registry_lookup("diffusion", "iters=7,block=3")
    assert e.influence_radius() == 7 and e.params_string() == "iters=7"
    assert T.registry_lookup("diffusion", "iters= 9x,,").influence_radius() == 9  # std::stoi
    with pytest.raises(ValueError, match="expected key=value"):
        T.registry_lookup("diffusion", "iters")
    with pytest.raises(ValueError, match="iterations must be >= 1"):
        T.registry_lookup("diffusion", "iters=0")
    if O.have_ref():
        for s in ("", "iters=7,block=3", "iters= 9x,,"):
            r = O.ref_registry("diffusion", s)
            assert r["params_string"] == T.registry_lookup("diffusion", s).params_string()
            assert r["influence"] == T.registry_lookup("diffusion", s).influence_radius()
