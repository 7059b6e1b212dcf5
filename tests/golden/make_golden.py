"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference (oracle/_ref/libtframe_ref.so, built from
/root/reference/proj/include by oracle/Makefile) on small inputs and stores
inputs + outputs.  Only this container can run it (the GPU box has no
/root/reference); the committed .npz files travel instead.

    make -C oracle ref && python tests/golden/make_golden.py

Fixture cases (reference test/acceptance files they mirror):
  kat_all_known      test_extrapolate.cpp:80-84   random 16x16, all known
  kat_constant       test_extrapolate.cpp:86-92   183-constant 24x24, gen_scatter_mask(24,24,0.25,3,5)
  kat_sinusoid       test_extrapolate.cpp:94-113  20x20, period-10 sinusoid, 4x4 hole at (8..11)
  kat_bandlimited    test_extrapolate.cpp:153-175 64x64 two-sinusoid truth, gen_scatter_mask(64,64,0.2,2,11)
  acc9_tiles6        acceptance.cpp:271-338       make_scene(96,80,21), gen_scatter_mask(96,80,0.4,3,22), 6 tiles d=12
  cfg{1..5}_small    BASELINE c1..c5 FSE params on small synthetic crops (generator v1), reference run_local
  tiling             plan_proposed + expand rects for the BASELINE configs and the (1024,480,22) layout
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from paper_2207_00238_b200 import tframe as T  # noqa: E402  (generator v1 for the cfg crops)
from paper_2207_00238_b200.configs import CONFIGS  # noqa: E402

DEF = dict(block=4, margin=8, iters=100, gamma=0.5, rho=0.8)  # FseLiteParams defaults


def fse_case(img, kn, tiles=1, overlap=0, **p):
    q = dict(DEF, **p)
    if tiles == 1 and overlap == 0:
        out, nb = O.ref_fse_lite(img, kn, q["block"], q["margin"], q["iters"], q["gamma"], q["rho"],
                                 count_blocks=True)
    else:
        out, _ = O.ref_run_local(img, kn, tiles, overlap, q["block"], q["margin"], q["iters"], q["gamma"],
                                 q["rho"], workers=min(tiles, 4))
        nb = -1
    return dict(img=img, known=kn, out=out, tiles=tiles, overlap=overlap, nblocks=nb,
                params=np.array([q["block"], q["margin"], q["iters"]], np.int32),
                fparams=np.array([q["gamma"], q["rho"]], np.float64))


def main():
    rng = np.random.default_rng(20220701)
    cases = {}
    img = rng.integers(0, 256, (16, 16), dtype=np.uint8)
    cases["kat_all_known"] = fse_case(img, np.ones_like(img))
    cases["kat_constant"] = fse_case(np.full((24, 24), 183, np.uint8), O.ref_gen_scatter_mask(24, 24, 0.25, 3, 5))
    x = np.arange(20)
    sin = np.round(128.0 + 60.0 * np.sin(2.0 * np.pi * x / 10.0)).astype(np.uint8)
    img = np.tile(sin, (20, 1))
    kn = np.ones((20, 20), np.uint8)
    kn[8:12, 8:12] = 0
    cases["kat_sinusoid"] = fse_case(img, kn)
    yy, xx = np.mgrid[0:64, 0:64]
    truth = np.clip(np.round(128.0 + 50.0 * np.sin(2 * np.pi * (3.0 * xx / 64)) +
                             30.0 * np.sin(2 * np.pi * (2.0 * yy / 64))), 0, 255).astype(np.uint8)
    cases["kat_bandlimited"] = fse_case(truth, O.ref_gen_scatter_mask(64, 64, 0.2, 2, 11))
    cases["acc9_tiles6"] = fse_case(O.ref_make_scene(96, 80, 21), O.ref_gen_scatter_mask(96, 80, 0.4, 3, 22),
                                    tiles=6, overlap=12)
    crops = {1: (128, 96, 1), 2: (160, 96, 4), 3: (96, 64, 8), 4: (160, 128, 8), 5: (128, 96, 1)}
    for c, (w, h, tiles) in crops.items():
        wl = CONFIGS[c]
        p = wl.params
        a, b = T.synth_frame(c, 0, w, h)
        cases[f"cfg{c}_small"] = fse_case(a, b, tiles=tiles, overlap=wl.overlap if tiles > 1 else 0,
                                          block=p.block_size, margin=p.support_margin,
                                          iters=p.model_iterations, gamma=p.compensation, rho=p.weight_decay)
    for name, d in cases.items():
        np.savez_compressed(HERE / f"{name}.npz", **d)
    # tiling goldens
    tl = {}
    for name, (W, H, N, d) in {"c1": (512, 512, 1, 14), "c2": (1920, 1080, 4, 12), "c3n2": (3840, 2160, 2, 6),
                               "c3n4": (3840, 2160, 4, 6), "c3n8": (3840, 2160, 8, 6), "c4": (7680, 4320, 8, 16),
                               "c4d14": (7680, 4320, 8, 14), "c5n8": (1920, 1080, 8, 16),
                               "ref1024x480x22": (1024, 480, 22, 32), "portrait480x1024x22": (480, 1024, 22, 32)}.items():
        cores = O.ref_plan_proposed(W, H, N)
        halos = np.stack([O.ref_expand(c, d, W, H) for c in cores])
        tl[name] = np.concatenate([np.array([[W, H, N, d]], np.int32), cores, halos])
        tl[name + "_ib"] = np.array([O.ref_interior_boundary(W, H, N)], np.int64)
    np.savez_compressed(HERE / "tiling.npz", **tl)
    print("wrote", len(cases), "fse fixtures + tiling.npz")


if __name__ == "__main__":
    main()
