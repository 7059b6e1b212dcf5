"""Randomised parity sweep (test infrastructure; tests/test_gpu_fuzz.py runs it): N random
cases over image shape, block size, margin, iterations, gamma, rho, tiles, overlap, frames
and six mask families (i.i.d. pixels, aligned cells, disks, almost nothing known, cell losses
with margins 0-2, c4-style scratch lines).  EXACT through the GPU must equal the C oracle
byte for byte with equal block counts; FAST must meet the north-star tolerance PER CASE
(>= 99.9 % of the reconstructed pixels within +-1 of EXACT and |dPSNR vs the truth| <= 0.05
dB).  Any FAST/EXACT difference is reported with the argmax-gap diagnosis of the blocks it
sits in (the oracle's smallest relative |R|^2 gap between the winner and the runner-up over
the block's iterations, and the iteration where it occurred; extrapolate.hpp:146-155).
    python tools/fuzz_parity.py [N=300] [seed=1]"""
import sys

sys.path.insert(0, '.')
import numpy as np

import oracle as O
from paper_2207_00238_b200 import tframe as T

WITHIN1 = 0.999
DPSNR_DB = 0.05


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(255.0 ** 2 / mse)


def make_case(rng):
    B = int(rng.choice([2, 3, 4, 5, 8, 16]))
    margin = int(rng.choice([0, 1, 2, 4, 6, 8, 12, 14, 16]))
    kind = int(rng.integers(0, 6))
    if kind == 4:
        margin = int(rng.integers(0, 3))
    if B + 2 * margin > 64:
        margin = (64 - B) // 2
    iters = int(rng.integers(1, 80))
    gamma = float(rng.uniform(0.1, 1.0))
    rho = float(rng.uniform(0.5, 0.95))
    W, H = int(rng.integers(8, 260)), int(rng.integers(8, 200))
    frames = int(rng.integers(1, 3))
    tiles = int(rng.integers(1, 7))
    overlap = int(rng.integers(0, 20))
    img = rng.integers(0, 256, (frames, H, W), dtype=np.uint8)
    yy, xx = np.mgrid[0:H, 0:W]
    img = np.clip(img // 4 + (96 + 60 * np.sin(xx / rng.uniform(3, 20)) * np.cos(yy / rng.uniform(3, 20))).astype(np.uint8), 0, 255).astype(np.uint8)
    if kind == 0:
        kn = (rng.random((frames, H, W)) > rng.uniform(0.05, 0.5)).astype(np.uint8)
    elif kind in (1, 4):
        c = int(rng.choice([4, 8, 16])) if kind == 1 else B
        cells = rng.random((frames, (H + c - 1) // c, (W + c - 1) // c)) > rng.uniform(0.1, 0.4)
        kn = np.repeat(np.repeat(cells, c, 1), c, 2)[:, :H, :W].astype(np.uint8)
    elif kind == 2:
        kn = np.ones((frames, H, W), np.uint8)
        for f in range(frames):
            for _ in range(int(rng.integers(1, 4))):
                cy, cx, r = rng.integers(0, H), rng.integers(0, W), rng.integers(3, 40)
                kn[f][(yy - cy) ** 2 + (xx - cx) ** 2 < r * r] = 0
    elif kind == 3:
        kn = (rng.random((frames, H, W)) > 0.97).astype(np.uint8)  # almost nothing known
    else:  # scratches: straight lines of width 1-3 (config 4's mask family)
        kn = np.ones((frames, H, W), np.uint8)
        for f in range(frames):
            for _ in range(int(rng.integers(1, 6))):
                x0, y0 = rng.uniform(0, W), rng.uniform(0, H)
                th, ln, pen = rng.uniform(0, np.pi), rng.uniform(10, 300), int(rng.integers(1, 4))
                t = np.arange(0, ln, 0.5)
                px = np.floor(x0 + t * np.cos(th)).astype(int)
                py = np.floor(y0 + t * np.sin(th)).astype(int)
                for j in range(pen):
                    for i in range(pen):
                        X, Y = px + i, py + j
                        ok = (X >= 0) & (X < W) & (Y >= 0) & (Y < H)
                        kn[f, Y[ok], X[ok]] = 0
    if frames == 1:
        img, kn = img[0], kn[0]
    return dict(img=img, kn=kn, B=B, m=margin, I=iters, g=gamma, r=rho, tiles=tiles, d=overlap, kind=kind,
                W=W, H=H, f=frames)


def divergence_report(c, ex, fa):
    """Blocks whose FAST output differs from EXACT, with the oracle's argmax-gap diagnosis."""
    imgs = c["img"] if c["f"] > 1 else c["img"][None]
    kns = c["kn"] if c["f"] > 1 else c["kn"][None]
    exs = ex if c["f"] > 1 else ex[None]
    fas = fa if c["f"] > 1 else fa[None]
    out = []
    cores = T.plan_proposed(c["W"], c["H"], c["tiles"])
    for f in range(c["f"]):
        diff = exs[f] != fas[f]
        if not diff.any():
            continue
        for core in cores.tiles:
            e = T.expand(core, c["d"], c["W"], c["H"])
            h = e.halo
            sub = diff[core.y:core.y + core.h, core.x:core.x + core.w]
            if not sub.any():
                continue
            _, st = O.fse_lite(imgs[f, h.y:h.y + h.h, h.x:h.x + h.w], kns[f, h.y:h.y + h.h, h.x:h.x + h.w],
                               c["B"], c["m"], c["I"], c["g"], c["r"], with_stats=True)
            ys, xs = np.nonzero(sub)
            blocks = {((core.x + x - h.x) // c["B"] * c["B"], (core.y + y - h.y) // c["B"] * c["B"])
                      for y, x in zip(ys, xs)}
            for s in st:
                if (int(s["bx"]), int(s["by"])) in blocks:
                    out.append(dict(frame=f, tile=(core.x, core.y), bx=int(s["bx"]), by=int(s["by"]),
                                    window=(int(s["M"]), int(s["L"])), min_gap=float(s["min_gap"]),
                                    gap_iter=int(s["gap_iter"]), iters=int(s["iters"])))
    return out


def run(n, seed, ex_ctx=None, fa_ctx=None, verbose=True):
    """Returns a list of per-case records (dict): exact_ok, within1, dpsnr, n_unknown,
    divergences (blocks) and the case parameters."""
    rng = np.random.default_rng(seed)
    ex_ctx = ex_ctx or T.Context(1, [0], "exact")
    fa_ctx = fa_ctx or T.Context(1, [0], "fast")
    recs = []
    for case in range(n):
        c = make_case(rng)
        p = T.FseLiteParams(c["B"], c["m"], c["I"], c["g"], c["r"])
        try:
            want, bpt = O.tiled(c["img"], c["kn"], c["tiles"], c["d"], c["B"], c["m"], c["I"], c["g"], c["r"])
        except O.OracleError:
            continue  # degenerate tiling: the GPU path raises too (tests/test_tiling.py)
        ex, st = ex_ctx.tiled(c["img"], c["kn"], c["tiles"], c["d"], p)
        fa, _ = fa_ctx.tiled(c["img"], c["kn"], c["tiles"], c["d"], p)
        u = c["kn"] == 0
        dd = np.abs(ex.astype(int) - fa.astype(int))[u]
        within1 = float((dd <= 1).mean()) if dd.size else 1.0
        pe, pf = psnr(ex, c["img"]), psnr(fa, c["img"])
        dpsnr = 0.0 if pe == pf else abs(pe - pf)
        rec = dict(case=case, exact_ok=bool(np.array_equal(ex, want) and st.blocks_reference == int(bpt.sum())),
                   within1=within1, dpsnr=dpsnr, n_unknown=int(dd.size), n_diff=int((dd > 0).sum()),
                   max_diff=int(dd.max()) if dd.size else 0,
                   params={k: (round(v, 3) if isinstance(v, float) else v) for k, v in c.items()
                           if k not in ("img", "kn")})
        rec["divergences"] = divergence_report(c, ex, fa) if rec["n_diff"] else []
        recs.append(rec)
        if verbose and (not rec["exact_ok"] or rec["n_diff"]):
            print(f"case {case}: exact_ok={rec['exact_ok']} within1={within1:.5f} dPSNR={dpsnr:.2e} "
                  f"diff={rec['n_diff']}/{rec['n_unknown']} {rec['params']}", flush=True)
            for dv in rec["divergences"][:4]:
                print(f"    block {dv}", flush=True)
    if verbose:
        bad = sum(not r["exact_ok"] for r in recs)
        worst = min((r["within1"] for r in recs), default=1.0)
        print(f"{len(recs)} cases: EXACT mismatches {bad}; FAST worst within +-1 {worst:.6f}, worst dPSNR "
              f"{max((r['dpsnr'] for r in recs), default=0):.2e} dB, cases with any difference "
              f"{sum(1 for r in recs if r['n_diff'])}")
    return recs


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 300, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
