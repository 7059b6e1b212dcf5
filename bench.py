#!/usr/bin/env python
"""Benchmark of the B200 FSE-lite hot path (BASELINE.json metric: reconstructed Mpixel/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode exact|fast]

Workload = BASELINE configs[1] (= SURVEY config c2): one 1920x1080 u8 frame,
8x8 aligned cell loss p=0.10, FSE block 8 / border 12 (32x32 window = DFT),
200 iterations, rho 0.8, gamma 0.5, tiled into 4 overlapping tiles (d = 12).
A "step" is one pass of the hot path over one frame per GPU.

N > 1 (torchrun, one process per GPU): every rank reconstructs its own frame
(per-rank seed) and the frames are gathered to rank 0 with NCCL over NVLink
(weak scaling; the gather is inside the timed region).

value  : device path, inputs resident in HBM (tf_tiled_extrapolate_device),
         L2 flushed between steps (a 256 MiB write outside the timed events), in the
         headline mode (default FAST: FMA + Hermitian half spectrum, within the north-star
         tolerance, checked on this very frame and reported under "parity"); the EXACT
         mode (byte-identical to the reference, also checked here) is timed and reported.
e2e    : the same through the public host-buffer call (tf_tiled_extrapolate on pinned
         HOST buffers): H2D of image + mask, FSE, D2H of the result inside the call
         (streamed in row bands so copies overlap the kernels), every rank its own frame.
roofline: FP64-bound kernels; achieved = executed FP64 flops per launch (== the
         SURVEY §8(d) algorithmic sum_b F_b in EXACT mode) / mean FSE time (CUDA events
         on the launch stream), peak = FP64 DFMA rate measured live (tf_calibrate).
--impl reference: the reference CPU FSE (oracle/_ref: the unmodified tframe
         headers compiled by oracle/Makefile), all host threads, same frame.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG = 2  # BASELINE configs[1]
METRIC = "reconstructed Mpixel/s (FSE, 1/2/4/8 B200) and % of FLOP roofline vs CPU ref"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def make_frames(wl, frame):
    from paper_2207_00238_b200 import tframe as T
    return T.synth_frame(wl.config, frame, wl.W, wl.H)


def cpu_reference(wl, img, kn, steps, warmup, threads=None):
    """The reference's own FSE (oracle/_ref, unmodified tframe headers), bit-exact
    band split over all host threads.  Returns (Mpix/s, out, info)."""
    import oracle as O
    p = wl.params
    threads = threads or os.cpu_count() or 1
    args = (wl.tiles, wl.overlap, p.block_size, p.support_margin, p.model_iterations,
            p.compensation, p.weight_decay)
    out = None
    for _ in range(warmup):
        out = O.ref_tiled_allcores(img, kn, *args, threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out = O.ref_tiled_allcores(img, kn, *args, threads=threads)
        times.append(time.perf_counter() - t0)
    mean = sum(times) / len(times)
    return wl.W * wl.H / mean / 1e6, out, {"threads": threads, "s_per_frame": mean}


def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    from paper_2207_00238_b200 import tframe as T  # noqa: F401  (synthetic generator only)
    import oracle as O
    if not O.have_ref():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libtframe_ref.so not built (needs /root/reference at build time)"}))
        return
    img, kn = make_frames(wl, 0)
    steps, warmup = max(1, args.steps), max(0, min(args.warmup, 1))
    v, _, info = cpu_reference(wl, img, kn, steps, warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "Mpixel/s",
        "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": round(info["s_per_frame"] * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.describe(), "frames_per_step": 1},
        "cpu_baseline": {"value": round(v, 3), "unit": "Mpixel/s", "cores": info["threads"],
                         "kind": "reference",
                         "sample": f"full c{wl.config} frame per step ({wl.W}x{wl.H}, {wl.tiles} tiles, d={wl.overlap}), "
                                   "bit-exact B-aligned band split over all host threads"},
        "e2e": {"value": round(v, 3), "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ncu_profile(mode, config=CONFIG):
    """DRAM bytes (read + write) per launch of the FSE kernels and their shared-memory
    wavefront utilisation, from the committed `ncu --set full` summary of this workload
    (profiles/rNN_ncu_fse_c2_<mode>_summary.csv, written by tools/ncu_summary.py)."""
    import csv
    import glob
    files = sorted(glob.glob(str(ROOT / "profiles" / f"r*_ncu_*_c{config}_{mode}_summary.csv")))
    if not files:
        return {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic, smem, found, fp64, pipe = 0.0, [], False, None, []
    with open(files[-1]) as f:
        rows = list(csv.DictReader(f))
    for r in rows:
        if "kernel" not in r or "fse" not in r["kernel"]:
            continue
        if r["metric"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            traffic += float(r["value"]) * scale.get(r["unit"], 1)
            found = True
        if r["metric"] == "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed":
            smem.append(round(float(r["value"]), 1))
        if r["metric"] == "derived_fp64_flops":
            fp64 = (fp64 or 0.0) + float(r["value"])
        if r["metric"] == "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active":
            pipe.append(round(float(r["value"]), 1))
    if not found:
        return {}
    return {"traffic": int(traffic), "smem_pct": smem, "source": Path(files[-1]).name,
            "fp64_flops": fp64, "fp64_pipe_pct": pipe}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default=os.environ.get("TF_BENCH_MODE", "fast"), choices=["exact", "fast"],
                    help="headline arithmetic mode; the other mode is timed and reported too")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", type=int, default=CONFIG, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config (default 2, the one the metric is quoted on; the others "
                         "for the per-config evidence in profiles/)")
    args = ap.parse_args()

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)

    from paper_2207_00238_b200.configs import workload
    wl = workload(args.config)

    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2207_00238_b200 import _native as N
    from paper_2207_00238_b200 import tframe as T
    import ctypes as C

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    sptr = stream.cuda_stream

    ctx = T.Context(1, [local], args.mode)
    L = N.lib()
    if world > 1:
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            N.check(L.tf_comm_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        N.check(L.tf_comm_init(ctx.handle, world, rank, uid))

    # ---- inputs: this rank's frame (seeded per rank), pinned host + HBM copies
    img_np, kn_np = make_frames(wl, rank)
    H, W = img_np.shape
    fb = W * H
    h_img = torch.from_numpy(img_np.reshape(-1)).pin_memory()
    h_kn = torch.from_numpy(kn_np.reshape(-1)).pin_memory()
    d_img = h_img.to(dev)
    d_kn = h_kn.to(dev)
    d_out = torch.empty_like(d_img)
    d_all = torch.empty(world * fb, dtype=torch.uint8, device=dev) if (world > 1 and rank == 0) else None
    h_res = torch.empty(fb, dtype=torch.uint8).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    p = wl.params._c()

    def device_step():
        N.check(L.tf_tiled_extrapolate_device(ctx.handle, 0, d_img.data_ptr(), d_kn.data_ptr(), W, H, 1,
                                              wl.tiles, wl.overlap, C.byref(p), 0, 1, d_out.data_ptr(),
                                              sptr, None))
        if world > 1:
            N.check(L.tf_comm_gather(ctx.handle, d_out.data_ptr(),
                                     d_all.data_ptr() if d_all is not None else None, fb, 0, sptr))

    def e2e_step():
        # the call a user makes: tf_tiled_extrapolate on pinned HOST buffers (the library
        # streams row bands: H2D, FSE and D2H overlap inside the call); every rank
        # reconstructs its own frame into its own host memory
        N.check(L.tf_tiled_extrapolate(ctx.handle, h_img.data_ptr(), h_kn.data_ptr(), W, H, 1, wl.tiles,
                                       wl.overlap, C.byref(p), h_res.data_ptr(), None))

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(step_fn, k, host_api=False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier()
        for i in range(k):
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xff)          # L2 flush, outside the timed events
                if host_api:
                    # the host-buffer call runs on the library's own streams: let the flush
                    # finish first so it neither overlaps nor competes with the timed call
                    stream.synchronize()
                evs[i][0].record(stream)
            step_fn()
            with torch.cuda.stream(stream):
                evs[i][1].record(stream)
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    other = "exact" if args.mode == "fast" else "fast"

    def run_mode(mode):
        """Warm up + time the device path in `mode`; returns timing, kernel times, stats, output."""
        ctx.set_mode(mode)
        for _ in range(max(3, args.warmup)):
            device_step()
        barrier()
        out = d_out.cpu().numpy().reshape(H, W).copy()
        assert np.array_equal(out[kn_np != 0], img_np[kn_np != 0]), "known pixels not preserved"
        with ClockSampler(local) as clk:
            ms = timed(device_step, args.steps)
        kt = (C.c_float * args.steps)()
        nk = L.tf_fse_kernel_times(ctx.handle, 0, kt, args.steps)
        st = ctx.tiled_device(d_img.data_ptr(), d_kn.data_ptr(), d_out.data_ptr(), W, H, 1, wl.tiles,
                              wl.overlap, wl.params, stream=sptr, want_stats=True)
        fse = [kt[i] for i in range(max(nk, 0))]
        return {"ms_step": ms / args.steps, "fse_ms": sum(fse) / len(fse) if fse else st.kernel_ms,
                "stats": st, "out": out, "clocks": clk.summary()}

    res_other = run_mode(other)
    res = run_mode(args.mode)  # headline mode last: the context stays in it for e2e
    ms_step = res["ms_step"]
    value = world * fb / (ms_step * 1e-3) / 1e6

    # ---- e2e through the C-ABI with host buffers (headline mode)
    for _ in range(2):
        e2e_step()
    ms_e2e = timed(e2e_step, args.steps, host_api=True) / args.steps
    e2e = world * fb / (ms_e2e * 1e-3) / 1e6

    # ---- roofline of the headline FSE launch: executed FP64 flops (== the algorithmic
    # sum_b F_b for EXACT; the FAST half-spectrum kernel executes ~1/3 of it, SURVEY §8(d)
    # says to use executed flops then) / mean FSE kernel time; peak = live DFMA calibration
    fp64 = C.c_double(0)
    smem = C.c_double(0)
    N.check(L.tf_calibrate(local, C.byref(fp64), C.byref(smem)))
    st = res["stats"]
    mean_k = res["fse_ms"]
    achieved = st.flops_executed / (mean_k * 1e-3) / 1e12
    prof = ncu_profile(args.mode, args.config)
    roof = {"bound": "fp64", "achieved": round(achieved, 3), "peak": round(fp64.value, 3),
            "unit": "TFLOP/s", "frac": round(achieved / fp64.value, 4),
            "traffic": prof.get("traffic"),
            "traffic_source": prof.get("source"),
            "smem_wavefront_pct_of_peak_ncu": prof.get("smem_pct"),
            # FP64-only view from the committed ncu capture: FP64 flops the FSE kernels
            # executed (packed FP32 excluded) over this run's FSE time, and the FP64 pipe's
            # utilisation per kernel — the kernels are latency/issue-bound, not FP64-pipe-bound
            "ncu_fp64_flops_per_launch": prof.get("fp64_flops"),
            "ncu_fp64_tflops": (round(prof["fp64_flops"] / (mean_k * 1e-3) / 1e12, 3)
                                if prof.get("fp64_flops") else None),
            "fp64_pipe_pct_of_peak_ncu": prof.get("fp64_pipe_pct"),
            "peak_source": "FP64 DFMA rate measured live by tf_calibrate (MEASURED_PEAKS.json has no FP64 figure)",
            "fse_kernel_ms": round(mean_k, 4), "flops_executed_per_launch": st.flops_executed,
            "flops_algorithmic_per_launch": st.flops,
            "algorithmic_tflops": round(st.flops / (mean_k * 1e-3) / 1e12, 3),
            "smem_peak_tbs": round(smem.value, 2),
            "kernel_share_of_step": round(mean_k / ms_step, 3)}

    # ---- parity of this run: FAST vs EXACT (north-star tolerance), EXACT vs the reference
    ex_out = res["out"] if args.mode == "exact" else res_other["out"]
    fa_out = res["out"] if args.mode == "fast" else res_other["out"]
    unk = kn_np == 0
    dd = np.abs(ex_out.astype(int) - fa_out.astype(int))[unk]

    # PSNR / SSIM against the ground truth on the GPU (tf_quality: bit-identical to metrics.hpp)
    qe, qf = ctx.quality(np.stack([img_np, img_np]), np.stack([ex_out, fa_out]), np.stack([kn_np, kn_np]))

    parity = {"fast_within1_of_exact": round(float((dd <= 1).mean()), 6),
              "fast_max_abs_diff": int(dd.max()) if dd.size else 0,
              "psnr_exact_db": round(qe["psnr"], 4), "psnr_fast_db": round(qf["psnr"], 4),
              "ssim_exact": round(qe["ssim"], 6), "ssim_fast": round(qf["ssim"], 6),
              "psnr_missing_exact_db": round(qe["psnr_missing"], 4),
              "psnr_missing_fast_db": round(qf["psnr_missing"], 4),
              "metrics_source": "GPU tf_quality (metrics.hpp restated)",
              "tolerance": ">= 0.999 within +-1 and |dPSNR| <= 0.05 dB (north star)"}
    parity["fast_dpsnr_db"] = round(abs(parity["psnr_exact_db"] - parity["psnr_fast_db"]), 5)
    parity["fast_within_tolerance"] = bool(parity["fast_within1_of_exact"] >= 0.999 and parity["fast_dpsnr_db"] <= 0.05)

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (versioned generator v1, per-rank seed 1000*{wl.config}+rank)",
        "config": {"workload": wl.describe(), "frames_per_gpu_per_step": 1, "mode": args.mode,
                   "l2": "flushed between steps (256 MiB write outside the timed events)",
                   "parallelism": f"dp{world} frames, NCCL gather to rank 0" if world > 1 else "single GPU",
                   "blocks_processed": st.blocks_processed, "blocks_reference": st.blocks_reference},
        "e2e": {"value": round(e2e, 3), "unit": "Mpixel/s", "ms_per_step": round(ms_e2e, 4),
                "h2d_bytes_per_step": 2 * fb, "d2h_bytes_per_step": fb,
                "path": "tf_tiled_extrapolate (host buffers, streamed row bands), per rank"},
        # per step, FAST: enumerate + half-spectrum FSE + border-window (GEN) FSE + the hybrid's
        # EXACT kernel (empty list on c2); EXACT: enumerate + CTA FSE
        "gpu_launches": args.steps * (4 if args.mode == "fast" else 2),
        "roofline": roof,
        "clocks": res["clocks"],
        other + "_mode": {"value": round(world * fb / (res_other["ms_step"] * 1e-3) / 1e6, 3),
                          "ms_per_step": round(res_other["ms_step"], 4),
                          "fse_kernel_ms": round(res_other["fse_ms"], 4)},
        "parity": parity,
    }

    # ---- CPU baseline: rank 0, N = 1 only, the reference on the host cores
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            if O.have_ref():
                v, ref_out, info = cpu_reference(wl, img_np, kn_np, 1, 0)
                line["cpu_baseline"] = {
                    "value": round(v, 3), "unit": "Mpixel/s", "cores": info["threads"],
                    "kind": "reference",
                    "sample": f"one full c{wl.config} frame ({W}x{H}), reference FSE-lite via bit-exact band split",
                }
                line["parity"]["exact_bytes_equal_reference"] = bool(np.array_equal(ref_out, ex_out))
                dr = np.abs(ref_out.astype(int) - fa_out.astype(int))[unk]
                line["parity"]["fast_within1_of_reference"] = round(float((dr <= 1).mean()), 6)
            else:
                line["cpu_baseline"] = None
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
