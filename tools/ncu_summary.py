"""Summaries committed under profiles/: key metrics of one ncu --set full capture, and the
per-kernel share of a `--metrics gpu__time_duration.sum` launch list.

    python tools/ncu_summary.py full  gpurun_out/x.ncu-rep  profiles/rN_ncu_..._summary.csv [first-n-launches]
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/rN_launches_....csv"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def full(rep, out, first=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "metric", "value", "unit"])
        for r in rows[2:2 + int(first)] if first else rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            for k in KEYS:
                if k in d:
                    w.writerow([d["Kernel Name"], k, d[k], u.get(k, "")])
            # FP64 flops the launch executed: (2 DFMA + DADD + DMUL) thread instructions, from
            # their per-elapsed-cycle rates x elapsed cycles (packed FP32 FFMA2/FADD2/FMUL2
            # have no thread-instruction counter here and are not included)
            try:
                rate = sum(m * float(d[f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"])
                           for op, m in (("dfma", 2), ("dadd", 1), ("dmul", 1)))
                dur = float(d["gpu__time_duration.sum"]) * {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(
                    u.get("gpu__time_duration.sum", "usecond"), 1e-6)
                hz = float(d["sm__cycles_elapsed.avg.per_second"]) * 1e9  # GHz
                w.writerow([d["Kernel Name"], "derived_fp64_flops", f"{rate * dur * hz:.6g}", "flop"])
            except (KeyError, ValueError):
                pass


def launches(src, out):
    lines = open(src).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in csv.DictReader(lines[i:]):
        if r["Metric Name"] == "gpu__time_duration.sum":
            tot[r["Kernel Name"]] += float(r["Metric Value"])
            cnt[r["Kernel Name"]] += 1
    s = sum(tot.values())
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ns", "mean_ns", "share_of_gpu_time"])
        for k in sorted(tot, key=lambda k: -tot[k]):
            w.writerow([k, cnt[k], f"{tot[k]:.0f}", f"{tot[k] / cnt[k]:.0f}", f"{tot[k] / s:.4f}"])


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](*sys.argv[2:])
