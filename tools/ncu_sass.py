"""Per-instruction view of an ncu --set full capture (SASS page): stall samples, executed
instructions and shared-memory wavefronts summed per address range.

    python tools/ncu_sass.py gpurun_out/x.ncu-rep [kernel-substring] [0xSTART-0xEND ...]"""
import csv
import io
import subprocess
import sys


def load(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    raw = subprocess.run(cmd, capture_output=True, text=True).stdout
    lines = raw.splitlines()
    i = next(k for k, ln in enumerate(lines) if ln.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
    out = []
    for r in rows:
        try:
            addr = int(r["Address"], 16)
        except (ValueError, KeyError):
            continue
        f = lambda k: float(r.get(k) or 0)  # noqa: E731
        out.append({"addr": addr, "src": r["Source"], "samples": f("Warp Stall Sampling (All Samples)"),
                    "inst": f("Instructions Executed"), "wf": f("L1 Wavefronts Shared"),
                    "wf_ideal": f("L1 Wavefronts Shared Ideal")})
    base = min(r["addr"] for r in out) if out else 0
    for r in out:
        r["addr"] -= base  # kernel-relative, as cuobjdump -sass prints them
    return out


def main():
    rep = sys.argv[1]
    kernel = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("0x") else None
    ranges = [tuple(int(x, 16) for x in a.split("-")) for a in sys.argv[2:] if a.startswith("0x")]
    rows = load(rep, kernel)
    tot = {k: sum(r[k] for r in rows) for k in ("samples", "inst", "wf", "wf_ideal")}
    print("total", {k: f"{v:.4g}" for k, v in tot.items()})
    for (a, b) in ranges:
        sel = [r for r in rows if a <= r["addr"] < b]
        s = {k: sum(r[k] for r in sel) for k in ("samples", "inst", "wf", "wf_ideal")}
        print(f"{a:#x}-{b:#x}", {k: f"{v:.4g} ({v / max(tot[k], 1):.1%})" for k, v in s.items()})
    ops = {}
    for r in rows:
        op = r["src"].split()[0] if r["src"] else "?"
        if op.startswith("@"):
            op = r["src"].split()[1]
        op = op.split(".")[0]
        d = ops.setdefault(op, [0.0, 0.0, 0.0])
        d[0] += r["inst"]
        d[1] += r["samples"]
        d[2] += r["wf"]
    print("by opcode (inst, samples, wavefronts):")
    for op, (i, s_, w) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"  {op:10s} {i:12.4g} {s_:10.4g} {w:12.4g}")
    print("top instructions by samples:")
    for r in sorted(rows, key=lambda r: -r["samples"])[:25]:
        print(f"  {r['addr']:#06x} {r['samples']:8.0f} {r['inst']:10.4g} {r['wf']:10.4g}  {r['src'][:70]}")


if __name__ == "__main__":
    main()
