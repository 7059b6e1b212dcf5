"""Per-instruction dump of one kernel of an ncu --set full capture (SASS page): address, executed
warp instructions, stall samples, shared-memory wavefronts, source text.

    python tools/ncu_dump.py gpurun_out/x.ncu-rep <launch-index> > dump.txt"""
import csv
import io
import subprocess
import sys

rep, skip = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = raw.splitlines()
print(lines[0])
i = next(k for k, ln in enumerate(lines) if ln.startswith('"Address"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[i:]))) if r["Address"].startswith("0x")]
base = int(rows[0]["Address"], 16)
for r in rows:
    print(f'{int(r["Address"], 16) - base:#07x} {float(r["Instructions Executed"] or 0):12.0f} '
          f'{float(r["Warp Stall Sampling (All Samples)"] or 0):8.0f} {float(r["L1 Wavefronts Shared"] or 0):12.0f}  '
          f'{r["Source"].strip()[:60]}')
