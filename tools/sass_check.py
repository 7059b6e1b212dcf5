"""profiles/rN_sass_fp64_check.txt: per FSE kernel, counts of FP32<->FP64 conversions, packed
FP32 and FP64 arithmetic in the built library's SASS (the FAST kernels must be binary64).

    python tools/sass_check.py > profiles/r2_sass_fp64_check.txt"""
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2207_00238_b200" / "_lib" / "libtframe_b200.so"
OPS = ["F2F.F64.F32", "F2F.F32.F64", "FFMA2", "FADD2", "FMUL2", "FFMA", "DFMA", "DMUL", "DADD", "DSETP"]
sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
print("# cuobjdump -sass paper_2207_00238_b200/_lib/libtframe_b200.so (round 2), per FSE kernel:")
print("# counts of FP32<->FP64 conversions, packed FP32 (FFMA2/FADD2/FMUL2), scalar FFMA and FP64 ops.")
print("# FAST kernels (fse_pair / fse_half / fse_wide, fse_block_kernel<..., false>) must show no")
print("# F2F.F64.F32 and no packed FP32: their arithmetic is binary64 throughout.")
print(f"{'kernel':70s} " + " ".join(f"{o:>11s}" if o.startswith("F2F") else f"{o:>5s}" for o in OPS))
cur, cnt = None, {}
def flush():
    if cur and "fse_" in cur:
        print(f"{cur:70s} " + " ".join(f"{cnt.get(o, 0):11d}" if o.startswith("F2F") else f"{cnt.get(o, 0):5d}" for o in OPS))
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        flush()
        cur, cnt = m.group(1), {}
        continue
    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_.]+)", ln)
    if m:
        op = m.group(1)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                cnt[o] = cnt.get(o, 0) + 1
                break
flush()
