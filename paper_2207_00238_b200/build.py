"""Build the sm_100a C-ABI library (and, for tests, the CPU oracle).

    python -m paper_2207_00238_b200.build          # libtframe_b200.so
    python -m paper_2207_00238_b200.build --oracle # + oracle/liboracle.so (+ oracle/_ref if /root/reference exists)

The library is built IN-TREE (paper_2207_00238_b200/_lib/) so that it travels
with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libtframe_b200.so"
SOURCES = ["fse_kernels.cu", "diffusion.cu", "metrics.cu", "capi.cpp", "tiling.cpp", "synth.cpp", "calibrate.cu"]
HEADERS = ["fse_kernels.cuh", "host_internal.hpp", "synth_gen.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False, out: Path | None = None,
              defines: tuple[str, ...] = ()) -> Path:
    """Build libtframe_b200.so (or a tuning variant at `out` with extra -D defines)."""
    target = out or LIB
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "tframe_fse.h", Path(__file__)]
    if not force and not _stale(target, deps):
        return target
    target.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = target.parent / (target.stem + "." + src.rsplit(".", 1)[0] + ".o")
        cmd = [NVCC, *ARCH, *[f"-D{d}" for d in defines], "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "-I", str(ROOT / "include"),
               "-c", str(CSRC / src), "-o", str(obj)]
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    target.parent.mkdir(parents=True, exist_ok=True)
    tmp = target.with_suffix(".so.tmp")
    subprocess.run([NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-ldl"], check=True)
    os.replace(tmp, target)
    for o in objs:
        os.remove(o)
    return target


def build_oracle(with_ref: bool | None = None) -> None:
    """Test infrastructure: the C restatement, and the compiled reference shim
    when /root/reference is present (this container; the GPU box uses the
    prebuilt oracle/_ref/libtframe_ref.so that travels with the snapshot)."""
    odir = ROOT / "oracle"
    subprocess.run(["make", "-s", "-C", str(odir), "liboracle.so"], check=True)
    ref_inc = Path(os.environ.get("TF_REF_INCLUDE", "/root/reference/proj/include"))
    if with_ref is None:
        with_ref = ref_inc.exists()
    if with_ref:
        subprocess.run(["make", "-s", "-C", str(odir), "ref", f"REF_INCLUDE={ref_inc}"], check=True)


def build_integration() -> None:
    """The reference's run_master driving GPU workers (integration/): built
    only where the reference headers exist; the binary travels to the GPU box."""
    ref_inc = Path(os.environ.get("TF_REF_INCLUDE", "/root/reference/proj/include"))
    if ref_inc.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "integration"), f"REF_INCLUDE={ref_inc}"],
                       check=True)


if __name__ == "__main__":
    if "--variant" in sys.argv:  # --variant NAME DEF1 DEF2 ... (tuning builds under _lib/variants/)
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], tuple(sys.argv[i + 2:])
        print(build_lib(force=True, out=LIBDIR / "variants" / f"{name}.so", defines=defs))
        sys.exit(0)
    build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv)
    if "--oracle" in sys.argv:
        build_oracle()
        build_integration()
    print(LIB)
