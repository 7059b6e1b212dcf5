"""Reference-driven GPU workers: the reference's own run_master and
LocalTransport (compiled from its unmodified headers, integration/Makefile) with the
CudaFseLiteExtrapolator worker loop, against the same master with the stock CPU workers."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "integration" / "_build" / "ref_master_gpu_workers"


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,W,H,workers", [(2, 480, 270, 4), (2, 480, 270, 3), (3, 320, 180, 8),
                                             (1, 256, 256, 1)])
def test_reference_master_with_gpu_workers_is_byte_identical(cfg, W, H, workers):
    if not EXE.exists():
        pytest.skip("integration binary not built (needs the reference headers at build time)")
    r = subprocess.run([str(EXE), str(cfg), str(W), str(H), str(workers), "exact"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bytes_equal"], out


@pytest.mark.gpu
def test_reference_master_with_gpu_workers_fast_within_tolerance():
    if not EXE.exists():
        pytest.skip("integration binary not built")
    r = subprocess.run([str(EXE), "2", "480", "270", "4", "fast"], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["within1"] >= 0.999, out


@pytest.mark.gpu
def test_reference_master_with_gpu_diffusion_workers():
    if not EXE.exists():
        pytest.skip("integration binary not built")
    r = subprocess.run([str(EXE), "2", "480", "270", "4", "diffusion=20"], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bytes_equal"], out
