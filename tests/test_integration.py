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


TCP_EXE = ROOT / "integration" / "_build" / "ref_tcp_gpu_workers"


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("workers,cfg,W,H", [(2, 2, 480, 270), (3, 3, 320, 180)])
def test_reference_tcp_master_with_gpu_workers_in_process(workers, cfg, W, H):
    """The reference's TcpMasterTransport + TcpWorkerEndpoint (TFRM frames over loopback
    sockets) with GPU worker loops: byte-identical to the stock CPU workers."""
    if not TCP_EXE.exists():
        pytest.skip("integration binary not built")
    r = subprocess.run([str(TCP_EXE), "selftest", str(_free_port()), str(workers), str(cfg), str(W), str(H),
                        "exact"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bytes_equal"], out


@pytest.mark.gpu
def test_reference_tcp_master_with_gpu_worker_processes():
    """Separate worker processes (one per GPU / box in a deployment) connecting to the
    reference's master over TCP."""
    if not TCP_EXE.exists():
        pytest.skip("integration binary not built")
    port = _free_port()
    master = subprocess.Popen([str(TCP_EXE), "master", str(port), "2", "2", "480", "270", "exact"],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    workers = [subprocess.Popen([str(TCP_EXE), "worker", f"127.0.0.1:{port}", "0", "exact"],
                                stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for _ in range(2)]
    try:
        out, err = master.communicate(timeout=120)
        for w in workers:
            w.wait(timeout=60)
    finally:
        for p in [master, *workers]:
            if p.poll() is None:
                p.kill()
    assert master.returncode == 0, err
    assert all(w.returncode == 0 for w in workers), [w.stderr.read() for w in workers]
    res = json.loads(out.strip().splitlines()[-1])
    assert res["bytes_equal"] and res["transport"] == "tcp", res
