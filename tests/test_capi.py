"""The C-ABI library loads on a CPU host, exports every symbol the header
declares, and refuses to compute without a GPU (no CPU fallback)."""
import re

import numpy as np
import pytest

from paper_2207_00238_b200 import _native as N
from paper_2207_00238_b200 import tframe as T
from paper_2207_00238_b200.configs import CONFIGS


def header_functions():
    text = N.HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tf_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    names = header_functions()
    assert len(names) >= 25
    L = N.lib()
    for n in names:
        assert hasattr(L, n), f"{n} not exported"
        assert n in N.SIGNATURES, f"{n} has no ctypes signature"
    assert set(N.SIGNATURES) == set(names)
    assert L.tf_abi_version() == 2


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = N.lib().tf_create(1, None)
    assert not h
    assert "device" in N.last_error().lower() or "cuda" in N.last_error().lower()
    with pytest.raises(N.TframeError):
        T.Context(1)


def test_synth_generator_is_deterministic_and_matches_config_shapes():
    a1, k1 = T.synth_frame(2, 0, 192, 108)
    a2, k2 = T.synth_frame(2, 0, 192, 108)
    assert np.array_equal(a1, a2) and np.array_equal(k1, k2)
    b, _ = T.synth_frame(2, 1, 192, 108)
    assert not np.array_equal(a1, b)
    # loss fractions roughly as specified (c1 cells .25, c2 .10, c3 iid .20)
    for c, p in ((1, 0.25), (2, 0.10), (3, 0.20)):
        _, kn = T.synth_frame(c, 0, 512, 512)
        assert abs((kn == 0).mean() - p) < 0.05, c
    _, kn = T.synth_frame(5, 0, 480, 270)
    assert (kn == 0).mean() > 0.25  # cells + >=10% disks
    # c2 loss is aligned 8x8 cells: every 8x8 cell is all-known or all-lost
    _, kn = T.synth_frame(2, 0, 64, 64)
    cells = kn.reshape(8, 8, 8, 8).transpose(0, 2, 1, 3).reshape(64, 64)
    assert all(c.min() == c.max() for c in cells)


def lpt_owners(cost, parts):
    """LPT restated: units by cost descending (ties: lower index first), each to the least
    loaded part (ties: lowest part) -- capi.cpp assign_owners."""
    order = sorted(range(len(cost)), key=lambda i: (-int(cost[i]), i))
    load = [0] * parts
    own = [0] * len(cost)
    for u in order:
        q = min(range(parts), key=lambda j: (load[j], j))
        own[u] = q
        load[q] += int(cost[u])
    return own


def test_core_layout_lpt_equal_costs_is_round_robin():
    """Equal core areas (c3: 8 tiles of 960x1080) give the reference's i mod n (runtime.hpp:102)."""
    for parts in (1, 2, 4, 8):
        own = np.zeros(8, np.int32)
        N.check(N.lib().tf_core_layout(3840, 2160, 1, 8, parts, None, None, own.ctypes.data, None, None))
        assert list(own) == [t % parts for t in range(8)]


def test_core_layout_partitions_every_tile_once():
    for frames, tiles, parts in ((1, 4, 1), (2, 4, 3), (3, 6, 8)):
        n = frames * tiles
        cores = (N.tf_rect * n)()
        fr = np.zeros(n, np.int32)
        own = np.zeros(n, np.int32)
        offs = np.zeros(n, np.int64)
        pb = np.zeros(parts, np.int64)
        N.check(N.lib().tf_core_layout(64, 48, frames, tiles, parts, cores, fr.ctypes.data,
                                       own.ctypes.data, offs.ctypes.data, pb.ctypes.data))
        area = np.array([c.w * c.h for c in cores])
        assert list(own) == lpt_owners(area, parts)
        load = np.bincount(own, weights=area, minlength=parts)
        assert load.max() - load.min() <= area.max()  # LPT balance bound
        assert pb.sum() == 64 * 48 * frames
        for p in range(parts):
            sel = np.where(own == p)[0]
            assert sorted(offs[sel]) == list(np.cumsum(np.r_[0, area[sel]])[:-1])


def test_configs_table():
    assert CONFIGS[2].tiles == 4 and CONFIGS[2].overlap == 12
    assert CONFIGS[2].params.support_margin == 12 and CONFIGS[2].params.model_iterations == 200
    assert CONFIGS[5].frames == 64


def test_cpp_adapter_header_compiles_and_runs(tmp_path):
    """include/tframe_b200.hpp (the C++ mirror of the reference interface) builds against the
    library and behaves like the reference on host-only calls."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("no g++")
    root = N.LIB_PATH.parent.parent.parent
    exe = tmp_path / "adapter_smoke"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", str(root / "include"),
                    str(root / "tests" / "cpp" / "adapter_smoke.cpp"), "-o", str(exe),
                    "-L", str(N.LIB_PATH.parent), "-ltframe_b200",
                    f"-Wl,-rpath,{N.LIB_PATH.parent}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
