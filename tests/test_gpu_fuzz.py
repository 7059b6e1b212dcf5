"""Randomised parity sweep on the GPU (tools/fuzz_parity.py): random shapes, block sizes
2-16, margins 0-16, iterations, gamma, rho, tiles, overlap, frames and four mask families
(i.i.d. pixels, aligned cells, disks, almost nothing known).  EXACT must equal the C oracle
byte for byte and match its block counts in every case; FAST (with its EXACT hybrid) must
keep >= 99.9 % of the reconstructed pixels within +-1 of EXACT over the sweep."""
import importlib.util
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _fuzz():
    spec = importlib.util.spec_from_file_location("fuzz_parity", ROOT / "tools" / "fuzz_parity.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [101, 202])
def test_randomised_parity_sweep(seed):
    from paper_2207_00238_b200 import tframe as T
    ex, fa = T.Context(1, [0], "exact"), T.Context(1, [0], "fast")
    try:
        bad, within1 = _fuzz().run(60, seed, ex, fa, verbose=False)
    finally:
        ex.close()
        fa.close()
    assert bad == 0
    assert within1 >= 0.999, within1
