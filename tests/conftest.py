import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU check")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the CPU oracle once per session (no-op when fresh)."""
    from paper_2207_00238_b200 import build

    build.build_lib()
    build.build_oracle(with_ref=Path(os.environ.get("TF_REF_INCLUDE", "/root/reference/proj/include")).exists()
                       and not (ROOT / "oracle" / "_ref" / "libtframe_ref.so").exists())
    yield
