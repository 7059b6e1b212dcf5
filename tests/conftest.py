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


@pytest.fixture
def tune_env(monkeypatch):
    """Set tuning variables (TF_STREAM_BANDS, TF_HYBRID, ...) for some contexts: the library
    reads them once per context (tf_create / tf_set_mode), so the contexts re-read them
    (Context.reload_tuning) now and again after the environment is restored."""
    touched = []

    def set_env(ctxs, **env):
        for k, v in env.items():
            if v is None:
                monkeypatch.delenv(k, raising=False)
            else:
                monkeypatch.setenv(k, str(v))
        for c in ctxs:
            c.reload_tuning()
            touched.append(c)

    yield set_env
    monkeypatch.undo()
    for c in touched:
        if c._h:
            c.reload_tuning()
