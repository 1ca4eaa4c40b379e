import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def _build_libme():
    """Build libme.so before any test imports the package (whose import loads
    it); build.py is loaded by path so a fresh tree can build."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_me_build", ROOT / "paper_2411_06465_b200" / "build.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()
    if os.environ.get("ME_CHECKED") == "1":
        b.build(checked=True)


def pytest_configure(config):
    _build_libme()
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through libme.so)")
    config.addinivalue_line("markers", "slow: long-running (full-space oracle walks)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle
