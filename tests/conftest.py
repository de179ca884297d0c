import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_built():
    import importlib.util
    spec = importlib.util.spec_from_file_location("fjg_build", os.path.join(ROOT, "paper_2301_10841_b200", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    need = [B.LIBFJG, B.LIBFJGEN, B.LIBORACLE]
    if not all(os.path.exists(p) for p in need):
        B.build_all()


_ensure_built()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def engine():
    import paper_2301_10841_b200 as fjg
    eng = fjg.Engine(0)
    yield eng
    eng.close()
