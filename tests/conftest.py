import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsnop_cuda.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def ctx():
    from paper_2509_01416_b200 import snop
    c = snop.Context(0)
    yield c
    c.close()


@pytest.fixture
def ctx_options():
    """Set execution options (snop_ctx_options) on the default context for one test; restored after."""
    from paper_2509_01416_b200 import snop
    c = snop.default_context()
    saved = c.options()

    def set_(**kw):
        c.set_options(**{**saved, **kw})

    yield set_
    c.set_options(**saved)
