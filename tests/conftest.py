import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds (incrementally) the product library and the oracle once."""
    from paper_2210_08804_b200 import _build

    if not _build.LIB.exists():
        _build.build()
    import oracle

    if not oracle.ORACLE_SO.exists() or (oracle.REF_SRC.exists() and not (
            oracle.REF_SO.exists() and oracle.REF_CACHE_TEST.exists()
            and oracle.REF_ENGINE_TEST.exists() and oracle.REF_REFRESH_TEST.exists()
            and oracle.REF_VDB_TEST.exists())):
        oracle.build()
    yield
