import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

CASES = os.path.join(REPO, "data")
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgridadmm.so")
    config.addinivalue_line("markers", "slow: long-running")


def case_path(name: str) -> str:
    return os.path.join(CASES, name + ".m")


@pytest.fixture(scope="session")
def gridadmm():
    import paper_2110_06879_b200 as ga
    ga.lib()  # raises LibraryMissing loudly if the extension is not built
    return ga


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    return oracle
