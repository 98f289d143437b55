import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")


def pytest_collection_modifyitems(config, items):
    # Any test marked gpu fails loudly (not skipped) if no GPU is present and gpu tests
    # were explicitly selected; unselected runs (-m "not gpu") never reach them.
    pass


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.lib()
    return oracle
