import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built_oracle():
    # The C restatement is test infrastructure; make sure it is compiled.
    from oracle import pyoracle

    if not os.path.exists(pyoracle.ORACLE_SO):
        pyoracle.build()
