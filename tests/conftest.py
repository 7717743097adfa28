import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsten.so")
    # experiment builds (tools/build_variants.py): run the suite against libsten_<tag>.so
    tag = os.environ.get("STEN_TEST_VARIANT")
    if tag:
        import paper_2010_03660_b200 as sten
        sten.LIB_PATH = os.path.join(ROOT, "paper_2010_03660_b200", f"libsten_{tag}.so")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle
