import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# parity records appended by the GPU tests (worst errors per comparison); written to
# $LSQ_PARITY_OUT at session end (profiles/r02/parity_table.json comes from it)
PARITY_LOG = []


@pytest.fixture(autouse=True)
def _parity_test_id(request):
    start = len(PARITY_LOG)
    yield
    for rec in PARITY_LOG[start:]:
        rec.setdefault("test", request.node.nodeid.split("::", 1)[-1])


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("LSQ_PARITY_OUT")
    if out and PARITY_LOG:
        import json

        os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
        with open(out, "w") as f:
            json.dump(PARITY_LOG, f, indent=1)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture
def golden():
    return load_golden
