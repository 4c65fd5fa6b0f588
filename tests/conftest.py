import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a real B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def planner_golden():
    with open(os.path.join(GOLDEN, "planner_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def streams_golden():
    with open(os.path.join(GOLDEN, "streams_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def readme_kat():
    with open(os.path.join(GOLDEN, "readme_kat.json")) as f:
        return json.load(f)
