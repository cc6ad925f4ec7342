"""Shared fixtures.  ``gpu`` tests need a B200 and the built CUDA library;
everything else runs on the CPU (oracle, front end, host logic, ABI loads)."""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblego_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_GOLDEN = None


def golden():
    global _GOLDEN
    if _GOLDEN is None:
        with open(os.path.join(TESTS, "golden", "layouts.json")) as fh:
            _GOLDEN = {c["name"]: c for c in json.load(fh)["cases"]}
    return _GOLDEN


@pytest.fixture(scope="session")
def golden_cases():
    return golden()
