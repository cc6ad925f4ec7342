"""pytest plugin: makes ``import lego`` (and ``lego.<module>``) resolve to this
backend's mirror of the reference API, so the reference package's own test
suite can run against it (tests/test_reference_suite.py)."""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
_pkg = importlib.import_module("paper_2505_08091_b200")
sys.modules["lego"] = _pkg
for _sub in ("expr", "layout", "simplify", "emit", "dsl", "template", "errors"):
    sys.modules["lego." + _sub] = importlib.import_module("paper_2505_08091_b200." + _sub)
