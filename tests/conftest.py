import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running check (minutes)")


def golden(name):
    return os.path.join(ROOT, "tests", "golden", name)


def paper_counts():
    out = {}
    with open(golden("paper_counts.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, v = line.split()[:2]
            out[k] = int(v)
    return out
