"""pytest configuration: markers, paths, shared fixtures.

`-m "not gpu"` runs the oracle pins, host-logic and ABI-load tests on a CPU-only box;
`-m gpu` runs the parity tests through the C ABI on a B200.
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: longer-running CPU test")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_key(name):
    k = load_golden(os.path.join("keys", name + ".json"))
    return {f: (int(v, 16) if isinstance(v, str) and f not in ("seed", "recipe") else v) for f, v in k.items()}


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def keys():
    return {n: load_key(n) for n in ("rsa1024", "rsa2048", "rsa3072")}
