import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libpinla.so)")


def load_golden(case):
    path = os.path.join(GOLDEN, f"{case}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden {case} not generated")
    return np.load(path, allow_pickle=False)


def golden_instance(G):
    from paper_2204_04678_b200.synth import make_instance

    return make_instance(str(G["config"]), **json.loads(str(G["overrides"])))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    oracle.lib()
    return oracle
