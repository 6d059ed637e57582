"""Shared fixtures.  `-m gpu` tests need a B200 and the built CUDA library;
everything else runs on the CPU (oracle pins, C-ABI host functions, the
multi-rank host logic over gloo)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_small():
    with open(os.path.join(GOLDEN, "golden_small.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_configs():
    path = os.path.join(GOLDEN, "golden_configs.json")
    if not os.path.exists(path):
        pytest.skip("golden_configs.json not generated")
    with open(path) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle
    return pyoracle.Port()


@pytest.fixture(scope="session")
def cuda_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_0264_b200 as mmm
    mmm.load()
    return mmm
