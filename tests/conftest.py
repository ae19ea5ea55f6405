"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``."""

import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _load_json(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as fh:
            return json.load(fh)
    with open(path) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def kb_graphs():
    return _load_json("graphs.json.gz")


@pytest.fixture(scope="session")
def mc_cases():
    return _load_json("mc_cases.json")


@pytest.fixture(scope="session")
def mc_full():
    return dict(np.load(os.path.join(GOLDEN, "mc_samples.npz")))


@pytest.fixture(scope="session")
def gittins_golden():
    return dict(np.load(os.path.join(GOLDEN, "gittins.npz")))


@pytest.fixture(scope="session")
def binning_golden():
    return _load_json("binning.json.gz")


@pytest.fixture(scope="session")
def prewarm_golden():
    return _load_json("prewarm.json")


@pytest.fixture(scope="session")
def config1_golden():
    return _load_json("config1.json.gz")
