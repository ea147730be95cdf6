import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")
    config.addinivalue_line("markers", "slow: builds a full-size BASELINE.json index")


_CACHE = {}


def load_cfg(name):
    """(cfg, index dict, queries, data) for a datagen config, built once per session."""
    if name not in _CACHE:
        import datagen
        from datagen import configs, index_file, synth
        cfg = configs.get(name)
        path = datagen.ensure_index(cfg)
        ix = index_file.read(path)
        Q = synth.generate_queries(cfg)
        _CACHE[name] = (cfg, ix, Q, path)
    return _CACHE[name]


@pytest.fixture(scope="session")
def load():
    return load_cfg


@pytest.fixture(scope="session")
def c1t():
    return load_cfg("C1t")


@pytest.fixture(scope="session")
def c3s():
    return load_cfg("C3s")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
