"""Shared fixtures.  Tests that need a GPU are marked ``gpu``; everything else
runs on CPU (the oracle, host logic, the C ABI symbol table, gloo multi-process
sharding)."""

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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def built():
    from paper_2511_19493_b200.build import build
    build()
    from oracle import oracle as orc
    orc.build()
    return True


@pytest.fixture(scope="session")
def orc(built):
    from oracle import oracle as o
    return o


@pytest.fixture(scope="session")
def fixtures():
    with open(os.path.join(GOLDEN, "fixtures.json")) as fh:
        return json.load(fh)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def wine_ds():
    from sklearn.datasets import load_wine
    from paper_2511_19493_b200.dataset import from_arrays
    w = load_wine()
    return from_arrays(w.data, w.target)


@pytest.fixture(scope="session")
def wine50(built, wine_ds):
    from oracle.trainer import train
    from paper_2511_19493_b200.forest import TrainConfig
    return train(wine_ds, TrainConfig(ntree=50, iseed=17))


@pytest.fixture(scope="session")
def synth2k(built):
    from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
    from oracle.trainer import train
    from paper_2511_19493_b200.forest import TrainConfig
    X, y = make_synthetic(2000, 20, seed=1)
    ds = from_arrays(X, y)
    return ds, train(ds, TrainConfig(ntree=40, iseed=1))


@pytest.fixture(scope="session")
def mixed(built):
    from paper_2511_19493_b200.dataset import ColumnKind, from_arrays
    from oracle.trainer import train
    from paper_2511_19493_b200.forest import TrainConfig
    g = golden("mixed.npz")
    cols = (ColumnKind("categorical", tuple("abcde")), ColumnKind("numeric"),
            ColumnKind("categorical", ("x", "y", "z")), ColumnKind("numeric"))
    ds = from_arrays(g["X"], g["y"], columns=cols)
    return ds, train(ds, TrainConfig(ntree=12, iseed=4))


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
