"""The input producer (C++ restatement of rfx.train) reproduces the
reference forests byte for byte (RFX1 sha256 pinned by tests/golden)."""

import hashlib

import numpy as np
import pytest

from oracle.trainer import train
from paper_2511_19493_b200 import forest as F
from paper_2511_19493_b200.dataset import from_arrays, make_synthetic


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_wine50_bytes(wine50, fixtures):
    assert sha(F.forest_to_bytes(wine50)) == fixtures["wine50"]["rfx1_sha"]


def test_wine_stumps_bytes(built, wine_ds, fixtures):
    f = train(wine_ds, F.TrainConfig(ntree=3, iseed=1, min_node_size=10**6))
    assert sha(F.forest_to_bytes(f)) == fixtures["wine_stumps"]["rfx1_sha"]
    assert all(t.node_count == 1 for t in f.trees)


def test_synth2k_bytes(synth2k, fixtures):
    assert sha(F.forest_to_bytes(synth2k[1])) == fixtures["synth2k"]["rfx1_sha"]


def test_mixed_categorical_bytes(mixed, fixtures):
    assert sha(F.forest_to_bytes(mixed[1])) == fixtures["mixed"]["rfx1_sha"]


def test_thread_count_invariance(built):
    X, y = make_synthetic(600, 8, seed=3)
    ds = from_arrays(X, y)
    a = train(ds, F.TrainConfig(ntree=9, iseed=2), nthreads=1)
    b = train(ds, F.TrainConfig(ntree=9, iseed=2), nthreads=4)
    assert F.forest_to_bytes(a) == F.forest_to_bytes(b)


def test_rfx1_roundtrip(wine50, tmp_path):
    p = tmp_path / "f.rfx"
    F.save_forest(wine50, p)
    g = F.load_forest(p)
    assert F.forest_to_bytes(g) == F.forest_to_bytes(wine50)


def test_rfx1_bad_magic():
    from paper_2511_19493_b200.errors import DataError
    with pytest.raises(DataError):
        F.forest_from_bytes(b"JUNKJUNK")


def test_max_nodes_overflow(built):
    from paper_2511_19493_b200.errors import RfxError
    X, y = make_synthetic(200, 5, seed=1)
    with pytest.raises(RfxError):
        train(from_arrays(X, y), F.TrainConfig(ntree=2, iseed=1, max_nodes=3))


def test_synthetic_is_f32_exact():
    X, _ = make_synthetic(500, 12, seed=4)
    assert np.array_equal(X, X.astype(np.float32).astype(np.float64))
