"""The drop-in boundary end to end on the GPU: the
REFERENCE package (baseline/_ref, the unmodified reference installed there;
or /root/reference in the build container) with ``rfx_compat.install``.

* the reference's own writers (save_proximity, proximity.py:602-751) store
  what the GPU computed: RFXP (FullTriangle) and RFXT (TriBlock) files are
  byte-identical to the ones the reference writes from its own CPU results;
  RFXQ (INT8 factor) round-trips through load_proximity
  (tests/test_proximity.py:326-337's contract) and matches the reference
  factor at the stated tolerance;
* ``python -m paper_2511_19493_b200.cli`` is the reference CLI with the
  device path installed: ``proximity`` writes the same RFXP bytes as
  ``--device cpu`` (the reference unchanged), ``mds`` on the RFXQ file
  reproduces the reference embedding;
* chained calls keep the device state: ``full_proximity(leaf_membership(...))``
  never materialises the (n, B) codes on the host."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


@pytest.fixture(scope="module")
def ref(built):
    from paper_2511_19493_b200 import rfx_compat
    try:
        r = rfx_compat.import_reference()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference package not importable: {e}")
    import rfx.mds  # noqa: F401
    import rfx.proximity  # noqa: F401
    return r


@pytest.fixture(scope="module")
def wine(ref):
    from sklearn.datasets import load_wine
    w = load_wine()
    ds = ref.from_arrays(w.data, w.target)
    forest = ref.train(ds, ref.TrainConfig(ntree=50, iseed=17))
    return ds, forest


@pytest.fixture()
def installed(ref):
    from paper_2511_19493_b200 import rfx_compat
    rfx_compat.install(ref)
    yield ref
    rfx_compat.uninstall(ref)


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


def test_writers_store_gpu_results_byte_identically(ref, wine, tmp_path):
    from paper_2511_19493_b200 import rfx_compat
    RP = ref.proximity
    ds, forest = wine
    # the reference on its own CPU path
    mem = RP.leaf_membership(forest, ds)
    RP.save_proximity(RP.full_proximity(mem), tmp_path / "cpu.rfxp")
    RP.save_proximity(RP.triblock_proximity(mem, tau=0.05), tmp_path / "cpu.rfxt")
    lr_cpu = RP.lowrank_proximity(mem, rank=16, mode="i8", seed=5)
    rfx_compat.install(ref)
    try:
        gmem = RP.leaf_membership(forest, ds)
        assert gmem._host_codes is None  # codes still only in HBM
        full = RP.full_proximity(gmem)
        assert isinstance(full, RP.FullTriangle) and gmem._host_codes is None
        RP.save_proximity(full, tmp_path / "gpu.rfxp")
        RP.save_proximity(RP.triblock_proximity(gmem, tau=0.05), tmp_path / "gpu.rfxt")
        lr = RP.lowrank_proximity(gmem, rank=16, mode="i8", seed=5)
        RP.save_proximity(lr, tmp_path / "gpu.rfxq")
        assert np.array_equal(gmem.codes, mem.codes)  # materialised on demand
    finally:
        rfx_compat.uninstall(ref)
    assert _bytes(tmp_path / "gpu.rfxp") == _bytes(tmp_path / "cpu.rfxp")
    assert _bytes(tmp_path / "gpu.rfxt") == _bytes(tmp_path / "cpu.rfxt")
    back = RP.load_proximity(tmp_path / "gpu.rfxq")
    assert isinstance(back, RP.LowRankQuantized)
    assert np.array_equal(back.factor.data, lr.factor.data)
    assert np.array_equal(back.factor.scales, lr.factor.scales) and back.pmax == lr.pmax
    from test_gpu_lowrank import frob_rel
    dq = lambda q: q.factor.data.astype(np.float64) * q.factor.scales[None, :]  # noqa: E731
    assert frob_rel(dq(back), dq(lr_cpu)) <= 1e-4


def test_cli_proximity_and_mds_on_the_device(ref, wine, tmp_path):
    import csv

    from paper_2511_19493_b200 import cli
    from sklearn.datasets import load_wine
    w = load_wine()
    data = tmp_path / "wine.csv"
    with open(data, "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow([f"f{j}" for j in range(w.data.shape[1])] + ["y"])
        for row, y in zip(w.data, w.target):
            wr.writerow([repr(float(v)) for v in row] + [int(y)])
    forest = tmp_path / "f.rfx"
    assert cli.main(["--device", "cpu", "train", "--data", str(data), "--label", "y",
                     "--trees", "40", "--seed", "3", "--out", str(forest)]) == 0
    for dev in ("cpu", "cuda"):
        assert cli.main(["--device", dev, "proximity", "--data", str(data), "--label", "y",
                         "--forest", str(forest), "--backend", "full",
                         "--out", str(tmp_path / f"{dev}.rfxp")]) == 0
        assert cli.main(["--device", dev, "proximity", "--data", str(data), "--label", "y",
                         "--forest", str(forest), "--backend", "lowrank", "--rank", "12",
                         "--out", str(tmp_path / f"{dev}.rfxq")]) == 0
        assert cli.main(["--device", dev, "mds", "--prox", str(tmp_path / f"{dev}.rfxq"),
                         "--out-json", str(tmp_path / f"{dev}.json")]) == 0
    assert _bytes(tmp_path / "cuda.rfxp") == _bytes(tmp_path / "cpu.rfxp")
    e_cpu = ref.mds.embedding_from_json(tmp_path / "cpu.json")
    e_gpu = ref.mds.embedding_from_json(tmp_path / "cuda.json")
    np.testing.assert_allclose(e_gpu.eigenvalues, e_cpu.eigenvalues, rtol=1e-5)
    assert ref.mds.mds_correlation(e_gpu, e_cpu) >= 0.99999


def test_chained_calls_reuse_device_state(installed, wine):
    RP = installed.proximity
    ds, forest = wine
    mem = RP.leaf_membership(forest, ds)
    lr = RP.lowrank_proximity(mem, rank=8, mode="i8", seed=0)
    assert mem._host_codes is None
    emb = installed.mds.mds_lowrank(lr)
    assert emb.coordinates.shape == (ds.n, 3)
    assert lr._mine is not None and lr.factor is lr._mine_factor
    # a caller replacing the codes invalidates the device copy
    mem.codes = np.zeros_like(mem.codes)
    full = RP.full_proximity(mem)
    assert np.all(full.packed == 1.0)
