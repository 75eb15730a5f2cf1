"""CPU checks of the host-side pieces added around the device path: the CLI
wrapper's device switch, the device-backed reference LeafMembership subclass
(rfx_compat), the rank limits checked before any device work, and bench.py's
bookkeeping helpers."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def test_cli_rejects_unknown_device(capsys):
    from paper_2511_19493_b200 import cli
    assert cli.main(["--device", "tpu", "proximity"]) == 2
    assert "--device must be cuda or cpu" in capsys.readouterr().err


def _ref_or_skip():
    from paper_2511_19493_b200 import rfx_compat
    try:
        return rfx_compat.import_reference()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference package not importable: {e}")


def test_device_membership_subclass_contract():
    rfx = _ref_or_skip()
    import rfx.proximity as RP

    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200 import rfx_compat
    cls = rfx_compat._device_classes(rfx)
    mine = P.LeafMembership(np.array([[0, 1], [0, 0]], np.int32), np.array([1, 2], np.int32))
    ref = cls(mine)
    assert isinstance(ref, RP.LeafMembership)
    assert ref._host_codes is None and ref.n == 2 and ref.tree_count == 2
    assert rfx_compat._ours_membership(ref) is mine       # device state reused
    assert np.array_equal(ref.codes, mine.codes)           # materialised on demand
    ref.codes = np.zeros((2, 2), np.int32)                 # a caller replaces the codes
    assert ref._mine is None
    other = rfx_compat._ours_membership(ref)
    assert other is not mine and np.array_equal(other.codes, np.zeros((2, 2)))


def test_rank_limit_before_device_work(monkeypatch):
    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.errors import DataError
    n = 400
    codes = (np.arange(n)[:, None] % np.array([[300, 301]])).astype(np.int32)
    mem = P.LeafMembership(codes, np.array([300, 301], np.int32))
    # no CUDA here: the limit must be reported before anything touches a device
    with pytest.raises(DataError, match="above this build's limit"):
        P.lowrank_proximity(mem, rank=P.MAX_RANK + 1)


def test_mds_rank_limit_before_device_work():
    from paper_2511_19493_b200 import mds as M
    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.errors import DataError
    from paper_2511_19493_b200.quantize import QuantFactor
    r = M.MAX_RANK + 1
    lr = P.LowRankQuantized(n=4, rank=r, mode="f32",
                            factor=QuantFactor("f32", (4, r), np.zeros((4, r), np.float32), None),
                            pmax=1.0, tree_count=1)
    with pytest.raises(DataError, match="above this build's limit"):
        M.mds_lowrank(lr)


def test_bench_helpers():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.dense_cpu_whole(bench.CONFIGS["10k-dense"])
    assert not bench.dense_cpu_whole(bench.CONFIGS["50k-dense"])
    n, B, k = 100_000, 500, 40
    ab = bench.algorithmic_bytes("sketch_pass", n, B, 4_744_201, k, 100, 9_490_000, 32)
    assert ab == 2 * n * B * 4 + (4_744_201 + 1) * 8 + n * k * 4 + n * k * 8
    assert bench.algorithmic_bytes("unknown_kernel", n, B, 1, k, 1, 1, 32) is None
