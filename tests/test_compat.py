"""rfx_compat: installing the B200 path into the reference package (CPU
checks: patching, signatures, exception translation, no CPU fallback).
Skipped where the reference is absent (the GPU box)."""

import inspect
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture()
def rfx():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rfx as r
    import rfx.mds  # noqa: F401
    import rfx.proximity  # noqa: F401
    from paper_2511_19493_b200 import rfx_compat
    orig = {n: getattr(r.proximity, n) for n in rfx_compat.PATCHED["proximity"]}
    rfx_compat.install(r)
    yield r, orig
    rfx_compat.uninstall(r)


def test_install_replaces_and_keeps_signatures(rfx):
    r, orig = rfx
    for name, fn in orig.items():
        new = getattr(r.proximity, name)
        assert new is not fn
        assert list(inspect.signature(new).parameters) == list(
            inspect.signature(fn).parameters), name


def test_errors_are_the_reference_types(rfx, monkeypatch):
    r, _ = rfx
    mem = r.proximity.LeafMembership(codes=np.zeros((3, 2), np.int32),
                                     leaf_counts=np.ones(2, np.int32))
    # budget refusal happens before any device work, as in the reference
    with pytest.raises(r.errors.BudgetError) as ei:
        r.proximity.full_proximity(mem, budget_bytes=1)
    assert isinstance(ei.value.plan, dict)
    with pytest.raises(r.errors.DataError):
        r.proximity.triblock_proximity(mem, tau=2.0)
    # no CPU fallback: without a CUDA device the product path raises
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(r.errors.RfxError):
        r.proximity.lowrank_proximity(mem, rank=1)


def test_uninstall_restores(rfx):
    r, orig = rfx
    from paper_2511_19493_b200 import rfx_compat
    rfx_compat.uninstall(r)
    for name, fn in orig.items():
        assert getattr(r.proximity, name) is fn
    rfx_compat.install(r)
