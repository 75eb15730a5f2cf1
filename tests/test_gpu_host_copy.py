"""The staged device->host copy behind FullTriangle.packed and
LeafMembership.codes (device.host_copy): chunked through a pinned ring, it
must return exactly what .cpu() returns, for sizes below, at and across the
chunk size, any dtype and shape."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


@pytest.mark.parametrize("numel,dtype", [(1000, "float64"), (2 * (64 << 20) // 8, "float64"),
                                          (3 * (64 << 20) // 4 + 12345, "int32"),
                                          (5 * (64 << 20) // 8 + 7, "float64")])
def test_host_copy_matches_cpu(built, numel, dtype):
    import torch
    from paper_2511_19493_b200 import device as D
    t = torch.arange(numel, dtype=getattr(torch, dtype), device="cuda") * 3 - 7
    got = D.host_copy(t)
    assert got.dtype == np.dtype(dtype) and got.shape == (numel,)
    assert np.array_equal(got, t.cpu().numpy())
    t2 = t[: numel - numel % 10].view(-1, 10)
    assert np.array_equal(D.host_copy(t2), t2.cpu().numpy())
