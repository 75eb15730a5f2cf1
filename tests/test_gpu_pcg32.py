"""Device PCG32 streams against known answers the REFERENCE produced
(rng.py:41-70 next/bounded, :102-115 fill_normals; tests/golden/make_golden.py).

* rfxc_normals(seed, seq, count) — Omega = Pcg32(seed, 3).normals((n, k))
  (proximity.py:392-393) and the MDS starts Pcg32(seed + c, 5).normals(n)
  (mds.py:210-211): the raw u32 stream must be the reference's exactly; the
  Box-Muller transform goes through the device's own log/sqrt/cos/sin (CUDA:
  log 1 ulp, cos/sin 2 ulp max error), which are not glibc's, so values are
  required to agree to ULP_TOL = 4 ulp (measured max: 3 over 3 x 10^5 draws);
  the count of bit-identical values is asserted to be the large majority.
* rfxc_pmax_draws(seed, n) — the 2048 bounded draws of the pmax pair sampler
  Pcg32(seed, 4) (proximity.py:409-417), generated in parallel by jump-ahead
  inside rfxc_pmax: bit-exact, including n > 2^31 and a tiny n with many
  rejections."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

ULP_TOL = 4


def ulps(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-0x8000000000000000) - ia, ia)
    ib = np.where(ib < 0, np.int64(-0x8000000000000000) - ib, ib)
    return np.abs(ia - ib)


def test_normals_known_answers(built):
    import torch

    from paper_2511_19493_b200 import _lib
    kats = json.load(open(os.path.join(GOLDEN, "pcg32.json")))
    exact = total = 0
    for k in kats:
        want = np.array([float.fromhex(h) for h in k["normals"]])
        out = torch.empty(len(want), dtype=torch.float64, device="cuda")
        _lib.call("rfxc_normals", int(k["seed"]), int(k["seq"]), len(want), _lib.ptr(out),
                  _lib.stream_handle())
        got = out.cpu().numpy()
        d = ulps(got, want)
        assert d.max() <= ULP_TOL, (k["seed"], k["seq"], got, want)
        exact += int((d == 0).sum())
        total += len(want)
    assert exact >= 0.8 * total, f"only {exact}/{total} bit-identical"


def test_normals_long_stream_against_the_oracle(orc, built):
    """Jump-ahead: 10^5 normals (threads start mid-stream) vs the pinned C
    oracle's sequential stream, through the same ulp bound."""
    import torch

    from paper_2511_19493_b200 import _lib
    n = 100_001
    for seed, seq in ((0, 3), (123, 5), (-7, 3)):
        want = orc.Pcg32(seed, seq).normals(n)
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("rfxc_normals", seed, seq, n, _lib.ptr(out), _lib.stream_handle())
        d = ulps(out.cpu().numpy(), want)
        assert d.max() <= ULP_TOL and (d == 0).mean() >= 0.8


def test_pmax_draws_known_answers(built):
    import torch

    from paper_2511_19493_b200 import _lib
    kats = json.load(open(os.path.join(GOLDEN, "pcg32_pmax.json")))
    for k in kats:
        out = torch.empty(2048, dtype=torch.int32, device="cuda")
        _lib.call("rfxc_pmax_draws", int(k["seed"]), int(k["n"]), _lib.ptr(out),
                  _lib.stream_handle())
        got = out.cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(got, np.array(k["draws"], np.int64)), (k["seed"], k["n"])
