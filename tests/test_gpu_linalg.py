"""K5 on the device: Jacobi eigensolver, orthonormalising map + CholeskyQR
step, Rayleigh-Ritz factor map (np.linalg.qr / eigh of proximity.py:395-403)
against numpy/LAPACK."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

from paper_2511_19493_b200 import _lib  # noqa: E402
from paper_2511_19493_b200 import proximity as P  # noqa: E402


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("k", [1, 2, 7, 40, 108])
def test_sym_eig_matches_lapack(k):
    import torch
    rng = np.random.default_rng(k)
    B = rng.normal(size=(k, k))
    A = B @ B.T + np.diag(rng.uniform(0, 1, k))
    w = torch.empty(k, dtype=torch.float64, device="cuda")
    V = torch.empty((k, k), dtype=torch.float64, device="cuda")
    _lib.call("rfxc_sym_eig", _lib.ptr(dev(A)), k, _lib.ptr(w), _lib.ptr(V), _lib.stream_handle())
    w, V = w.cpu().numpy(), V.cpu().numpy()
    ref = np.linalg.eigvalsh(A)[::-1]
    np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-12 * ref[0])
    np.testing.assert_allclose(V.T @ V, np.eye(k), atol=1e-12)
    np.testing.assert_allclose(A @ V, V * w[None, :], atol=1e-10 * ref[0])


@pytest.mark.parametrize("deficient", [False, True])
def test_orthonormalize_spans_and_is_orthonormal(deficient):
    rng = np.random.default_rng(3)
    n, k = 5000, 40
    Y = rng.normal(size=(n, k)) * np.logspace(0, -6, k)[None, :]
    if deficient:  # exactly dependent and zero columns
        Y[:, 5] = 2.0 * Y[:, 3]
        Y[:, 9] = 0.0
    Q, Q32 = P.orthonormalize(dev(Y), 40)
    Q = Q.cpu().numpy()
    # an exactly zero column of Y stays a zero column; the rest is orthonormal
    live = np.linalg.norm(Y, axis=0) > 0
    np.testing.assert_allclose(Q[:, ~live], 0.0)
    np.testing.assert_allclose(Q[:, live].T @ Q[:, live], np.eye(live.sum()), atol=1e-12)
    # range(Q) contains range(Y) (like LAPACK QR, extra columns complete the basis)
    np.testing.assert_allclose(Q @ (Q.T @ Y), Y, atol=1e-10 * np.abs(Y).max())
    assert np.array_equal(Q32.cpu().numpy()[:, :k], Q.astype(np.float32))


def test_ritz_factor_map_matches_host():
    import torch
    rng = np.random.default_rng(5)
    k, r = 40, 32
    B = rng.normal(size=(k, k))
    T = B @ B.T - 3.0 * np.eye(k)  # some negative eigenvalues get clipped
    Wr = torch.empty((k, r), dtype=torch.float64, device="cuda")
    _lib.call("rfxc_ritz_factor_map", _lib.ptr(dev(T)), k, r, _lib.ptr(Wr), _lib.stream_handle())
    Wr = Wr.cpu().numpy()
    lam, W = np.linalg.eigh(T)
    order = np.argsort(lam)[::-1][:r]
    ref = W[:, order] * np.sqrt(np.clip(lam[order], 0, None))[None, :]
    # eigenvectors are defined up to sign
    np.testing.assert_allclose(np.abs(Wr), np.abs(ref), atol=1e-10)
    np.testing.assert_allclose(Wr @ Wr.T, ref @ ref.T, atol=1e-10)


@pytest.mark.parametrize("n,ka,kb,same", [(1, 3, 3, True), (5, 8, 8, True), (178, 24, 24, True),
                                          (178, 24, 24, False), (1000, 40, 16, False),
                                          (100_003, 40, 40, True), (4099, 108, 108, True),
                                          (777, 130, 24, False)])
def test_gram_matches_numpy(built, n, ka, kb, same):
    """rfxc_gram (A^T B, f64, fixed-order partial sums) against numpy."""
    import torch
    from paper_2511_19493_b200 import proximity as P
    rng = np.random.default_rng(n + ka)
    A = rng.normal(size=(n, ka))
    B = A if same else rng.normal(size=(n, kb))
    dA = torch.from_numpy(A).cuda()
    dB = dA if same else torch.from_numpy(B).cuda()
    got = P._gram(dA, dB).cpu().numpy()
    want = A.T @ B
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
