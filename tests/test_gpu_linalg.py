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


def _chol_inv_host(G, shift_rel):
    """The textbook loop rfxc_chol_inv restates (right-looking, unscaled rows,
    a non-positive pivot leaves its row/column zero)."""
    k = G.shape[0]
    R = 0.5 * (G + G.T)
    R = R + np.eye(k) * shift_rel * np.trace(R)
    for j in range(k - 1):
        d = R[j, j]
        if d > 0:
            R[j + 1:, j + 1:] -= np.triu(np.outer(R[j, j + 1:], R[j, j + 1:]) / d)
    dg = np.diag(R).copy()
    R = np.triu(R) / np.sqrt(np.where(dg > 0, dg, 1.0))[:, None]
    R[dg <= 0, :] = 0.0
    X = np.eye(k)
    for m in range(k - 1, -1, -1):
        X[m, m:] = X[m, m:] / R[m, m] if R[m, m] > 0 else 0.0
        X[:m, m:] -= np.outer(R[:m, m], X[m, m:])
    return X


@pytest.mark.parametrize("k,shift,rankdef", [(1, 0.0, False), (5, 0.0, False), (40, 0.0, False),
                                             (40, 1e-12, False), (40, 0.0, True), (64, 0.0, False),
                                             (110, 1e-12, False)])
def test_chol_inv_matches_host(k, shift, rankdef):
    import torch
    rng = np.random.default_rng(k)
    B = rng.normal(size=(k + 3, k)) * np.logspace(0, -3, k)[None, :]
    if rankdef and k > 4:
        B[:, 3] = 0.0  # a zero pivot: its row and column of R^-1 stay zero
    G = B.T @ B
    out = torch.empty((k, k), dtype=torch.float64, device="cuda")
    _lib.call("rfxc_chol_inv", _lib.ptr(dev(G)), k, shift, _lib.ptr(out), _lib.stream_handle())
    X = out.cpu().numpy()
    ref = _chol_inv_host(G, shift)
    np.testing.assert_allclose(X, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
    assert np.array_equal(np.tril(X, -1), np.zeros_like(X))
    if not rankdef:  # R^-T G R^-1 = I (shift 0)
        Gs = 0.5 * (G + G.T) + np.eye(k) * shift * np.trace(G)
        np.testing.assert_allclose(X.T @ Gs @ X, np.eye(k), atol=1e-8)
    # run to run identical
    out2 = torch.empty_like(out)
    _lib.call("rfxc_chol_inv", _lib.ptr(dev(G)), k, shift, _lib.ptr(out2), _lib.stream_handle())
    assert torch.equal(out, out2)


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
                                          (777, 130, 24, False), (5003, 120, 120, False),
                                          (5003, 128, 96, False), (70_001, 40, 40, False)])
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
