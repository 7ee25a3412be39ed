"""Pins for oracle.factorize, Alg 1's "A, B <- SVD(K)".

Pinned against: exact reconstruction of keys whose true rank is <= r; the Eckart-Young
truncation error sqrt(sum_{i>r} sigma_i^2) computed by an independent SVD (one-sided Jacobi, S:50,
S:88); the per-head split of the flattened factor (A shared, B per head); and A^T A = Sigma_r^2
(orthogonal columns of U scaled by the singular values).
"""
import math

import numpy as np
import pytest

from oracle import shadowkv_oracle as O


def _keys(rng, b, hk, s, d, true_rank, noise=0.0):
    K = np.zeros((b, hk, s, d))
    for bi in range(b):
        X = rng.normal(size=(s, true_rank)) @ rng.normal(size=(true_rank, hk * d))
        X += noise * rng.normal(size=X.shape)
        K[bi] = X.reshape(s, hk, d).transpose(1, 0, 2)
    return K


def _rebuild(A, B):
    """K~[b][h][t] = A[b][t] . B[b][h] (Alg 2's rebuild without RoPE)."""
    return np.einsum("btr,bhrd->bhtd", A, B)


@pytest.mark.parametrize("true_rank,r", [(5, 5), (5, 8), (12, 16)])
def test_exact_rank_keys_rebuild_exactly(true_rank, r):
    rng = np.random.default_rng(true_rank * 10 + r)
    K = _keys(rng, 2, 2, 48, 8, true_rank)
    A, B, sig = O.factorize(K, r)
    np.testing.assert_allclose(_rebuild(A, B), K, atol=1e-10)
    assert np.all(sig[:, true_rank:] < 1e-9)


def test_truncation_error_is_eckart_young_with_independent_svd():
    rng = np.random.default_rng(3)
    K = _keys(rng, 1, 2, 30, 6, 12, noise=0.3)
    r = 5
    A, B, sig = O.factorize(K, r)
    X = K[0].transpose(1, 0, 2).reshape(30, 12)
    _, sj, _ = O.jacobi_svd(X)                        # independent algorithm
    np.testing.assert_allclose(sig[0], sj, rtol=1e-10)
    err = np.linalg.norm(_rebuild(A, B) - K)
    assert abs(err - math.sqrt((sj[r:] ** 2).sum())) < 1e-9


def test_jacobi_and_lapack_factorizations_rebuild_the_same_keys():
    """The factor split is unique only up to signs/rotations; the rebuilt keys A.B are unique when
    sigma_r > sigma_{r+1}."""
    rng = np.random.default_rng(4)
    K = _keys(rng, 1, 3, 40, 4, 12, noise=0.2)
    A1, B1, _ = O.factorize(K, 6)
    A2, B2, _ = O.factorize(K, 6, svd=O.jacobi_svd)
    np.testing.assert_allclose(_rebuild(A1, B1), _rebuild(A2, B2), atol=1e-9)


def test_factor_structure():
    """A = U_r Sigma_r: columns orthogonal with squared norms sigma_i^2; B_h rows are head slices of
    orthonormal right singular vectors (sum over heads of B_h B_h^T = I_r)."""
    rng = np.random.default_rng(5)
    K = _keys(rng, 1, 2, 50, 8, 16, noise=0.1)
    r = 7
    A, B, sig = O.factorize(K, r)
    np.testing.assert_allclose(A[0].T @ A[0], np.diag(sig[0, :r] ** 2), atol=1e-9)
    G = sum(B[0, h] @ B[0, h].T for h in range(2))
    np.testing.assert_allclose(G, np.eye(r), atol=1e-12)


# ---------------------------------------------------------------- NEXT-4: low-rank generated keys
def _inv(d):
    return (1.0 / 10000 ** (np.arange(0, d, 2) / d)).astype(np.float32)


def test_lowrank_generated_key_exact_inside_the_subspace():
    """A generated pre-RoPE key that lies in the context's rank-r subspace is reproduced exactly:
    Psi Psi^T k' = k' (orthonormal Psi from the SVD), so the attended key is RoPE_t(k')."""
    rng = np.random.default_rng(30)
    K = _keys(rng, 1, 2, 64, 8, 6)
    A, B, _ = O.factorize(K, 6)
    Vt = B[0].transpose(1, 0, 2).reshape(6, 16)                          # Psi^T, heads concatenated
    kp = (rng.normal(size=(1, 6)) @ Vt).reshape(1, 2, 1, 8)              # [b][h][n=1][d], inside the span
    pos = np.array([70])
    a, keys = O.lowrank_generated_keys(kp, B, pos, _inv(8), 8, False, store=O.identity_store)
    want = np.stack([O.rope(kp[0, h], pos, _inv(8), 8, False) for h in range(2)])
    np.testing.assert_allclose(keys[0], want, atol=1e-12)


def test_lowrank_generated_key_error_is_the_distance_to_the_subspace():
    """Pythagoras with orthonormal Psi: ||k'||^2 = ||a||^2 + ||k' - a Psi^T||^2 (pre-RoPE; RoPE is an
    isometry, so the post-RoPE error is the same), and a is r numbers instead of h_kv * d."""
    rng = np.random.default_rng(31)
    K = _keys(rng, 1, 3, 80, 8, 24, noise=0.1)
    r = 8
    A, B, _ = O.factorize(K, r)
    kp = rng.normal(size=(1, 3, 2, 8))
    pos = np.array([90, 91])
    a, keys = O.lowrank_generated_keys(kp, B, pos, _inv(8), 8, False, store=O.identity_store)
    assert a.shape == (1, 2, r)
    for n in range(2):
        x = kp[0, :, n].reshape(-1)
        rec = np.concatenate([a[0, n] @ B[0, h] for h in range(3)])
        assert abs(x @ x - (a[0, n] @ a[0, n] + (x - rec) @ (x - rec))) < 1e-10
        exact = np.stack([O.rope(kp[0, h, n:n + 1], pos[n:n + 1], _inv(8), 8, False)[0] for h in range(3)])
        assert abs(np.linalg.norm(keys[0, :, n] - exact) - np.linalg.norm(x - rec)) < 1e-10
