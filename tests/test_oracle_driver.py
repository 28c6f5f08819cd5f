"""Pins of the oracle's iterative driver (§4.2).

  * power_norm vs the spectrum of the dense n = 32 operator (numpy.linalg.eigvalsh of
    omega A^T A, an independent library route);
  * the gradient identity E:operators (L164-167) by central finite differences of the data
    fidelity J(f) = 1/2 ||A f - g||_Y^2 in the X inner product;
  * the projected-gradient fixed point: consistent non-negative data are reproduced exactly;
  * monotone decrease of ||A f_k - g||_Y for 0 < lambda < 2/lambda_max (descent lemma), and
    f_k >= 0 and zero outside the region of interest (projection invariants).
"""
import numpy as np
import pytest

import synth
from oracle import tat_oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")


@pytest.fixture(scope="module")
def t32():
    return O.derive_geom(synth.geometry("T32"))


@pytest.fixture(scope="module")
def dense_t32(t32):
    C = t32
    n = C.n
    A = np.empty((C.n_t * C.n_det, n * n))
    for i in range(n * n):
        e = np.zeros(n * n)
        e[i] = 1.0
        A[:, i] = O.forward(e.reshape(n, n), C).ravel()
    return A


def _weights(C):
    return C.dt * 2 * np.pi * C.R / C.n_ring, C.h * C.h      # w_Y, w_X (reading G18)


def test_power_norm_vs_dense_spectrum(t32, dense_t32):
    C = t32
    lam_dense = np.linalg.eigvalsh(C.omega * dense_t32.T @ dense_t32).max()
    lam = O.power_norm(C, synth.random_image(C.n, 7), 200)
    assert abs(lam - lam_dense) <= 1e-6 * lam_dense


def test_gradient_identity_finite_differences(t32):
    C = t32
    wY, wX = _weights(C)
    f = synth.random_image(C.n, 11).astype(np.float64)
    d = synth.random_image(C.n, 12).astype(np.float64)
    g = synth.random_data(C.n_t, C.n_det, 13).astype(np.float64)
    J = lambda x: 0.5 * wY * np.sum((O.forward(x, C) - g) ** 2)
    eps = 1e-3
    fd = (J(f + eps * d) - J(f - eps * d)) / (2 * eps)      # J is quadratic: exact up to rounding
    grad = O.adjoint(O.forward(f, C) - g, C)                 # E:operators / 2
    assert abs(fd - wX * np.sum(grad * d)) <= 1e-9 * abs(fd)


def test_fixed_point_of_consistent_nonnegative_data(t32):
    C = t32
    f = np.maximum(synth.phantom("C1", 0, n=C.n).astype(np.float64), 0.0)
    g = O.forward(f, C)
    lam = 1.0 / O.power_norm(C, synth.random_image(C.n, 3), 30)
    f1 = O.nnls(g, f, C, lam, 1)
    assert np.abs(f1 - f).max() <= 1e-12 * np.abs(f).max()


def test_monotone_descent_and_projection_invariants(t32):
    C = t32
    wY, _ = _weights(C)
    f_true = np.maximum(synth.phantom("C1", 1, n=C.n).astype(np.float64), 0.0)
    g = O.forward(f_true, C) + 0.02 * synth.random_data(C.n_t, C.n_det, 5)
    lam = 1.0 / O.power_norm(C, synth.random_image(C.n, 4), 30)
    n = C.n
    yy, xx = np.mgrid[0:n, 0:n]
    roi = ((yy >= n // 2)).astype(np.float64)               # upper half (eqn:projectionHalfCircle)
    f = np.zeros((n, n))
    prev = np.inf
    for _ in range(8):
        f = O.nnls(g, f, C, lam, 1, nonneg=True, roi=roi)
        res = wY * np.sum((O.forward(f, C) - g) ** 2)
        assert res <= prev * (1 + 1e-12)
        assert f.min() >= 0.0 and np.all(f[roi == 0] == 0.0)
        prev = res


def test_stopping_rule_against_eigendecomposition(t32, dense_t32):
    """nnls_converge (reading G28) pinned by an independent route: for the
    unconstrained iteration from f0 = 0 the update is f^k - f^(k-1) = (I - lam M)^(k-1) lam b,
    M = A*A = omega A^T A, b = A* g (dense T32 operator), evaluated through numpy.linalg.eigh of
    M; the first k >= 2 whose update norm is below 0.3 % of ||f^1|| = ||lam b|| is the stop."""
    C = t32
    A = dense_t32
    M = C.omega * A.T @ A
    w, V = np.linalg.eigh(0.5 * (M + M.T))
    lam = 1.0 / w.max()
    g = synth.random_data(C.n_t, C.n_det, 31).astype(np.float64)
    b = C.omega * A.T @ g.ravel()
    c = V.T @ (lam * b)
    s = np.linalg.norm(lam * b)
    k_ref = next(k for k in range(2, 5000)
                 if np.linalg.norm((1.0 - lam * w) ** (k - 1) * c) < 3e-3 * s)
    f, k = O.nnls_converge(g, np.zeros((C.n, C.n)), C, lam, 5000, nonneg=False)
    assert k == k_ref
    x = np.clip(lam * w, 0.0, None)
    f_ref = V @ (lam * np.where(x > 0, -np.expm1(k * np.log1p(-x)) / np.where(x > 0, x, 1), k) * (V.T @ b))
    # (k float64 iterations vs the spectral closed form; the near-null modes amplify rounding)
    assert np.linalg.norm(f.ravel() - f_ref) <= 1e-6 * np.linalg.norm(f_ref)
    # checked every m-th iteration: the update norms are non-increasing (|1 - lam w| <= 1), so
    # the stop is the first multiple of m at or after k_ref
    for m in (3, 7):
        _, km = O.nnls_converge(g, np.zeros((C.n, C.n)), C, lam, 5000, check_every=m, nonneg=False)
        assert km == -(-k_ref // m) * m
    # not converged within the cap: negative count
    _, kc = O.nnls_converge(g, np.zeros((C.n, C.n)), C, lam, k_ref - 1, nonneg=False)
    assert kc == -(k_ref - 1)
