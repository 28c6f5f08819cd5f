"""Pins of the oracle's dense mode (reading G24): detectors at angles
off every canonical ring, with D6/D7 evaluated as dense sums at the exact angles.

  * on a canonical geometry the dense synthesis equals the pinned ring path (restriction of
    the n_phi-point synthesis) and its adjoint equals the ring adjoint;
  * the adjoint identity of eqn:innerProducts (weights 2 pi R / n_phi per detector, G24);
  * the continuous Gaussian solution (check (1), E:green_conv by 1-D quadrature) at irregular
    detector positions, within the same error budget as the canonical case.
"""
import numpy as np
from scipy import integrate, special

import synth
from oracle import tat_oracle as O


def _irregular_angles(n_det, seed):
    rng = np.random.default_rng(seed)
    base = np.sort(rng.uniform(0.0, 2 * np.pi, n_det))
    return base


def test_dense_equals_ring_path_on_canonical_geometry():
    C = O.derive_geom(synth.geometry("T32"))
    Cd = O.Constants(**{**C.__dict__, "dense": True,
                        "angles": tuple(2 * np.pi * np.asarray(C.ring) / C.n_ring)})
    G = synth.random_data(C.n_t, C.n_phi, 1).astype(np.float64) @ np.ones((C.n_phi, 1)) * 0
    rng = np.random.default_rng(3)
    G = rng.standard_normal((C.n_t, 2 * C.K)) + 1j * rng.standard_normal((C.n_t, 2 * C.K))
    # Hermitian structure of a real signal: G[-k] = conj G[k], G[-K] real
    k = O._harmonics(C)
    for i, kk in enumerate(k):
        if kk > 0:
            G[:, np.where(k == -kk)[0][0]] = np.conj(G[:, i])
    G[:, k == 0] = G[:, k == 0].real
    G[:, k == -C.K] = G[:, k == -C.K].real
    ring = O.restrict(O.synthesis(G, C), C)
    dense = O.dense_synthesis(G, Cd)
    assert np.abs(ring - dense).max() <= 1e-12 * np.abs(ring).max()
    g = synth.random_data(C.n_t, C.n_det, 2).astype(np.float64)
    a_ring = O.synthesis_adjoint(O.restrict_adjoint(g, C), C)
    a_dense = O.dense_synthesis_adjoint(g, Cd)
    assert np.abs(a_ring - a_dense).max() <= 1e-12 * np.abs(a_ring).max()


def test_dense_geometry_derives_and_adjoint_identity():
    n, n_det = 32, 24
    ang = _irregular_angles(n_det, 5)
    C = O.derive(n, n_det, 64, 1.0, 1.0, 2.0, ang)
    assert C.dense and C.n_ring == 32 and C.ring == ()
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    for s in range(5):
        f = synth.random_image(n, 300 + s).astype(np.float64)
        g = synth.random_data(C.n_t, n_det, 400 + s).astype(np.float64)
        Af = O.forward(f, C)
        Asg = O.adjoint(g, C)
        lhs, rhs = wY * np.sum(Af * g), wX * np.sum(f * Asg)
        assert abs(lhs - rhs) <= 1e-12 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(g * g))


def _g_cont(a, sig, x0, z, t):
    rho = np.hypot(z[0] - x0[0], z[1] - x0[1])
    f = lambda lam: lam * np.exp(-sig * sig * lam * lam / 2) * special.j0(lam * rho) * np.cos(lam * t)
    return a * sig * sig * integrate.quad(f, 0.0, 40.0 / sig, limit=400)[0]


def test_dense_continuous_gaussian():
    """A Gaussian initial pressure at n = 64: the dense-mode A f at irregular detector positions
    matches the continuous solution within the canonical error budget (raw rel-L2 <= 1.5e-2)."""
    n, n_det, n_t = 64, 48, 64
    ang = _irregular_angles(n_det, 9)
    C = O.derive(n, n_det, n_t, 1.0, 1.0, 2.0, ang)
    assert C.dense
    x = (np.arange(n) - n // 2) * C.h
    X, Y = np.meshgrid(x, x)
    a, sig, x0 = 1.0, 0.07, (0.2, -0.15)
    f = a * np.exp(-((X - x0[0]) ** 2 + (Y - x0[1]) ** 2) / (2 * sig * sig))
    g = O.forward(f, C)
    ts = (np.arange(n_t) + 1) * C.dt
    sel_t = np.arange(3, n_t, 6)
    sel_d = np.arange(0, n_det, 5)
    ref = np.array([[_g_cont(a, sig, x0, (np.cos(ang[d]), np.sin(ang[d])), ts[m]) for d in sel_d]
                    for m in sel_t])
    got = g[np.ix_(sel_t, sel_d)]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1.5e-2
