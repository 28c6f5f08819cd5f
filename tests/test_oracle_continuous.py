"""Whole-chain pins of the oracle (SURVEY §8(c) checks (1), (2), (3)).

(1) the continuous wave solution of a Gaussian initial pressure, E:kwave / E:green_conv
    (P:L210-216), evaluated by 1-D quadrature in lambda;
(2) the unaccelerated spectral propagator E:kwave evaluated exactly at the detectors
    (the paper's own verification method) on the n=32 grid;
(3) the adjoint identity of eqn:innerProducts and the dense transpose.

Error model used by the "calibrated" comparisons (reading G9 and the
bilinear window): the discrete A f ~ A_cont(K f) - (dlam^2/12) fhat_0(0), where
K(x) = sinc^2(pi x1 / 2L) sinc^2(pi x2 / 2L) is the Fourier dual of bilinear
interpolation on the Cartesian frequency grid and the constant is the Euler-Maclaurin
endpoint term of the trapezoid rule at lambda = 0.
"""
import numpy as np
import pytest
from scipy import integrate, special

import synth
from oracle import tat_oracle as O


def g_continuous(t, rho, a, s, c=1.0):
    """a s^2 int_0^inf lam exp(-s^2 lam^2/2) J0(lam rho) cos(c lam t) dlam, composite
    64-point Gauss-Legendre on [0, 40/s] (2000 panels)."""
    lmax = 40.0 / s
    nodes, wts = np.polynomial.legendre.leggauss(64)
    edges = np.linspace(0.0, lmax, 2001)
    half = (edges[1:] - edges[:-1])[:, None] / 2
    lam = ((edges[:-1, None] + edges[1:, None]) / 2 + half * nodes[None, :]).ravel()
    w = (half * wts[None, :]).ravel()
    base = w * lam * np.exp(-s * s * lam * lam / 2)
    return a * s * s * (np.cos(c * np.outer(t, lam)) * base) @ special.j0(np.outer(rho, lam)).T


def test_quadrature_matches_quad():
    a, s, t, rho = 1.0, 0.08, 1.1, 0.9
    ref, _ = integrate.quad(lambda l: l * np.exp(-s * s * l * l / 2) * special.j0(l * rho) * np.cos(l * t),
                            0, 40 / s, limit=2000, epsabs=1e-13)
    assert g_continuous(np.array([t]), np.array([rho]), a, s)[0, 0] == pytest.approx(a * s * s * ref, abs=1e-12)


def _gauss(n, a, s, x0):
    x = synth.grid(n)
    X, Y = np.meshgrid(x, x, indexing="xy")
    return a * np.exp(-((X - x0[0]) ** 2 + (Y - x0[1]) ** 2) / (2 * s * s))


def _window(C, x0):
    return np.sinc(x0[0] / (2 * C.L)) ** 2 * np.sinc(x0[1] / (2 * C.L)) ** 2


# sigma in [0.06, 0.09], |x0| <= 0.5, angular aliasing exp(-s^2 (K/|x0|)^2/2) <= 1e-3 at n=64 (G15)
GAUSSIANS = [(1.0, 0.08, (0.3, -0.2)), (0.8, 0.07, (-0.45, 0.1)), (1.0, 0.09, (0.1, 0.5))]


def _errors(C, a, s, x0):
    f = _gauss(C.n, a, s, x0)
    g = O.forward(f, C)
    th = 2 * np.pi * np.asarray(C.ring) / C.n_ring
    rho = np.hypot(C.R * np.cos(th) - x0[0], C.R * np.sin(th) - x0[1])
    t = (np.arange(C.n_t) + 1) * C.dt
    gc = g_continuous(t, rho, a, s, C.c)
    off = -(C.dlam ** 2 / 12) * a * s * s            # fhat_0(0) = a s^2 for a Gaussian
    nrm = np.linalg.norm(gc)
    raw = np.linalg.norm(g - gc) / nrm
    off_only = np.linalg.norm(g - (gc + off)) / nrm
    cal = np.linalg.norm(g - (_window(C, x0) * gc + off)) / nrm
    return raw, off_only, cal


@pytest.mark.parametrize("n", [64, 256])
def test_check1_continuous_gaussian(n):
    """Raw error is the paper's own size (0.58% L2); calibrated residual frozen at
    ~2x its first measured value (6.5e-4 at n=64, 5.8e-4 at n=256)."""
    geo = synth.Geometry(n, n, 2 * n, angles=synth.ring_angles(n))
    C = O.derive_geom(geo)
    for a, s, x0 in (GAUSSIANS if n == 64 else GAUSSIANS[:1]):
        raw, _, cal = _errors(C, a, s, x0)
        assert raw <= 1.5e-2
        assert cal <= 1.5e-3


def test_check1_refinement_in_L():
    """The bilinear-window error must fall ~4x when L goes 8 -> 16 ((pi/2L)^2 law)."""
    geo = synth.Geometry(64, 64, 128, angles=synth.ring_angles(64))
    for a, s, x0 in GAUSSIANS:
        e8 = _errors(O.derive_geom(geo), a, s, x0)[1]
        e16 = _errors(O.derive_geom(geo, L_override=16.0), a, s, x0)[1]
        assert 3.0 <= e8 / e16 <= 5.0


def _brute_force(f, C):
    """E:kwave on the Cartesian frequency grid, evaluated at the detectors:
    g(t, z) = (dxi^2 / 2pi) sum_{|xi| <= pi/h} F(xi) cos(c|xi|t) exp(i xi.z).  No polar grid,
    no Bessel functions, no cosine transform.  F from numpy.fft (not the oracle's D1)."""
    n, N = C.n, C.N
    big = np.zeros((N, N))
    idx = (np.arange(n) - n // 2) % N
    big[np.ix_(idx, idx)] = f
    A = np.fft.fft2(big) * (C.h * C.h / (2 * np.pi))
    fr = np.arange(-N // 2, N // 2)
    F = A[np.ix_(fr % N, fr % N)].T                    # F[p, q]
    XI, ETA = np.meshgrid(fr * C.dxi, fr * C.dxi, indexing="ij")
    lam = np.hypot(XI, ETA)
    msk = lam <= np.pi / C.h * (1 + 1e-12)
    th = 2 * np.pi * np.asarray(C.ring) / C.n_ring
    t = (np.arange(C.n_t) + 1) * C.dt
    ph = np.exp(1j * C.R * (np.outer(np.cos(th), XI[msk]) + np.outer(np.sin(th), ETA[msk])))
    return ((C.dxi ** 2 / (2 * np.pi)) * ((np.cos(C.c * np.outer(t, lam[msk])) * F[msk][None, :]) @ ph.T)).real


def test_check2_brute_force_kwave_n32():
    C = O.derive_geom(synth.geometry("T32"))
    n = C.n
    x = synth.grid(n)
    X, Y = np.meshgrid(x, x, indexing="xy")
    Kw = np.sinc(X / (2 * C.L)) ** 2 * np.sinc(Y / (2 * C.L)) ** 2
    for seed in (7, 8):
        rng = np.random.default_rng(seed)
        f = np.zeros((n, n))
        for _ in range(4):
            c0 = rng.uniform(-0.3, 0.3, 2)
            s = rng.uniform(2 * C.h, 4 * C.h)
            f += rng.uniform(0.5, 1) * np.exp(-((X - c0[0]) ** 2 + (Y - c0[1]) ** 2) / (2 * s * s))
        g = O.forward(f, C)
        gb = _brute_force(f, C)
        nrm = np.linalg.norm(gb)
        # reading G27: at n = 32 the raw error is dominated by the G9 trapezoid
        # offset -(dlam^2/12)(h^2/2pi) sum f, a t-independent constant fixed by the definition;
        # its size e_off is predicted here, not fitted.  Hard gates: the survey's 1.5e-2 on the
        # raw error with only that analytic constant removed, and the raw error itself within
        # e_off + 1.5e-2 (measured: 1.2e-3 .. 2.1e-3 and 1.57e-2 .. 2.15e-2 over seeds 7-16).
        off = (C.dlam ** 2 / 12) * (C.h ** 2 / (2 * np.pi)) * f.sum()
        e_off = abs(off) * np.sqrt(g.size) / nrm
        raw = np.linalg.norm(g - gb) / nrm
        assert np.linalg.norm(g - (gb - off)) / nrm <= 1.5e-2             # raw, G9 offset removed
        assert raw <= e_off + 1.5e-2                                       # raw, derived bound
        gk = _brute_force(Kw * f, C) - off
        assert np.linalg.norm(g - gk) / nrm <= 1.5e-3                       # calibrated


@pytest.mark.parametrize("name", ["T32", "C1", "C2"])
def test_check3_adjoint_identity(name):
    C = O.derive_geom(synth.geometry(name))
    wY = C.dt * 2 * np.pi * C.R / C.n_ring             # <g1,g2>_Y weight (G18)
    wX = C.h * C.h                                     # <f1,f2>_X weight
    pairs = 20 if name != "C2" else 3
    for s in range(pairs):
        f = synth.random_image(C.n, 100 + s).astype(np.float64)
        g = synth.random_data(C.n_t, C.n_det, 200 + s).astype(np.float64)
        Af = O.forward(f, C)
        Asg = O.adjoint(g, C)
        lhs = wY * np.sum(Af * g)
        rhs = wX * np.sum(f * Asg)
        assert abs(lhs - rhs) <= 1e-12 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(g * g))


def test_check3_dense_transpose_n32():
    C = O.derive_geom(synth.geometry("T32"))
    n, nt, nd = C.n, C.n_t, C.n_det
    A = np.empty((nt * nd, n * n))
    for i in range(n * n):
        e = np.zeros(n * n)
        e[i] = 1.0
        A[:, i] = O.forward(e.reshape(n, n), C).ravel()
    As = np.empty((n * n, nt * nd))
    for i in range(nt * nd):
        e = np.zeros(nt * nd)
        e[i] = 1.0
        As[:, i] = O.adjoint(e.reshape(nt, nd), C).ravel()
    assert np.abs(As - C.omega * A.T).max() <= 1e-13 * np.abs(A).max() * C.omega
