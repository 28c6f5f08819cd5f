"""Pins of the low-harmonic quadrature variant (DESIGN reading G25) against
references that do not use it: the continuous Gaussian solution (E:kwave by 1-D quadrature), the
brute-force E:kwave on the Cartesian grid (n = 32), and the adjoint identity of
eqn:innerProducts."""
import numpy as np
import pytest

import synth
from oracle import tat_oracle as O
import test_oracle_continuous as T


def test_lowk_removes_the_endpoint_offset_continuous_gaussian():
    """Against the bilinear-window model K f (no offset term): the base trapezoid leaves the
    -(dlam^2/12) fhat_0(0) offset (~5e-3 relative here); the G25 variant must remove it, i.e.
    land at the window model's own residual (<= 1.5e-3) and gain >= 4x.  A wrong sign doubles
    the error, a wrong factor leaves >= 2.5e-3."""
    geo = synth.Geometry(64, 64, 128, angles=synth.ring_angles(64))
    C = O.derive_geom(geo)
    for a, s, x0 in T.GAUSSIANS:
        f = T._gauss(C.n, a, s, x0)
        th = 2 * np.pi * np.asarray(C.ring) / C.n_ring
        rho = np.hypot(C.R * np.cos(th) - x0[0], C.R * np.sin(th) - x0[1])
        t = (np.arange(C.n_t) + 1) * C.dt
        gc = T.g_continuous(t, rho, a, s, C.c)
        wgc = T._window(C, x0) * gc
        nrm = np.linalg.norm(gc)
        e_base = np.linalg.norm(O.forward(f, C) - wgc) / nrm
        e_lowk = np.linalg.norm(O.forward_lowk(f, C) - wgc) / nrm
        assert e_base >= 4e-3
        assert e_lowk <= 1.5e-3
        assert e_base / e_lowk >= 4.0


def test_lowk_brute_force_kwave_n32():
    """n = 32: the variant matches brute-force E:kwave of K f with no offset term (the base
    rule needs the explicit -(dlam^2/12) fhat_0(0) in test_check2)."""
    C = O.derive_geom(synth.geometry("T32"))
    n = C.n
    x = synth.grid(n)
    X, Y = np.meshgrid(x, x, indexing="xy")
    Kw = np.sinc(X / (2 * C.L)) ** 2 * np.sinc(Y / (2 * C.L)) ** 2
    rng = np.random.default_rng(9)
    f = np.zeros((n, n))
    for _ in range(4):
        c0 = rng.uniform(-0.3, 0.3, 2)
        s = rng.uniform(2 * C.h, 4 * C.h)
        f += rng.uniform(0.5, 1) * np.exp(-((X - c0[0]) ** 2 + (Y - c0[1]) ** 2) / (2 * s * s))
    gk = T._brute_force(Kw * f, C)
    nrm = np.linalg.norm(gk)
    e_lowk = np.linalg.norm(O.forward_lowk(f, C) - gk) / nrm
    e_base = np.linalg.norm(O.forward(f, C) - gk) / nrm
    assert e_lowk <= 1.5e-3
    assert e_base / e_lowk >= 2.0


@pytest.mark.parametrize("name", ["T32", "C1"])
def test_lowk_adjoint_identity(name):
    C = O.derive_geom(synth.geometry(name))
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    for s in range(5):
        f = synth.random_image(C.n, 300 + s).astype(np.float64)
        g = synth.random_data(C.n_t, C.n_det, 400 + s).astype(np.float64)
        Af = O.forward_lowk(f, C)
        Asg = O.adjoint_lowk(g, C)
        lhs = wY * np.sum(Af * g)
        rhs = wX * np.sum(f * Asg)
        assert abs(lhs - rhs) <= 1e-12 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(g * g))


def test_lowk_batched_shapes():
    C = O.derive_geom(synth.geometry("T32"))
    f = np.stack([synth.random_image(C.n, 500 + b) for b in range(2)]).astype(np.float64)
    g = O.forward_lowk(f, C)
    assert g.shape == (2, C.n_t, C.n_det)
    np.testing.assert_allclose(g[1], O.forward_lowk(f[1], C), rtol=0, atol=1e-15)


# ---- de-apodised bilinear (DESIGN reading G26)

def test_deapod_weights_are_the_window_reciprocal():
    """D is 1/K on the D1 nodes: K from the hat kernel's transform, checked against a direct
    numerical Fourier transform of the hat of width dxi (not the sinc formula)."""
    C = O.derive_geom(synth.geometry("T32"))
    D = O.deapod_weights(C)
    x = (np.arange(C.n) - C.n // 2) * C.h
    u = np.linspace(-1.0, 1.0, 40001)                   # hat(u) = 1 - |u| on [-1, 1], u = xi / dxi
    hat = 1.0 - np.abs(u)
    K = np.array([np.trapezoid(hat * np.cos(C.dxi * u * xx), u) for xx in x])   # = sinc^2(x/2L)
    np.testing.assert_allclose(D, 1.0 / np.outer(K, K), rtol=1e-7)
    assert D[C.n // 2, C.n // 2] == 1.0 and D.min() >= 1.0


def test_deapod_and_lowk_reach_the_continuous_solution():
    """With both variants the discrete A f matches the continuous Gaussian solution itself (no
    window, no offset) to the model's residual; each variant alone leaves its own error term."""
    geo = synth.Geometry(64, 64, 128, angles=synth.ring_angles(64))
    C = O.derive_geom(geo)
    for a, s, x0 in T.GAUSSIANS:
        f = T._gauss(C.n, a, s, x0)
        th = 2 * np.pi * np.asarray(C.ring) / C.n_ring
        rho = np.hypot(C.R * np.cos(th) - x0[0], C.R * np.sin(th) - x0[1])
        t = (np.arange(C.n_t) + 1) * C.dt
        gc = T.g_continuous(t, rho, a, s, C.c)
        nrm = np.linalg.norm(gc)
        e = {k: np.linalg.norm(O.forward_variant(f, C, *k) - gc) / nrm
             for k in [(False, False), (True, False), (False, True), (True, True)]}
        assert e[(True, True)] <= 1e-3                       # measured 3.7e-4 .. 7.5e-4
        assert e[(False, False)] / e[(True, True)] >= 7.0    # measured 8 .. 15x
        assert e[(True, False)] > 1.5 * e[(True, True)] and e[(False, True)] > 1.5 * e[(True, True)]


@pytest.mark.parametrize("lowk", [False, True])
def test_variant_adjoint_identity(lowk):
    C = O.derive_geom(synth.geometry("C1"))
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    for s in range(3):
        f = synth.random_image(C.n, 700 + s).astype(np.float64)
        g = synth.random_data(C.n_t, C.n_det, 800 + s).astype(np.float64)
        Af = O.forward_variant(f, C, lowk, True)
        Asg = O.adjoint_variant(g, C, lowk, True)
        lhs = wY * np.sum(Af * g)
        rhs = wX * np.sum(f * Asg)
        assert abs(lhs - rhs) <= 1e-12 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(g * g))
