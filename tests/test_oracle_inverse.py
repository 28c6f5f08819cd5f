"""Pins of the oracle's A^{-1} (Alg. 3, reading G21).

  * left inverse: A^{-1} A f ~ f for smooth phantoms with full-view data and T = 4 (the
    paper's §4.1 time horizon), within the error the discretisation leaves (measured 0.58 %
    rel. L2 at n = 64; the paper reports 0.22 % / 0.9 % for its phantom at n = 257, L961-966);
    with the printed prefactor -4 pi the result is 2 pi f (reading G21);
  * J'_m from the Appendix identities vs scipy.special.jvp (an independent library route);
  * the sine sums vs scipy.fft.dst type I on the DST grid (library route);
  * exact equivariance under the quarter turn (ring shift by n_ring / 4) and the reflection
    y -> -y (ring index r -> -r), and g = 0 -> 0.
"""
import numpy as np
import pytest
from scipy import fft as sfft
from scipy import special

import synth
from oracle import tat_oracle as O


def _geom(n=64, T=4.0):
    return synth.Geometry(n, n, int(n * T), T=T, batch=1, angles=synth.ring_angles(n))


def _smooth_phantom(C):
    x = (np.arange(C.n) - C.n // 2) * C.h
    X, Y = np.meshgrid(x, x)
    f = (np.exp(-((X - 0.2) ** 2 + (Y + 0.1) ** 2) / (2 * 0.08 ** 2))
         + 0.5 * np.exp(-((X + 0.25) ** 2 + (Y - 0.2) ** 2) / (2 * 0.12 ** 2)))
    f[np.hypot(X, Y) > 0.9] = 0.0
    return f


@pytest.fixture(scope="module")
def c64():
    return O.derive_geom(_geom())


def test_left_inverse_smooth_phantom(c64):
    C = c64
    f = _smooth_phantom(C)
    fr = O.inverse(O.forward(f, C), C, 0.9)
    rel = np.linalg.norm(fr - f) / np.linalg.norm(f)
    linf = np.abs(fr - f).max() / np.abs(f).max()
    assert rel <= 1.2e-2 and linf <= 1.5e-2, (rel, linf)


def test_bessel_derivative_identities(c64):
    C = c64
    lam = np.arange(C.J + 1) * C.dlam
    ref = -2.0 * special.jvp(np.arange(C.K + 1)[:, None], lam[None, :])
    assert np.abs(O.inverse_multiplier_table(C) - ref).max() <= 1e-13


def test_sine_sums_vs_dst1(c64):
    C = c64
    S = O._sin_matrix(C)                                # [m, j]: sin(pi j (m+1) / M)
    x = synth.random_data(C.J + 1, 1, 3)[:, 0].astype(np.float64)
    y = S @ x                                           # y[m] = sum_j x_j sin(pi j (m+1)/M)
    # DST-I of length M-1 on x_1..x_{M-1} (x_j = 0 for j > J): 2 sum_j x_j sin(pi j k / M)
    xp = np.zeros(C.M - 1)
    xp[:C.J] = x[1:C.J + 1]
    d = sfft.dst(xp, type=1) / 2.0                      # k = 1..M-1
    assert np.abs(y[: min(C.n_t, C.M - 1)] - d[: min(C.n_t, C.M - 1)]).max() <= 1e-12 * np.abs(d).max()


def test_quarter_turn_and_reflection_equivariance(c64):
    C = c64
    n = C.n
    g = synth.random_data(C.n_t, C.n_det, 4).astype(np.float64)
    u = O.inverse(g, C, 0.9)
    grot = g[:, (np.arange(C.n_ring) - C.n_ring // 4) % C.n_ring]   # data of the rotated image
    urot = O.inverse(grot, C, 0.9)
    exp = np.zeros_like(u)
    exp[:, 1:] = u[n - np.arange(1, n), :].T                        # f_rot[iy][ix] = f[n-ix][iy]
    inner = np.ones((n, n), bool)
    inner[0, :] = inner[:, 0] = False
    assert np.abs(urot - exp)[inner].max() <= 1e-10 * np.abs(u).max()
    # reflection y -> -y: g_ref[m][r] = g[m][-r], f_ref[iy][ix] = f[n - iy][ix] (exact)
    gref = g[:, (-np.arange(C.n_ring)) % C.n_ring]
    uref = O.inverse(gref, C, 0.9)
    exp2 = np.zeros_like(u)
    exp2[1:, :] = u[n - np.arange(1, n), :]
    assert np.abs(uref - exp2)[inner].max() <= 1e-10 * np.abs(u).max()
    assert np.all(O.inverse(np.zeros_like(g), C, 0.9) == 0.0)
