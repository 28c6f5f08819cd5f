"""Pins of the float64 oracle against things other than itself.

Each test names the paper passage it checks and the independent truth it uses: a
library routine computing the same quantity a different way, a closed form, an
exactness class, a symmetry, or a textbook value from tests/golden/.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import fft as sfft

import synth
from oracle import tat_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _C(name, **kw):
    return O.derive_geom(synth.geometry(name), **kw)


def _gauss_image(n, a, s, x0):
    x = synth.grid(n)
    X, Y = np.meshgrid(x, x, indexing="xy")
    return a * np.exp(-((X - x0[0]) ** 2 + (Y - x0[1]) ** 2) / (2 * s * s))


def jacobi_anger_J(k, x, extra=64):
    """J_k(x) from the Jacobi-Anger expansion E:Anger: the k-th Fourier
    coefficient of e^{i x sin tau}, by the trapezoid rule on M >= 2(x+k)+64 nodes
    (exponentially accurate for periodic integrands).  Independent of scipy."""
    k = np.atleast_1d(np.asarray(k))
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    M = int(2 * (x.max() + k.max()) + extra)
    tau = 2 * np.pi * np.arange(M) / M
    out = np.empty((k.size, x.size))
    for i, kk in enumerate(k):
        out[i] = np.cos(np.outer(x, np.sin(tau)) - kk * tau[None, :]).mean(axis=1)
    return out


# --------------------------------------------------------------------------- D0
def test_grid_rules_match_paper():
    """P:L509 T_new = max(2T,6); P:L531-533 L ~ T_new + 2; §4.1 grid coincidence (G7)."""
    gold = json.load(open(os.path.join(GOLDEN, "paper_grid_rules.json")))
    for T, Tn in gold["T_new_examples"]:
        n_t = 512
        C = O.derive(256, 8, n_t, 1.0, 1.0, T, synth.ring_angles(8))
        assert C.T_new == pytest.approx(Tn, rel=1e-12)
        assert C.L >= Tn + 2 and C.L < 2 * (Tn + 2)
        assert 2 * (C.L - 1) > C.T_new           # T_refl > T_new
    s = gold["section_4_1"]
    # the paper's 513 samples on [0,4] include t=0; ours are t_m=(m+1)T/n_t (G2): n_t = 512
    C = O.derive(256, 360, s["n_time_samples_on_0_T"] - 1, 1.0, 1.0, s["T"],
                 synth.ring_angles(360))
    assert C.dt == pytest.approx(C.h)
    assert C.M == 1024 and C.J == C.M            # M dlam = pi/h exactly (reading G7)
    assert C.n_ring == 360 and C.K == 180


def test_constants_of_configs():
    """N = 8n, N_lambda = 3n+1, M = 6n, K+1 = n_ring/2+1."""
    for name, n_ring in [("C1", 64), ("C2", 256), ("C3", 512), ("C4", 256), ("C5", 1024)]:
        g = synth.geometry(name)
        C = _C(name)
        assert (C.N, C.J, C.M, C.n_ring, C.K) == (8 * g.n, 3 * g.n, 6 * g.n, n_ring, n_ring // 2)
        assert C.wJ == 0.5
    C5 = _C("C5")
    assert C5.ring == tuple((896 + d) % 1024 for d in range(768))


def test_ring_rejection():
    with pytest.raises(ValueError):
        O.infer_ring(np.array([0.0, 0.1234567, 1.0]), 3)


# --------------------------------------------------------------------------- P1 (D1)
def test_P1_cartesian_spectrum_vs_numpy_fft():
    C = _C("C1")
    f = synth.phantom("C1").astype(np.float64)
    F = O.cartesian_spectrum(f, C)
    n, N = C.n, C.N
    big = np.zeros((N, N))
    idx = (np.arange(n) - n // 2) % N
    big[np.ix_(idx, idx)] = f                                  # big[y mod N, x mod N]
    A = np.fft.fft2(big) * (C.h * C.h / (2 * np.pi))           # A[q mod N, p mod N]
    fr = np.arange(-N // 2, N // 2) % N
    ref = A[np.ix_(fr, fr)].T                                  # ref[p, q]
    assert np.abs(F - ref).max() <= 1e-12 * np.abs(ref).max()


def test_P1_cartesian_spectrum_gaussian_closed_form():
    """F_2D of a Gaussian: a s^2 exp(-s^2|xi|^2/2) exp(-i xi.x0)."""
    geo = synth.Geometry(256, 8, 512, angles=synth.ring_angles(8))
    C = O.derive_geom(geo)
    for a, s, x0 in [(1.0, 3 * C.h, (0.31, -0.22)), (0.7, 0.05, (-0.4, 0.25))]:
        F = O.cartesian_spectrum(_gauss_image(C.n, a, s, x0), C)
        xi = np.arange(-C.N // 2, C.N // 2) * C.dxi
        XI, ETA = np.meshgrid(xi, xi, indexing="ij")
        ref = a * s * s * np.exp(-s * s * (XI ** 2 + ETA ** 2) / 2) * np.exp(-1j * (XI * x0[0] + ETA * x0[1]))
        assert np.abs(F - ref).max() <= 1e-10 * np.abs(ref).max()


def test_P1_delta_is_flat():
    C = _C("C1")
    f = np.zeros((C.n, C.n))
    f[C.n // 2, C.n // 2] = 1.0
    F = O.cartesian_spectrum(f, C)
    assert np.abs(F - C.h * C.h / (2 * np.pi)).max() <= 1e-16


# --------------------------------------------------------------------------- P2 (D2)
def test_P2_bilinear_exact_on_bilinear_functions():
    C = _C("C1")
    N = C.N
    p = np.arange(-N // 2, N // 2)
    Pg, Qg = np.meshgrid(p, p, indexing="ij")
    co = np.array([0.3 - 0.1j, 1.7 + 0.2j, -0.9 + 1.1j, 0.013 - 0.021j])
    F = co[0] + co[1] * Pg + co[2] * Qg + co[3] * Pg * Qg
    P = O.polar_resample(F, C)
    p0, q0, a, b = O.polar_cells(C)
    u, v = p0 + a, q0 + b
    ref = co[0] + co[1] * u + co[2] * v + co[3] * u * v
    # corners with non-zero weight must not wrap past N/2 - 1 for the function to be periodic-free
    ok = ((p0 + (a > 0)) < N // 2) & ((q0 + (b > 0)) < N // 2)
    assert ok.mean() > 0.99
    assert np.abs(P - ref)[ok].max() <= 1e-14 * np.abs(ref).max()
    assert np.all((a >= 0) & (a < 1) & (b >= 0) & (b < 1))


def test_P2_cells_dihedral_symmetry():
    """Polar node set and cells are symmetric under (u,v) -> (-u,-v) and (u,v) -> (v,-u)."""
    C = _C("C1")
    u, v = O.polar_nodes(C)
    half, quarter = C.n_phi // 2, C.n_phi // 4
    assert np.array_equal(np.roll(u, -half, axis=1), -u)
    assert np.array_equal(np.roll(v, -half, axis=1), -v)
    assert np.array_equal(np.roll(u, -quarter, axis=1), -v)
    assert np.array_equal(np.roll(v, -quarter, axis=1), u)


# --------------------------------------------------------------------------- P3 (D3, D6)
def test_P3_pure_harmonics_and_roundtrip():
    C = _C("C1")
    phi = 2 * np.pi * np.arange(C.n_phi) / C.n_phi
    P = np.stack([np.cos(3 * phi), np.sin(5 * phi) + 0.25]).astype(np.complex128)
    fk = O.angular_coefficients(P, C)
    k = np.arange(-C.K, C.K)
    ref0 = 0.5 * ((k == 3) | (k == -3))
    ref1 = 0.25 * (k == 0) + (-0.5j) * (k == 5) + (0.5j) * (k == -5)
    assert np.abs(fk[0] - ref0).max() <= 1e-14
    assert np.abs(fk[1] - ref1).max() <= 1e-14
    back = O.synthesis(fk, C)                    # sum_k fk e^{ik phi} = P
    assert np.abs(back - P).max() <= 1e-13
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((4, C.n_phi)) + 1j * rng.standard_normal((4, C.n_phi))
    ref = np.fft.fftshift(np.fft.fft(Z, axis=1), axes=1) / C.n_phi
    assert np.abs(O.angular_coefficients(Z, C) - ref).max() <= 1e-14


# --------------------------------------------------------------------------- P4 (J)
def test_P4_bessel_textbook_values():
    gold = json.load(open(os.path.join(GOLDEN, "bessel_textbook.json")))
    for z in gold["j0_zeros"]:
        assert abs(jacobi_anger_J(0, z)[0, 0]) <= 1e-14
        assert abs(O._bessel.__wrapped__(0, 1, z, 1.0)[0, 1]) <= 1e-14   # oracle's scipy route
    for k, x, val in gold["values"]:
        assert jacobi_anger_J(k, x)[0, 0] == pytest.approx(val, abs=1e-14)


def test_P4_multiplier_table_vs_jacobi_anger():
    """D4 table m[k,j] = w_j dlam lambda_j J_k(R lambda_j): J via E:Anger, not scipy."""
    for name in ["C1", "C2"]:
        C = _C(name)
        m = O.multiplier_table(C)
        j = np.arange(C.J + 1)
        lam = j * C.dlam
        w = np.ones(C.J + 1)
        w[0] = 0.5
        w[-1] = 0.5
        ks = np.arange(C.K + 1)
        Jref = jacobi_anger_J(ks, C.R * lam)
        wl = (w * C.dlam * lam)[None, :]
        # |J error| <= 1e-13 absolute (the trapezoid sum's rounding ~ sqrt(M) eps)
        assert np.abs(m - wl * Jref).max() <= 1e-13 * wl.max()
        assert np.abs(m[:, 1:] / wl[:, 1:] - Jref[:, 1:]).max() <= 1e-13


def test_P4_bessel_large_argument_and_order():
    """C5 extremes: x up to pi/h = 1024 pi, k up to 512."""
    x = np.array([1.0, 100.0, 1608.5, 2000.0])
    k = np.array([0, 1, 37, 512])
    Jr = jacobi_anger_J(k, x)
    from scipy import special
    assert np.abs(Jr - special.jv(k[:, None], x[None, :])).max() <= 1e-13
    # Neumann identity J0 + 2 sum J_2m = 1
    kk = np.arange(0, 4000, 2)
    s = special.jv(kk[:, None], x[None, :])
    assert np.abs(s[0] + 2 * s[1:].sum(axis=0) - 1).max() <= 1e-12


# --------------------------------------------------------------------------- P5 (D5)
def test_P5_cosine_transform_single_node_and_dct1():
    C = _C("C1")
    H = np.zeros((C.J + 1, 3), dtype=np.complex128)
    j0 = 17
    H[j0, 0] = 1.0
    G = O.cosine_transform(H, C)
    t = (np.arange(C.n_t) + 1) * C.dt
    assert np.abs(G[:, 0] - np.cos(C.c * j0 * C.dlam * t)).max() <= 1e-13
    rng = np.random.default_rng(5)
    Hr = rng.standard_normal(C.J + 1)
    x = np.zeros(C.M + 1)
    x[: C.J + 1] = Hr
    y = sfft.dct(x, type=1)
    mp = np.arange(1, C.n_t + 1)
    ref = (y[mp] + x[0] + (-1.0) ** mp * x[C.M]) / 2
    G = O.cosine_transform(Hr[:, None].astype(np.complex128), C)[:, 0]
    assert np.abs(G - ref).max() <= 1e-12 * np.abs(ref).max()


# --------------------------------------------------------------------------- P6, P8
def test_P6_forward_is_real():
    for name in ["C1", "T32"]:
        C = _C(name)
        st = O.forward_stages(synth.phantom(name).astype(np.float64), C)
        sub = st["gfull"][:, list(C.ring)]
        assert np.abs(sub.imag).max() <= 1e-12 * np.abs(sub.real).max()


def test_P8_delta_at_origin_closed_form():
    """f = delta at node n/2: F == h^2/2pi, only k=0 survives, so
    A delta[m, d] = (h^2/2pi) sum_j w_j dlam lambda_j J0(R lambda_j) cos(c lambda_j t_m)."""
    for name in ["C1", "T32"]:
        C = _C(name)
        f = np.zeros((C.n, C.n))
        f[C.n // 2, C.n // 2] = 1.0
        g = O.forward(f, C)
        lam = np.arange(C.J + 1) * C.dlam
        w = np.ones(C.J + 1)
        w[0] = 0.5
        w[-1] = C.wJ
        t = (np.arange(C.n_t) + 1) * C.dt
        J0 = jacobi_anger_J(0, C.R * lam)[0]
        col = (C.h ** 2 / (2 * np.pi)) * (np.cos(C.c * np.outer(t, lam)) @ (w * C.dlam * lam * J0))
        ref = np.repeat(col[:, None], C.n_det, axis=1)
        assert np.abs(g - ref).max() <= 1e-13 * np.abs(ref).max()
        rng = np.random.default_rng(11)
        gg = rng.standard_normal((C.n_t, C.n_det))
        u = O.adjoint(gg, C)
        centre = C.omega * np.sum(ref * gg)
        assert u[C.n // 2, C.n // 2] == pytest.approx(centre, rel=1e-12)


# --------------------------------------------------------------------------- P7
@pytest.mark.parametrize("name", ["T32", "C1"])
def test_P7_rotation_reflection_equivariance(name):
    C = _C(name)
    n = C.n
    f = synth.phantom(name).astype(np.float64)
    f[0, :] = 0.0
    f[:, 0] = 0.0
    g = O.forward(f, C)
    frot = np.zeros_like(f)
    frot[:, 1:] = f[n - np.arange(1, n), :].T        # f_rot[iy][ix] = f[n-ix][iy], ix >= 1
    fref = np.zeros_like(f)
    fref[1:, :] = f[n - np.arange(1, n), :]          # f_ref[iy][ix] = f[n-iy][ix]
    r = np.arange(C.n_ring)
    grot = O.forward(frot, C)
    gref = O.forward(fref, C)
    scale = np.abs(g).max()
    assert np.abs(grot - g[:, (r - C.n_ring // 4) % C.n_ring]).max() <= 1e-12 * scale
    assert np.abs(gref - g[:, (-r) % C.n_ring]).max() <= 1e-12 * scale
    # the same rotation must NOT be satisfied with the opposite sense (sign sensitivity)
    assert np.abs(grot - g[:, (r + C.n_ring // 4) % C.n_ring]).max() > 1e-3 * scale


def test_linearity():
    C = _C("T32")
    rng = np.random.default_rng(9)
    a, b = rng.standard_normal((2, C.n, C.n))
    lhs = O.forward(2.5 * a - 0.75 * b, C)
    rhs = 2.5 * O.forward(a, C) - 0.75 * O.forward(b, C)
    assert np.abs(lhs - rhs).max() <= 1e-13 * np.abs(rhs).max()
