"""TEST INFRASTRUCTURE ONLY -- float64 direct-sum oracle of the paper's discrete A and A*.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs.
Shares no code with paper_2510_24687_b200 (the CUDA path); the only common module is
``synth`` (input generators).

What it computes.  Every FFT of the paper's
Algorithm 1 is written as the DFT it stands for -- a dense matrix of
roots of unity with exact integer index reduction, applied by BLAS -- so a reader can
check each line against the paper:

  D1  Alg.1 steps 1-2, F_2D convention P:L256-260:
      F[p,q] = (h^2/2pi) sum_{iy,ix} f[iy,ix] exp(-2 pi i [p(ix-n/2) + q(iy-n/2)]/N)
  D2  Alg.1 step 3 (bilinear):
      P[j,l] = bilinear interpolation of F at (u,v) = (lambda_j/dxi)(cos phi_l, sin phi_l)
  D3  Alg.1 step 4, E:eq3:   fhat_k(lambda_j) = (1/n_phi) sum_l P[j,l] e^{-i k phi_l}
  D4  E:eq2 + quadrature:    H_k(lambda_j) = i^|k| w_j dlam lambda_j J_|k|(R lambda_j) fhat_k
  D5  Alg.1 step 5, E:inverse_cos_tr:  G_k(t_m) = sum_j H_k(lambda_j) cos(c lambda_j t_m)
  D6  Alg.1 step 6, E:FourSerForg:     g(t_m, phi_l) = sum_{k=-K}^{K-1} G_k(t_m) e^{i k phi_l}
  D7  Alg.1 step 7: restriction to the detectors, real part.

The adjoint is the exact conjugate-transposed chain (reading G4), scaled to the L2 inner
products of eqn:innerProducts (reading G18):
  A* g = omega * Re( D1^H D2^T D3^H D4^H D5^T D6^H D7^T g ),  omega = dt * 2 pi R / (n_ring h^2),
which is the discrete counterpart of E:adjoint and follows Alg. 2's step
order with step 5's interpolation replaced by the transpose of Alg. 1 step 3.

Pins (tests/test_oracle_*.py): P1 numpy.fft + Gaussian closed form; P2 bilinear
exactness; P3 pure harmonics; P4 Bessel via Jacobi-Anger (E:Anger) and the J0 zero;
P5 scipy DCT-I; P6 Im A f == 0; P7 rotation/reflection equivariance; P8 delta at the
origin; (1) continuous Gaussian solution by 1-D quadrature; (2) brute-force E:kwave at
n=32; (3) adjoint identity and dense transpose.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
from scipy import special

ANGLE_TOL = 1e-9


# ----------------------------------------------------------------------------- D0
@dataclass(frozen=True)
class Constants:
    """D0 constants (readings G1, G2, G6, G7, G8, G9, G11, G15)."""
    n: int
    n_det: int
    n_t: int
    R: float
    c: float
    T: float
    h: float          # pixel pitch 2/n (G1)
    T_new: float      # model time max(2cT, 6) rounded up to M*c*dt (G7)
    L: float          # extended half-width, power of two >= T_new0 + 2 (G6)
    N: int            # Cartesian FFT size 2L/h
    dxi: float        # Cartesian frequency pitch pi/L
    dt: float         # time step T/n_t (G2)
    M: int            # DCT-I length T_new/(c dt)
    dlam: float       # radial pitch pi/T_new (G7)
    J: int            # last radial index floor(lambda_max/dlam), lambda_max = pi/h (G8)
    wJ: float         # trapezoid weight of the last node (1/2 if J dlam == lambda_max)
    n_ring: int       # canonical ring the detectors sit on (G3)
    ring: tuple       # ring index r_d of each detector
    K: int            # n_phi/2, harmonics k in [-K, K-1] (G11)
    omega: float      # L2 adjoint scale dt * 2 pi R / (n_ring h^2) (G18, G20)
    dense: bool = False   # detectors off any canonical ring (reading G24): D6/D7 as dense sums
    angles: tuple = ()    # detector angles (dense mode)

    @property
    def n_phi(self) -> int:
        return self.n_ring

    @property
    def NL(self) -> int:
        return self.J + 1


def infer_ring(angles: np.ndarray, n_det: int) -> tuple[int, np.ndarray]:
    """Smallest n_ring (multiple of 4, >= n_det) with every angle on 2 pi r / n_ring (G3)."""
    a = np.asarray(angles, dtype=np.float64)
    start = max(4, 4 * ((n_det + 3) // 4))
    for n_ring in range(start, 65537, 4):
        x = a * n_ring / (2.0 * np.pi)
        r = np.rint(x)
        if np.all(np.abs(x - r) * (2.0 * np.pi / n_ring) < ANGLE_TOL):
            ring = np.mod(r.astype(np.int64), n_ring)
            if len(np.unique(ring)) != len(ring):
                raise ValueError("detectors are not distinct ring positions")
            return n_ring, ring
    raise ValueError("detector angles are not on a canonical uniform ring")


def derive(n, n_det, n_t, R, c, T, angles, L_override: float | None = None) -> Constants:
    """D0: every constant of the discretisation, in float64.

    ``L_override`` exists only for the oracle-only refinement study of check (1)."""
    if n < 8 or n % 2:
        raise ValueError("n must be even and >= 8")
    h = 2.0 / n
    T_new0 = max(2.0 * c * T, 6.0)
    L = float(2 ** math.ceil(math.log2(T_new0 + 2.0) - 1e-12))   # P:L531-533, G6
    if L_override is not None:
        L = float(L_override)
    N = int(round(2 * L / h))
    dxi = math.pi / L                                            # 2 pi / (N h)
    dt = T / n_t                                                 # t_m = (m+1) dt, G2
    M = int(math.ceil(T_new0 / (c * dt) - 1e-9))
    T_new = M * c * dt
    dlam = math.pi / T_new                                       # G7
    lam_max = math.pi / h                                        # G8
    J = int(math.floor(lam_max / dlam + 1e-9))
    wJ = 0.5 if abs(J * dlam - lam_max) <= 1e-9 * lam_max else 1.0
    a = np.asarray(angles, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise ValueError("detector angles must be finite")
    dense = False
    try:
        n_ring, ring = infer_ring(a, n_det)
    except ValueError:
        # reading G24: detectors off every canonical ring -> polar grid n_phi = the smallest
        # power of two >= max(n_det, 8); synthesis/analysis at the exact angles (dense sums)
        n_ring, ring, dense = max(8, 1 << int(math.ceil(math.log2(max(n_det, 1))))), (), True
    K = n_ring // 2
    omega = dt * 2.0 * math.pi * R / (n_ring * h * h)
    return Constants(n, n_det, n_t, R, c, T, h, T_new, L, N, dxi, dt, M, dlam, J, wJ,
                     n_ring, tuple(int(r) for r in ring), K, omega, dense,
                     tuple(float(x) for x in a) if dense else ())


def derive_geom(geom, **kw) -> Constants:
    return derive(geom.n, geom.n_det, geom.n_t, geom.R, geom.c, geom.T, geom.angles_array(), **kw)


# ----------------------------------------------------------------------------- helpers
@lru_cache(maxsize=None)
def _roots(Nr: int) -> np.ndarray:
    """exp(-2 pi i r / Nr) for r = 0..Nr-1 in float64 (index-reduced twiddle table)."""
    r = np.arange(Nr, dtype=np.float64)
    return np.cos(2 * np.pi * r / Nr) - 1j * np.sin(2 * np.pi * r / Nr)


def _dft_matrix(freqs: np.ndarray, pos: np.ndarray, Nr: int, sign: int = -1) -> np.ndarray:
    """E[a, b] = exp(sign * 2 pi i freqs[a] * pos[b] / Nr), exponent reduced mod Nr in integers."""
    idx = np.mod(np.outer(freqs.astype(np.int64), pos.astype(np.int64)), Nr)
    E = _roots(Nr)[idx]
    return E if sign < 0 else np.conj(E)


def _freqs(N: int) -> np.ndarray:
    return np.arange(-N // 2, N // 2, dtype=np.int64)


def _unit_circle(n_phi: int) -> tuple[np.ndarray, np.ndarray]:
    """(cos phi_l, sin phi_l), phi_l = 2 pi l / n_phi, quadrant-reduced so that multiples of
    pi/2 are exactly 0 and +-1."""
    l = np.arange(n_phi)
    if n_phi % 4 == 0:
        Q = n_phi // 4
        qd, rem = l // Q, l % Q
        base = 2 * np.pi * rem / n_phi
        c0, s0 = np.cos(base), np.sin(base)
        cs = np.choose(qd, [c0, -s0, -c0, s0])
        sn = np.choose(qd, [s0, c0, -s0, -c0])
        return cs, sn
    return np.cos(2 * np.pi * l / n_phi), np.sin(2 * np.pi * l / n_phi)


def _i_pow(k: np.ndarray) -> np.ndarray:
    """i^|k| exactly."""
    return np.array([1, 1j, -1, -1j])[np.abs(k) % 4]


# ----------------------------------------------------------------------------- D1
def cartesian_spectrum(f: np.ndarray, C: Constants) -> np.ndarray:
    """D1, Alg. 1 steps 1-2 with the F_2D convention of P:L256-260.

    Returns F[p + N/2, q + N/2] for p, q in [-N/2, N/2): p pairs with x (column index ix),
    q with y (row index iy).  Zero-extension to the box [-L, L]^2 is implicit: the sum runs
    over the image nodes only."""
    n, N = C.n, C.N
    pos = np.arange(n) - n // 2
    E = _dft_matrix(_freqs(N), pos, N)              # E[p, i] = exp(-2 pi i p (i - n/2)/N)
    scale = C.h * C.h / (2 * np.pi)
    return scale * (E @ (np.asarray(f, np.float64).T @ E.T))   # F[p,q] = s sum E[p,ix] f[iy,ix] E[q,iy]


def cartesian_spectrum_adjoint(Ft: np.ndarray, C: Constants) -> np.ndarray:
    """D1^H: f~[iy, ix] = (h^2/2pi) sum_{p,q} Ft[p,q] exp(+2 pi i [p(ix-n/2) + q(iy-n/2)]/N)."""
    n, N = C.n, C.N
    pos = np.arange(n) - n // 2
    E = _dft_matrix(_freqs(N), pos, N)
    scale = C.h * C.h / (2 * np.pi)
    G = E.conj().T @ Ft @ E.conj()                   # G[ix, iy]
    return scale * G.T


# ----------------------------------------------------------------------------- D2
def polar_nodes(C: Constants):
    """Polar nodes in Cartesian index units: (u, v) = (lambda_j / dxi)(cos phi_l, sin phi_l)."""
    j = np.arange(C.J + 1, dtype=np.float64)
    rho = (j * C.L) / C.T_new                         # lambda_j / dxi = j dlam / dxi
    cs, sn = _unit_circle(C.n_phi)
    return rho[:, None] * cs[None, :], rho[:, None] * sn[None, :]


def polar_cells(C: Constants):
    """Bilinear cells of the polar nodes (j, l), j in [0, J], l in [0, n_phi):
    u = (lambda_j/dxi) cos phi_l, v = (lambda_j/dxi) sin phi_l, p0 = floor(u), alpha = u - p0,
    q0 = floor(v), beta = v - q0 (reading G13)."""
    u, v = polar_nodes(C)
    p0 = np.floor(u)
    q0 = np.floor(v)
    return p0.astype(np.int64), q0.astype(np.int64), u - p0, v - q0


def polar_resample(F: np.ndarray, C: Constants) -> np.ndarray:
    """D2, Alg. 1 step 3: P[j, l] on the polar grid, F periodic mod N."""
    N = C.N
    p0, q0, a, b = polar_cells(C)
    ip0 = np.mod(p0 + N // 2, N)
    ip1 = np.mod(p0 + 1 + N // 2, N)
    iq0 = np.mod(q0 + N // 2, N)
    iq1 = np.mod(q0 + 1 + N // 2, N)
    return ((1 - a) * (1 - b) * F[ip0, iq0] + a * (1 - b) * F[ip1, iq0]
            + (1 - a) * b * F[ip0, iq1] + a * b * F[ip1, iq1])


def polar_resample_transpose(Pt: np.ndarray, C: Constants) -> np.ndarray:
    """D2^T: scatter-add of Pt[j, l] into the Cartesian grid with D2's weights."""
    N = C.N
    p0, q0, a, b = polar_cells(C)
    ip0 = np.mod(p0 + N // 2, N)
    ip1 = np.mod(p0 + 1 + N // 2, N)
    iq0 = np.mod(q0 + N // 2, N)
    iq1 = np.mod(q0 + 1 + N // 2, N)
    Ft = np.zeros((N, N), dtype=np.complex128)
    np.add.at(Ft, (ip0, iq0), (1 - a) * (1 - b) * Pt)
    np.add.at(Ft, (ip1, iq0), a * (1 - b) * Pt)
    np.add.at(Ft, (ip0, iq1), (1 - a) * b * Pt)
    np.add.at(Ft, (ip1, iq1), a * b * Pt)
    return Ft


# ----------------------------------------------------------------------------- D3 / D6
def _harmonics(C: Constants) -> np.ndarray:
    return np.arange(-C.K, C.K, dtype=np.int64)


def angular_coefficients(P: np.ndarray, C: Constants) -> np.ndarray:
    """D3, E:eq3: fk[j, k+K] = (1/n_phi) sum_l P[j, l] exp(-2 pi i k l / n_phi)."""
    W = _dft_matrix(np.arange(C.n_phi), _harmonics(C), C.n_phi)      # W[l, k]
    return (P @ W) / C.n_phi


def angular_coefficients_adjoint(fkt: np.ndarray, C: Constants) -> np.ndarray:
    """D3^H: Pt[j, l] = (1/n_phi) sum_k fkt[j, k] exp(+2 pi i k l / n_phi)."""
    W = _dft_matrix(np.arange(C.n_phi), _harmonics(C), C.n_phi)
    return (fkt @ W.conj().T) / C.n_phi


def synthesis(G: np.ndarray, C: Constants) -> np.ndarray:
    """D6, E:FourSerForg: g[m, l] = sum_{k=-K}^{K-1} G[m, k] exp(+2 pi i k l / n_phi)."""
    S = _dft_matrix(_harmonics(C), np.arange(C.n_phi), C.n_phi, sign=+1)   # S[k, l]
    return G @ S


def synthesis_adjoint(gfull: np.ndarray, C: Constants) -> np.ndarray:
    """D6^H: Gt[m, k] = sum_l gfull[m, l] exp(-2 pi i k l / n_phi)."""
    S = _dft_matrix(_harmonics(C), np.arange(C.n_phi), C.n_phi, sign=+1)
    return gfull @ S.conj().T


# ----------------------------------------------------------------------------- D4
@lru_cache(maxsize=8)
def _bessel(K: int, J: int, dlam: float, R: float) -> np.ndarray:
    lam = np.arange(J + 1) * dlam
    return special.jv(np.arange(K + 1)[:, None], R * lam[None, :])     # [|k|, j]


def multiplier_table(C: Constants) -> np.ndarray:
    """m[|k|, j] = w_j dlam lambda_j J_|k|(R lambda_j), |k| = 0..K (E:eq2 P:L463-466 with the
    trapezoid rule in lambda, readings G9, G17); real float64."""
    j = np.arange(C.J + 1)
    lam = j * C.dlam
    w = np.ones(C.J + 1)
    w[0] = 0.5
    w[C.J] = C.wJ if C.J > 0 else w[C.J]
    return (w * C.dlam * lam)[None, :] * _bessel(C.K, C.J, C.dlam, C.R)


def apply_multiplier(fk: np.ndarray, C: Constants, conj: bool = False) -> np.ndarray:
    """D4: H[j, k] = i^|k| m[|k|, j] fk[j, k]  (conj=True: D4^H with (-i)^|k|, E:Four_coef_u)."""
    k = _harmonics(C)
    m = multiplier_table(C)[np.abs(k), :].T                              # [j, k]
    ph = _i_pow(k)
    if conj:
        ph = np.conj(ph)
    return fk * (m * ph[None, :])


# ----------------------------------------------------------------------------- D5
def _cos_matrix(C: Constants) -> np.ndarray:
    """cosm[m, j] = cos(c lambda_j t_m) = cos(pi j (m+1) / M), argument reduced mod 2M."""
    m1 = np.arange(1, C.n_t + 1, dtype=np.int64)
    j = np.arange(C.J + 1, dtype=np.int64)
    r = np.mod(np.outer(m1, j), 2 * C.M)
    table = np.cos(np.pi * np.arange(2 * C.M) / C.M)
    return table[r]


def cosine_transform(H: np.ndarray, C: Constants) -> np.ndarray:
    """D5, E:inverse_cos_tr: G[m, k] = sum_j cos(c lambda_j t_m) H[j, k]."""
    return _cos_matrix(C) @ H


def cosine_transform_adjoint(Gt: np.ndarray, C: Constants) -> np.ndarray:
    """D5^T: Ht[j, k] = sum_m cos(c lambda_j t_m) Gt[m, k]."""
    return _cos_matrix(C).T @ Gt


# ----------------------------------------------------------------------------- D7
def restrict(gfull: np.ndarray, C: Constants, check: bool = True) -> np.ndarray:
    """D7, Alg. 1 step 7: g[m, d] = Re g(t_m, phi_{r_d}); Im must vanish (G19)."""
    sub = gfull[:, np.asarray(C.ring)]
    if check:
        scale = max(np.abs(sub.real).max(), 1e-300)
        im = np.abs(sub.imag).max()
        if im > 1e-10 * scale:
            raise AssertionError(f"imaginary residue {im:.3e} vs {scale:.3e} (G19)")
    return sub.real


def restrict_adjoint(g: np.ndarray, C: Constants) -> np.ndarray:
    """D7^T: zero-extend detector data to the full ring (Alg. 2 step 1)."""
    out = np.zeros((g.shape[0], C.n_phi), dtype=np.complex128)
    out[:, np.asarray(C.ring)] = g
    return out


# ----------------------------------------------------------------------------- D6/D7, dense mode
def _detector_phases(C: Constants) -> np.ndarray:
    """E[k, d] = exp(i k theta_d), k in [-K, K-1] (reading G24)."""
    k = _harmonics(C).astype(np.float64)
    th = np.asarray(C.angles, dtype=np.float64)
    return np.exp(1j * np.outer(k, th))


def dense_synthesis(G: np.ndarray, C: Constants) -> np.ndarray:
    """D6+D7 at arbitrary detector angles: g[m, d] = Re sum_{k=-K}^{K-1} G[m, k] e^{i k theta_d}
    (E:FourSerForg P:L407-411 evaluated at the detectors, then D7's real part).  Off the polar
    grid the unpaired harmonic k = -K has an imaginary part; D7's Re keeps G_{-K} cos(K theta_d),
    the symmetric split of the Nyquist term (reading G24).  Im is not asserted to vanish."""
    return (G @ _detector_phases(C)).real


def dense_synthesis_adjoint(g: np.ndarray, C: Constants) -> np.ndarray:
    """(D6 D7)^H: Gt[m, k] = sum_d g[m, d] e^{-i k theta_d}."""
    return np.asarray(g, np.float64) @ _detector_phases(C).conj().T


# ----------------------------------------------------------------------------- chains
def forward_stages(f: np.ndarray, C: Constants) -> dict:
    """Algorithm 1 on one image, keeping every intermediate (full layout)."""
    st = {}
    st["F"] = cartesian_spectrum(f, C)             # steps 1-2
    st["P"] = polar_resample(st["F"], C)           # step 3
    st["fk"] = angular_coefficients(st["P"], C)    # step 4
    st["H"] = apply_multiplier(st["fk"], C)        # E:eq2 multiplier
    st["G"] = cosine_transform(st["H"], C)         # step 5
    if C.dense:                                     # steps 6-7 at arbitrary angles (G24)
        st["g"] = dense_synthesis(st["G"], C)
        return st
    st["gfull"] = synthesis(st["G"], C)            # step 6
    st["g"] = restrict(st["gfull"], C)             # step 7
    return st


def adjoint_stages(g: np.ndarray, C: Constants) -> dict:
    """Exact transpose of Algorithm 1, in Algorithm 2's step order."""
    st = {}
    if C.dense:                                                       # steps 1-2 (G24)
        st["G"] = dense_synthesis_adjoint(g, C)
    else:
        st["gfull"] = restrict_adjoint(np.asarray(g, np.float64), C)  # step 1
        st["G"] = synthesis_adjoint(st["gfull"], C)                   # step 2
    st["Hc"] = cosine_transform_adjoint(st["G"], C)                   # step 3 (cos sums)
    st["H"] = apply_multiplier(st["Hc"], C, conj=True)                # step 3 ((-i)^|k| J)
    st["P"] = angular_coefficients_adjoint(st["H"], C)                # step 4
    st["F"] = polar_resample_transpose(st["P"], C)                    # step 5 (transpose)
    st["u"] = cartesian_spectrum_adjoint(st["F"], C)                  # step 6
    st["f"] = C.omega * st["u"].real                                  # step 7, omega (G18)
    return st


def _batched(fn, x, C):
    x = np.asarray(x)
    if x.ndim == 2:
        return fn(x, C)
    return np.stack([fn(xi, C) for xi in x])


def forward(f: np.ndarray, C: Constants) -> np.ndarray:
    """A f for one image [n, n] or a batch [B, n, n]; returns [.., n_t, n_det] float64."""
    return _batched(lambda x, c: forward_stages(x, c)["g"], f, C)


def adjoint(g: np.ndarray, C: Constants) -> np.ndarray:
    """A* g for [n_t, n_det] or [B, n_t, n_det]; returns [.., n, n] float64."""
    return _batched(lambda x, c: adjoint_stages(x, c)["f"], g, C)


# ---------------------------------------------------------------------------------------------
# Low-harmonic quadrature variant (reading G25).  PAPER.md L510-513: for
# k in {-1, 0, 1} "a quadrature rule with discretization points clustering toward lambda = 0".
# The paper gives no law or node count.  Reading G25: the variant adds what such a rule
# converges to, the Euler-Maclaurin endpoint term of the trapezoid rule at lambda = 0,
#     int_0^Lam phi = sum_j w_j dlam phi(lambda_j) + (dlam^2/12) phi'(0) + O(dlam^4),
# with phi_k(lambda) = lambda J_|k|(R lambda) fhat_k(lambda) cos(c lambda t) (D4-D5).  For k = 0,
# phi_0'(0) = fhat_0(0) = F(0, 0) = (h^2/2pi) sum f (D1 at the origin: every polar node at
# lambda = 0 is the Cartesian origin); for k = +-1, phi ~ lambda^3 and the term vanishes.  So
# G_0(t) gains the constant (dlam^2/12)(h^2/2pi) sum f, and D6-D7 carry it unchanged to every
# (t_m, detector).  The adjoint gains the transpose of that rank-one term, times omega.

def lowk_coefficient(C: Constants) -> float:
    """(dlam^2 / 12) (h^2 / 2 pi): the G25 constant per unit sum of f."""
    return (C.dlam ** 2 / 12.0) * (C.h * C.h / (2.0 * math.pi))


def forward_lowk(f: np.ndarray, C: Constants) -> np.ndarray:
    """A f with the G25 low-harmonic quadrature: forward(f) + c_G25 sum(f) on every sample."""
    f = np.asarray(f, np.float64)
    s = f.sum(axis=(-2, -1))
    return forward(f, C) + (lowk_coefficient(C) * s)[..., None, None]


def adjoint_lowk(g: np.ndarray, C: Constants) -> np.ndarray:
    """The L2 adjoint of forward_lowk: adjoint(g) + omega c_G25 sum(g) on every pixel."""
    g = np.asarray(g, np.float64)
    s = g.sum(axis=(-2, -1))
    return adjoint(g, C) + (C.omega * lowk_coefficient(C) * s)[..., None, None]


# ---------------------------------------------------------------------------------------------
# De-apodised bilinear variant (reading G26; not in the paper).  Bilinear
# interpolation of F on the Cartesian frequency grid (pitch dxi = pi/L, D2) is, to leading order,
# the exact polar sampling of the transform of K f, K(x) = sinc^2(x1/2L) sinc^2(x2/2L) with
# sinc(u) = sin(pi u)/(pi u) (the Fourier dual of the hat kernel; DESIGN G9 error model).  The
# variant pre-divides f by K on the image nodes: A_D = A D, D = diag(1/K(x)), so A_D f ~ A_cont f.
# Its L2 adjoint (the X inner product has a constant weight) is D A*.

def deapod_weights(C: Constants) -> np.ndarray:
    """D[iy, ix] = 1 / (K(x_ix) K(y_iy)), x_i = (i - n/2) h (the D1 node positions)."""
    x = (np.arange(C.n) - C.n // 2) * C.h
    k = np.sinc(x / (2.0 * C.L)) ** 2
    return 1.0 / np.outer(k, k)


def forward_variant(f: np.ndarray, C: Constants, lowk: bool = False, deapod: bool = False) -> np.ndarray:
    """A with the f4 variants: fd = D f (deapod), then forward (+ the G25 term on fd if lowk)."""
    f = np.asarray(f, np.float64)
    fd = f * deapod_weights(C) if deapod else f
    return forward_lowk(fd, C) if lowk else forward(fd, C)


def adjoint_variant(g: np.ndarray, C: Constants, lowk: bool = False, deapod: bool = False) -> np.ndarray:
    """The L2 adjoint of forward_variant: (adjoint_lowk or adjoint)(g), then times D."""
    u = adjoint_lowk(g, C) if lowk else adjoint(g, C)
    return u * deapod_weights(C) if deapod else u


# ---------------------------------------------------------------------------------------------
# Iterative reconstruction: NNLS as projected gradient descent,
# PAPER.md §4.2 "Reconstruction methods" L838-850, with the gradient of the data fidelity
# E:operators (L164-167): grad ||A f - g||^2 = 2 A*(A f - g).
#     f^(k+1/2) = f^(k) - lambda A*(A f^(k) - g)             (L841-843)
#     f^(k+1)   = Pi_Omega0 max(0, f^(k+1/2))                (eq:NNLS-projstep L845,
#                                                             eqn:projectionHalfCircle L848-850)
# Pi_Omega0 is a 0/1 mask over the pixels (None: the whole image).  f^(0) = 0 in the paper.

def nnls(g_obs: np.ndarray, f0: np.ndarray, C: Constants, lam: float, iters: int,
         nonneg: bool = True, roi: np.ndarray | None = None) -> np.ndarray:
    f = np.array(f0, dtype=np.float64)
    for _ in range(iters):
        f = f - lam * adjoint(forward(f, C) - g_obs, C)              # L841-843
        if nonneg:
            f = np.maximum(f, 0.0)                                     # L845
        if roi is not None:
            f = f * roi                                                # L848-850
    return f


def nnls_converge(g_obs: np.ndarray, f0: np.ndarray, C: Constants, lam: float, max_iters: int,
                  rel_tol: float = 3e-3, check_every: int = 1, nonneg: bool = True,
                  roi: np.ndarray | None = None) -> tuple[np.ndarray, int]:
    """The NNLS iteration above with the paper's stopping criterion (§4.3:
    "the L2 norm of an update to the current approximation is smaller than 0.3% of the L2 norm
    of the very first (non-zero) approximation"), reading G28: the first iterate f^k0 (k0 >= 1)
    with ||f^k0|| > 0 fixes s = ||f^k0||; the iteration stops after the first checked k > k0
    with ||f^k - f^(k-1)|| < rel_tol s.  Iterations are checked until s is known, then every
    check_every-th (k % check_every == 0).  Returns (f, k), or (f, -max_iters) if the rule
    was not met."""
    f = np.array(f0, dtype=np.float64)
    scale = 0.0
    for k in range(1, max_iters + 1):
        prev = f
        f = f - lam * adjoint(forward(f, C) - g_obs, C)              # L841-843
        if nonneg:
            f = np.maximum(f, 0.0)                                     # L845
        if roi is not None:
            f = f * roi                                                # L848-850
        if scale == 0.0:
            scale = float(np.linalg.norm(f))
        elif k % check_every == 0 and np.linalg.norm(f - prev) < rel_tol * scale:
            return f, k
    return f, -max_iters


def power_norm(C: Constants, v0: np.ndarray, iters: int) -> float:
    """Largest eigenvalue of A*A (self-adjoint in X; eqn:innerProducts P:L217-222) by power
    iteration from v0: the last Rayleigh quotient <v, A*A v> / <v, v>.  The NNLS step must
    satisfy 0 < lambda < 2 / lambda_max for the projected gradient to be a descent method."""
    v = np.array(v0, dtype=np.float64)
    lam = 0.0
    for _ in range(iters):
        v = v / np.linalg.norm(v)
        u = adjoint(forward(v, C), C)
        lam = float(np.sum(v * u))
        v = u
    return lam


# ---------------------------------------------------------------------------------------------
# Inverse A^{-1}: PAPER.md §3.3 "Inverse operator" L703-784, Algorithm 3,
# E:approx_UBP (L721-726), E:Four_ser_v / E:Four_coef_v (L733-739), E:silly_integral (L747-749);
# derivation in the Appendix (L1174-1249) for R = c = 1.
#
# Reading G21: E:Four_coef_v's prefactor -4 pi inherits the 2 pi of E:Fourier_Green
# (reading G5: under the paper's F_2D convention P:L256-260, G = F^{-1}_2D(sin|xi|t / (2 pi |xi|)));
# with the consistent Green's function the coefficient is
#     vhat_k(lambda) = -2 (-i)^|k| J'_|k|(lambda) int_0^T g_k(t) sin(lambda t) dt.
# The scale is pinned by A^{-1} A f ~ f (tests/test_oracle_inverse.py); -4 pi gives 2 pi f.
#
# Discretisation (the forward's grids, Alg. 3 "same sizes of grids ... as for A*" L743-745):
#   1-2  g_k(t_m) = (1/n_phi) sum_l ghat(t_m, phi_l) e^{-i k phi_l}, ghat zero off the detectors
#   3    vhat_k(lambda_j) = -2 (-i)^|k| J'_|k|(lambda_j) dt sum_m g_k(t_m) sin(lambda_j t_m)
#        (rectangle rule on t_m = (m+1) dt, reading G18), J'_0 = -J_1,
#        J'_m = (J_{m-1} - J_{m+1}) / 2 (the identities quoted in the Appendix)
#   4    vhat(lambda_j, phi_l) = sum_{k=-K}^{K-1} vhat_k(lambda_j) e^{i k phi_l}
#   5    bilinear interpolation in (lambda, phi) to the Cartesian nodes xi_pq = dxi (p, q) with
#        |xi| < lambda_max (zero elsewhere; reading G22)
#   6    v(x) = (dxi^2 / 2 pi) Re sum_{p,q} vhat(xi_pq) e^{i xi_pq . x} at the image nodes
#   7    C = -mean of v over the image nodes with r0 < |x| < R (Omega \ Omega_0, open at the
#        detector circle; reading G23)
#   8    A^{-1} g = (v + C) on |x| <= r0, 0 elsewhere (Pi_Omega0)

def inverse_multiplier_table(C: Constants) -> np.ndarray:
    """mi[|k|, j] = -2 J'_|k|(lambda_j), |k| = 0..K (step 3 without dt and the phase)."""
    lam = np.arange(C.J + 1) * C.dlam
    Jv = special.jv(np.arange(C.K + 2)[:, None], lam[None, :])
    Jp = np.empty((C.K + 1, C.J + 1))
    Jp[0] = -Jv[1]
    Jp[1:] = 0.5 * (Jv[0:C.K] - Jv[2:C.K + 2])
    return -2.0 * Jp


def _sin_matrix(C: Constants) -> np.ndarray:
    """sinm[m, j] = sin(c lambda_j t_m) = sin(pi j (m+1) / M), argument reduced mod 2M."""
    m1 = np.arange(1, C.n_t + 1, dtype=np.int64)
    j = np.arange(C.J + 1, dtype=np.int64)
    r = np.mod(np.outer(m1, j), 2 * C.M)
    table = np.sin(np.pi * np.arange(2 * C.M) / C.M)
    return table[r]


def cartesian_polar_cells(C: Constants):
    """Step 5 cells: for every Cartesian node (p, q) (centred indices, [N, N]) the polar cell
    (j0, l0) and bilinear fractions (a, b) of rho = |xi| / dlam and theta / (2 pi / n_phi),
    plus the mask rho < J."""
    N = C.N
    p = np.arange(N) - N // 2
    Pg, Qg = np.meshgrid(p, p, indexing="ij")
    rho = np.hypot(Pg.astype(np.float64), Qg.astype(np.float64)) * (C.dxi / C.dlam)
    th = np.mod(np.arctan2(Qg.astype(np.float64), Pg.astype(np.float64)), 2 * np.pi) * (C.n_phi / (2 * np.pi))
    inside = rho < C.J - 1e-9        # open disk: the grid holds only one side of each
                                     # axis point |xi| = lambda_max (reading G22)
    j0 = np.minimum(np.floor(rho), C.J - 1).astype(np.int64)
    a = np.where(inside, rho - j0, 0.0)
    l0f = np.floor(th)
    b = th - l0f
    l0 = np.mod(l0f.astype(np.int64), C.n_phi)
    return j0, l0, a, b, inside


def polar_to_cartesian(vpol: np.ndarray, C: Constants) -> np.ndarray:
    """Step 5 (Alg. 3): V[p + N/2, q + N/2] from vpol[j, l]."""
    j0, l0, a, b, inside = cartesian_polar_cells(C)
    j0c = np.where(inside, j0, 0)
    l1 = np.mod(l0 + 1, C.n_phi)
    V = ((1 - a) * (1 - b) * vpol[j0c, l0] + a * (1 - b) * vpol[j0c + 1, l0]
         + (1 - a) * b * vpol[j0c, l1] + a * b * vpol[j0c + 1, l1])
    return np.where(inside, V, 0.0)


def inverse(g: np.ndarray, C: Constants, r0: float) -> np.ndarray:
    """A^{-1} g for one data set [n_t, n_det] (Algorithm 3, steps 1-8 above); [n, n] float64."""
    if C.R != 1.0 or C.c != 1.0:
        raise NotImplementedError("the paper derives A^{-1} for R = c = 1 (Appendix)")
    if C.dense:
        raise NotImplementedError("A^{-1} needs detectors on a canonical ring")
    if not (0.0 < r0 < C.R):
        raise ValueError("r0 must lie in (0, R)")
    gfull = restrict_adjoint(np.asarray(g, np.float64), C)                 # step 1
    gk = synthesis_adjoint(gfull, C) / C.n_phi                              # step 2 [m, k]
    sk = C.dt * (_sin_matrix(C).T @ gk)                                     # step 3 [j, k]
    k = _harmonics(C)
    mi = inverse_multiplier_table(C)[np.abs(k), :].T                        # [j, k]
    vk = mi * np.conj(_i_pow(k))[None, :] * sk                              # (-i)^|k|
    vpol = synthesis(vk, C)                                                 # step 4 [j, l]
    V = polar_to_cartesian(vpol, C)                                         # step 5
    n, N = C.n, C.N
    pos = np.arange(n) - n // 2
    E = _dft_matrix(_freqs(N), pos, N)
    v = (C.dxi ** 2 / (2 * np.pi)) * (E.conj().T @ V @ E.conj())           # step 6 [ix, iy]
    v = v.T.real
    x = pos * C.h
    X, Y = np.meshgrid(x, x)
    r = np.hypot(X, Y)
    ann = (r > r0) & (r < C.R)
    Cc = -v[ann].mean() if ann.any() else 0.0                               # step 7
    return np.where(r <= r0, v + Cc, 0.0)                                   # step 8


def inverse_batch(g: np.ndarray, C: Constants, r0: float) -> np.ndarray:
    g = np.asarray(g)
    if g.ndim == 2:
        return inverse(g, C, r0)
    return np.stack([inverse(gi, C, r0) for gi in g])
