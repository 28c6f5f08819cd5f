"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no spectra, no interpolation, no
Bessel functions).  It only draws phantoms and describes acquisition geometries,
following the workload recipe of BASELINE.json ``configs`` and SURVEY.md §8(d)
("Synthetic inputs").  Both the oracle side and the CUDA side import it; neither
imports the other.

Grid convention (reading G1): pixel (iy, ix) of an n x n image sits at
x = (ix - n/2) h, y = (iy - n/2) h with h = 2/n, so node n/2 is the origin.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Geometry", "CONFIGS", "geometry", "grid", "gaussians", "ellipses",
    "phantom_batch", "noise_like", "ring_angles",
]

MASK_RADIUS = 0.95      # f = 0 where |x| > 0.95 (SURVEY §8(d) common rules)
CENTRE_RADIUS = 0.7     # centres uniform by area in r <= 0.7 (BASELINE.json configs)


@dataclass(frozen=True)
class Geometry:
    """Acquisition geometry: the scalar arguments of tat_plan_create plus the angles."""
    n: int
    n_det: int
    n_t: int
    R: float = 1.0
    c: float = 1.0
    T: float = 2.0
    batch: int = 1
    angles: tuple = field(default=(), repr=False)   # radians, CCW from +x, length n_det

    def angles_array(self) -> np.ndarray:
        return np.asarray(self.angles, dtype=np.float64)


def ring_angles(n_det: int, n_ring: int | None = None, first: int = 0) -> tuple:
    """Detector angles theta_d = 2*pi*r_d/n_ring, r_d = (first + d) mod n_ring (float64)."""
    n_ring = n_det if n_ring is None else n_ring
    r = (first + np.arange(n_det)) % n_ring
    return tuple(float(v) for v in 2.0 * np.pi * r / n_ring)


def _arc_angles_270(n_det: int) -> tuple:
    """C5: 768 detectors over a 270 deg arc centred on +y, endpoint-exclusive (reading G3):
    theta_d = -45 deg + d * 270 deg / n_det, which is the ring subset r_d = (896 + d) mod 1024."""
    return tuple(float(v) for v in (-0.25 * np.pi + np.arange(n_det) * (1.5 * np.pi / n_det)))


def geometry(name: str) -> Geometry:
    """The five BASELINE.json workloads (C1..C5) plus small test geometries."""
    if name == "C1":
        return Geometry(64, 64, 128, batch=1, angles=ring_angles(64))
    if name == "C2":
        return Geometry(256, 256, 512, batch=1, angles=ring_angles(256))
    if name == "C3":
        return Geometry(512, 512, 1024, batch=16, angles=ring_angles(512))
    if name == "C4":
        return Geometry(256, 256, 512, batch=64, angles=ring_angles(256))
    if name == "C5":
        return Geometry(1024, 768, 2048, batch=4, angles=_arc_angles_270(768))
    if name == "T32":    # brute-force / dense-transpose size (SURVEY §8(c) checks (2), (3))
        return Geometry(32, 32, 64, batch=1, angles=ring_angles(32))
    raise KeyError(name)


CONFIGS = ("C1", "C2", "C3", "C4", "C5")


def grid(n: int) -> np.ndarray:
    """Node coordinates (i - n/2) * h, h = 2/n (float64)."""
    return (np.arange(n, dtype=np.float64) - n // 2) * (2.0 / n)


def _centre(rng) -> tuple:
    u, v = rng.random(), rng.random()
    r = CENTRE_RADIUS * math.sqrt(u)
    return r * math.cos(2 * math.pi * v), r * math.sin(2 * math.pi * v)


def gaussians(n: int, count: int, rng) -> np.ndarray:
    """Sum of isotropic Gaussians a*exp(-|x-c|^2/(2 s^2)), draw order (u, v, s, a),
    s ~ U[0.02, 0.1], a ~ U[0, 1]; float64, not yet masked."""
    x = grid(n)
    X, Y = np.meshgrid(x, x, indexing="xy")     # X[iy, ix] = x_ix, Y[iy, ix] = y_iy
    f = np.zeros((n, n))
    for _ in range(count):
        cx, cy = _centre(rng)
        s = rng.uniform(0.02, 0.1)
        a = rng.uniform(0.0, 1.0)
        f += a * np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2 * s * s))
    return f


def ellipses(n: int, count: int, rng) -> np.ndarray:
    """Sum of hard-edged ellipses, draw order (u, v, s1, s2, alpha, a),
    semi-axes ~ U[0.03, 0.3], angle ~ U[0, pi), amplitude ~ U[-0.5, 1]; float64, unclipped."""
    x = grid(n)
    X, Y = np.meshgrid(x, x, indexing="xy")
    f = np.zeros((n, n))
    for _ in range(count):
        cx, cy = _centre(rng)
        s1 = rng.uniform(0.03, 0.3)
        s2 = rng.uniform(0.03, 0.3)
        al = rng.uniform(0.0, math.pi)
        a = rng.uniform(-0.5, 1.0)
        ca, sa = math.cos(al), math.sin(al)
        xr = (X - cx) * ca + (Y - cy) * sa
        yr = -(X - cx) * sa + (Y - cy) * ca
        f += a * ((xr / s1) ** 2 + (yr / s2) ** 2 <= 1.0)
    return f


def _mask(f: np.ndarray) -> np.ndarray:
    x = grid(f.shape[-1])
    X, Y = np.meshgrid(x, x, indexing="xy")
    return np.where(X * X + Y * Y > MASK_RADIUS ** 2, 0.0, f)


def phantom(name: str, b: int = 0, n: int | None = None) -> np.ndarray:
    """Image b of workload `name` as float32 (the exact array both sides consume)."""
    g = geometry(name) if name in CONFIGS or name == "T32" else None
    n = n if n is not None else g.n
    if name in ("C1", "T32"):
        rng = np.random.default_rng(0 + b)
        f = gaussians(n, 8, rng)
    elif name == "C2":
        rng = np.random.default_rng(2000 + b)
        f = np.maximum(ellipses(n, 20, rng), 0.0)
    elif name == "C3":
        rng = np.random.default_rng(3000 + b)
        f = np.maximum(ellipses(n, 20, rng), 0.0)
    elif name == "C4":
        rng = np.random.default_rng(4000 + b)
        f = gaussians(n, 8, rng) + ellipses(n, 20, rng)
        f = np.maximum(f, 0.0)
    elif name == "C5":
        rng = np.random.default_rng(5000 + b)
        f = np.maximum(ellipses(n, 20, rng), 0.0)
    else:
        raise KeyError(name)
    return _mask(f).astype(np.float32)


def phantom_batch(name: str, batch: int | None = None) -> np.ndarray:
    g = geometry(name)
    B = g.batch if batch is None else batch
    return np.stack([phantom(name, b) for b in range(B)])


def noise_like(shape, seed: int) -> np.ndarray:
    """Standard normal draws (float64) for the measurement-noise recipe
    g = A f + level * max|A f| * noise (seeds 3100+b, level 0.02)."""
    return np.random.default_rng(seed).standard_normal(shape)


def random_image(n: int, seed: int) -> np.ndarray:
    """Unstructured N(0,1) image (float32) for adjoint tests."""
    return np.random.default_rng(seed).standard_normal((n, n)).astype(np.float32)


def random_data(n_t: int, n_det: int, seed: int) -> np.ndarray:
    """Unstructured N(0,1) data (float32) for adjoint tests."""
    return np.random.default_rng(seed).standard_normal((n_t, n_det)).astype(np.float32)
