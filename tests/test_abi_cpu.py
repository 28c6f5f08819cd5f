"""Host-side checks of the C ABI (no GPU): the library loads, exports every symbol that
include/tat.h declares, validates arguments, and derives the same D0 constants and Bessel
multiplier as the oracle (computed independently: Miller recurrence vs scipy)."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import tat_oracle as O
from paper_2510_24687_b200 import tat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    return tat.load_library()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "tat.h")).read()
    declared = set(re.findall(r"\b(tat_[a-z_]+)\s*\(", hdr))
    assert declared == set(tat.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


@pytest.mark.parametrize("name", ["T32", "C1", "C2", "C3", "C4", "C5"])
def test_derived_constants_match_oracle(name):
    g = synth.geometry(name)
    info, ring, st = tat.derive(g.n, g.n_det, g.n_t, g.R, g.c, g.T, g.batch, g.angles_array())
    assert st == tat.TAT_OK
    C = O.derive_geom(g)
    for k in ("N", "J", "M", "n_ring", "K"):
        assert info[k] == getattr(C, k), k
    for k in ("L", "T_new", "dxi", "dlam", "omega", "dt", "h", "wJ"):
        assert info[k] == pytest.approx(getattr(C, k), rel=1e-14), k
    assert tuple(ring) == C.ring
    assert info["n_nodes_half"] == (C.n_ring // 2) * (C.J + 1)


def test_paper_section41_geometry_derives():
    """§4.1 grid: 360 angles -> n_ring = 360 (valid, but not a power of two)."""
    info, ring, st = tat.derive(256, 360, 512, 1.0, 1.0, 4.0, 1, synth.ring_angles(360))
    assert st == 2 and info["n_ring"] == 360 and info["M"] == 1024


@pytest.mark.parametrize("args,code", [
    (dict(n=6), 1), (dict(n=48), 1), (dict(n_det=0), 1), (dict(n_t=0), 1), (dict(batch=0), 1),
    (dict(R=float("nan")), 1), (dict(c=-1.0), 1), (dict(T=0.0), 1),
    (dict(n=2048), 2), (dict(n=16), 2),
])
def test_argument_validation(args, code):
    base = dict(n=64, n_det=64, n_t=128, R=1.0, c=1.0, T=2.0, batch=1)
    base.update(args)
    ang = synth.ring_angles(base["n_det"]) if base["n_det"] > 0 else (0.0,)
    if base["n_det"] < 1:
        base["n_det"] = 0
        ang = np.zeros(0)
    _, _, st = tat.derive(base["n"], base["n_det"], base["n_t"], base["R"], base["c"], base["T"],
                          base["batch"], np.asarray(ang, dtype=np.float64))
    assert st == code


def test_off_ring_angles_dense_mode():
    """Angles off every canonical ring select the dense mode (reading G24): n_ring = the
    smallest power of two >= max(n_det, 8), ring indices -1, same n_ring as the oracle."""
    ang = np.array([0.0, 0.1234567, 1.0, 2.0])
    info, ring, st = tat.derive(64, 4, 128, 1.0, 1.0, 2.0, 1, ang)
    assert st == 0 and info["n_ring"] == 8 and (ring == -1).all()
    C = O.derive(64, 4, 128, 1.0, 1.0, 2.0, ang)
    assert C.dense and C.n_ring == info["n_ring"]
    assert info["omega"] == pytest.approx(C.omega, rel=1e-14)
    bad = np.array(synth.ring_angles(8))
    bad[3] = np.nan
    _, _, st = tat.derive(64, 8, 128, 1.0, 1.0, 2.0, 1, bad)
    assert st == 1
    dup = np.array(synth.ring_angles(8))
    dup[3] = dup[2]
    _, _, st = tat.derive(64, 8, 128, 1.0, 1.0, 2.0, 1, dup)
    assert st == 2


@pytest.mark.parametrize("name", ["T32", "C1", "C2", "C5"])
def test_host_multiplier_matches_oracle(name):
    """Plan Bessel table (Miller recurrence, float64 -> float32) vs the oracle's scipy table."""
    g = synth.geometry(name)
    C = O.derive_geom(g)
    m = tat.host_multiplier(g.n, g.n_det, g.n_t, g.R, g.c, g.T, g.angles_array())
    ref = O.multiplier_table(C) * (C.h ** 2 / (2 * np.pi)) / C.n_phi
    assert m.shape == ref.shape
    assert np.abs(m - ref).max() <= 2e-7 * np.abs(ref).max()
    big = np.abs(ref) > 1e-3 * np.abs(ref).max()
    assert np.abs(m[big] / ref[big] - 1).max() <= 1e-6


def test_plan_create_without_device_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import ctypes
    h = ctypes.c_void_p()
    a = np.asarray(synth.ring_angles(64), dtype=np.float64)
    st = lib.tat_plan_create(ctypes.byref(h), 64, 64, 128, 1.0, 1.0, 2.0, 1,
                             a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert st == 4 and h.value is None
