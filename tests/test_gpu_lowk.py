"""GPU parity of the low-harmonic quadrature variant (DESIGN reading G25)
through the C ABI (tat_plan_set_quadrature) against the oracle's forward_lowk / adjoint_lowk."""
import numpy as np
import pytest

import synth
from oracle import tat_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def _check(out, ref, what):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    mx = np.abs(out - ref).max() / np.abs(ref).max()
    assert rel <= 1e-4 and mx <= 1e-3, f"{what}: rel-L2 {rel:.3e}, max {mx:.3e}"


def _geo(name, batch):
    g = synth.geometry(name)
    return synth.Geometry(g.n, g.n_det, g.n_t, g.R, g.c, g.T, batch, angles=g.angles_array())


@pytest.mark.parametrize("name,dense", [("T32", False), ("C2", False), ("T32", True)])
def test_lowk_parity_and_adjoint(torch_cuda, name, dense):
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    geo = _geo(name, 2)
    ang = (np.sort(np.random.default_rng(5).uniform(0, 2 * np.pi, geo.n_det)) if dense
           else geo.angles_array())
    C = O.derive(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, ang)
    assert C.dense == dense
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, 2, ang)
    plan.set_quadrature("lowk")
    f = np.stack([synth.phantom(name if name != "T32" else "C1", b, n=geo.n) for b in range(2)])
    gd = np.stack([synth.random_data(geo.n_t, geo.n_det, 60 + b) for b in range(2)])
    g = plan.forward(torch.from_numpy(f).cuda())
    u = plan.adjoint(torch.from_numpy(gd).cuda())
    torch.cuda.synchronize()
    gh, uh = g.cpu().numpy(), u.cpu().numpy()
    for b in range(2):
        _check(gh[b], O.forward_lowk(f[b].astype(np.float64), C), f"A_lowk {b}")
        _check(uh[b], O.adjoint_lowk(gd[b].astype(np.float64), C), f"A*_lowk {b}")
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    Af = gh.astype(np.float64)
    lhs = wY * np.sum(Af * gd)
    rhs = wX * np.sum(f.astype(np.float64) * uh)
    assert abs(lhs - rhs) <= 1e-5 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(gd.astype(np.float64) ** 2))
    # back to the base rule: the plain A again, and the variant's shift is the G25 constant
    plan.set_quadrature("trapezoid")
    g0 = plan.forward(torch.from_numpy(f).cuda()).cpu().numpy()
    for b in range(2):
        _check(g0[b], O.forward(f[b].astype(np.float64), C), f"A {b}")
        shift = (gh[b].astype(np.float64) - g0[b]).ravel()
        want = O.lowk_coefficient(C) * f[b].astype(np.float64).sum()
        assert np.abs(shift - want).max() <= 1e-3 * np.abs(gh[b]).max()


def test_lowk_driver_and_transpose(torch_cuda):
    """The variant flows into the fused driver epilogues and the autograd transpose."""
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    geo = _geo("C1", 2)
    C = O.derive_geom(geo)
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, 2, geo.angles_array())
    plan.set_quadrature("lowk")
    f = np.stack([synth.phantom("C1", b, n=geo.n) for b in range(2)])
    gobs = np.stack([synth.random_data(geo.n_t, geo.n_det, 90 + b) for b in range(2)])
    r = plan.residual(torch.from_numpy(f).cuda(), torch.from_numpy(gobs).cuda())
    wt = plan.transpose(torch.from_numpy(gobs).cuda())
    torch.cuda.synchronize()
    for b in range(2):
        ref_r = O.forward_lowk(f[b].astype(np.float64), C) - gobs[b]
        _check(r[b].cpu().numpy(), ref_r, f"residual {b}")
        _check(wt[b].cpu().numpy(), O.adjoint_lowk(gobs[b].astype(np.float64), C) / C.omega, f"A^T {b}")


@pytest.mark.parametrize("name,lowk,n_override", [("C1", False, None), ("C2", True, None),
                                                 ("C1", True, 64)])
def test_deapod_parity_and_adjoint(torch_cuda, name, lowk, n_override):
    """G26 (with and without G25) on the first-generation engine (n = 128, 64) and the
    two-stage engine (n = 256), against forward_variant / adjoint_variant."""
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    base = _geo(name, 2)
    n = n_override or base.n
    geo = synth.Geometry(n, base.n_det, base.n_t, base.R, base.c, base.T, 2, angles=base.angles)
    C = O.derive_geom(geo)
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, 2, geo.angles_array())
    plan.set_interpolation("deapod")
    if lowk:
        plan.set_quadrature("lowk")
    f = np.stack([synth.phantom("C1", b, n=n) for b in range(2)])
    gd = np.stack([synth.random_data(geo.n_t, geo.n_det, 70 + b) for b in range(2)])
    g = plan.forward(torch.from_numpy(f).cuda())
    u = plan.adjoint(torch.from_numpy(gd).cuda())
    torch.cuda.synchronize()
    gh, uh = g.cpu().numpy(), u.cpu().numpy()
    for b in range(2):
        _check(gh[b], O.forward_variant(f[b], C, lowk, True), f"A_D {b}")
        _check(uh[b], O.adjoint_variant(gd[b], C, lowk, True), f"A_D* {b}")
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    Af = gh.astype(np.float64)
    lhs = wY * np.sum(Af * gd)
    rhs = wX * np.sum(f.astype(np.float64) * uh)
    assert abs(lhs - rhs) <= 1e-5 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(gd.astype(np.float64) ** 2))


def test_variant_rules_validated(torch_cuda):
    """Unknown rules are rejected with TAT_ERR_INVALID_ARGUMENT and leave the plan unchanged."""
    from paper_2510_24687_b200 import Plan
    from paper_2510_24687_b200.tat import TatError
    geo = _geo("T32", 1)
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, 1, geo.angles_array())
    for bad in (2, -1):
        with pytest.raises(TatError) as e:
            plan.set_quadrature(bad)
        assert e.value.status == 1
        with pytest.raises(TatError) as e:
            plan.set_interpolation(bad)
        assert e.value.status == 1
    assert plan.quadrature == "trapezoid" and plan.interpolation == "bilinear"
