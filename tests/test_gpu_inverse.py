"""GPU inverse A^{-1} (Algorithm 3) through the C ABI vs the float64 oracle.
Bar as the operators: rel-L2 <= 1e-4 and max|diff| <= 1e-3 max|ref| (A^{-1} is linear up to
the constant C, which is itself linear in g)."""
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


def _run(torch, geo, g, r0):
    from paper_2510_24687_b200 import Plan
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, g.shape[0], geo.angles_array())
    out = plan.inverse(torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda(), r0)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _t4(n=64):
    return synth.Geometry(n, n, 4 * n, T=4.0, batch=1, angles=synth.ring_angles(n))


@pytest.mark.parametrize("geo_name", ["T4n64", "C1", "C2"])
def test_inverse_parity(torch_cuda, geo_name):
    geo = _t4() if geo_name == "T4n64" else synth.geometry(geo_name)
    C = O.derive_geom(geo)
    gs = np.stack([synth.random_data(geo.n_t, geo.n_det, 60 + b) for b in range(2)])
    out = _run(torch_cuda, geo, gs, 0.9)
    for b in range(2):
        _check(out[b], O.inverse(gs[b].astype(np.float64), C, 0.9), f"{geo_name} A^-1 image {b}")


def test_inverse_recovers_smooth_phantom(torch_cuda):
    geo = _t4()
    C = O.derive_geom(geo)
    x = (np.arange(C.n) - C.n // 2) * C.h
    X, Y = np.meshgrid(x, x)
    f = (np.exp(-((X - 0.2) ** 2 + (Y + 0.1) ** 2) / (2 * 0.08 ** 2))
         + 0.5 * np.exp(-((X + 0.25) ** 2 + (Y - 0.2) ** 2) / (2 * 0.12 ** 2)))
    f[np.hypot(X, Y) > 0.9] = 0.0
    g = O.forward(f, C)[None]
    fr = _run(torch_cuda, geo, g, 0.9)[0]
    assert np.linalg.norm(fr - f) / np.linalg.norm(f) <= 1.2e-2


def test_inverse_full_size_c3_sampled(torch_cuda):
    """C3 (n = 512, batch 16) in the launch configuration of the operators, images 0 and 15."""
    geo = synth.geometry("C3")
    C = O.derive_geom(geo)
    f = synth.phantom_batch("C3")
    from paper_2510_24687_b200 import Plan
    torch = torch_cuda
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
    g = plan.forward(torch.from_numpy(f).cuda())
    u = plan.inverse(g, 0.95)
    torch.cuda.synchronize()
    gh, uh = g.cpu().numpy(), u.cpu().numpy()
    for b in (0, 15):
        _check(uh[b], O.inverse(gh[b].astype(np.float64), C, 0.95), f"C3 A^-1 image {b}")
