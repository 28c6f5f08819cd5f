"""GPU parity of libtat (through the C ABI) against the float64 oracle.

Bar (BASELINE.json north_star): per image, rel-L2 <= 1e-4 and max|diff| <= 1e-3 max|ref| for
A and A*; the fp32 adjoint identity within 1e-5 (inner products in float64 on the host).
Inputs: the seeded synth workloads (the same fp32 arrays feed both sides).
"""
import numpy as np
import pytest

import synth
from oracle import tat_oracle as O

pytestmark = pytest.mark.gpu

REL_L2 = 1e-4
MAX_ABS = 1e-3
ADJ_TOL = 1e-5


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def _plan(geo, batch=None):
    from paper_2510_24687_b200 import Plan
    return Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T,
                geo.batch if batch is None else batch, geo.angles_array())


def _check(out, ref, what):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    mx = np.abs(out - ref).max() / np.abs(ref).max()
    assert rel <= REL_L2 and mx <= MAX_ABS, f"{what}: rel-L2 {rel:.3e}, max {mx:.3e}"
    return rel, mx


def _run(torch, plan, f=None, g=None):
    if f is not None:
        x = torch.from_numpy(np.ascontiguousarray(f, np.float32)).cuda()
        y = plan.forward(x)
    else:
        x = torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda()
        y = plan.adjoint(x)
    torch.cuda.synchronize()
    return y.cpu().numpy()


SMALL = ["T32", "C1", "C2"]


@pytest.mark.parametrize("name", SMALL)
def test_forward_adjoint_parity_small(torch_cuda, name):
    geo = synth.geometry(name)
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = synth.phantom_batch(name)
    g_gpu = _run(torch_cuda, plan, f=f)
    g_ref = O.forward(f.astype(np.float64), C)
    for b in range(geo.batch):
        _check(g_gpu[b], g_ref[b], f"{name} A image {b}")
    gr = np.stack([synth.random_data(geo.n_t, geo.n_det, 50 + b) for b in range(geo.batch)])
    u_gpu = _run(torch_cuda, plan, g=gr)
    u_ref = O.adjoint(gr.astype(np.float64), C)
    for b in range(geo.batch):
        _check(u_gpu[b], u_ref[b], f"{name} A* image {b}")


def _arc_geometry(n=64, n_det=48, n_ring=64, first=56):
    return synth.Geometry(n, n_det, 2 * n, batch=3,
                          angles=synth.ring_angles(n_det, n_ring, first))


def test_parity_arc_and_batch(torch_cuda):
    """Limited view (ring subset, as C5) with batch 3 of different images."""
    geo = _arc_geometry()
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = np.stack([synth.phantom("C1", b) for b in range(3)])
    g_gpu = _run(torch_cuda, plan, f=f)
    g_ref = O.forward(f.astype(np.float64), C)
    for b in range(3):
        _check(g_gpu[b], g_ref[b], f"arc A {b}")
    u_gpu = _run(torch_cuda, plan, g=g_ref.astype(np.float32))
    u_ref = O.adjoint(g_ref.astype(np.float32).astype(np.float64), C)
    for b in range(3):
        _check(u_gpu[b], u_ref[b], f"arc A* {b}")


@pytest.mark.parametrize("n,n_t,T", [(32, 96, 2.0), (64, 160, 2.5), (128, 256, 4.0)])
def test_parity_other_grids(torch_cuda, n, n_t, T):
    """Ragged DCT lengths (2M = 2^a 3^b), T > 3 (oversampling L = 16), n_t not 2n."""
    geo = synth.Geometry(n, n, n_t, T=T, batch=1, angles=synth.ring_angles(n))
    from paper_2510_24687_b200 import derive
    info, _, st = derive(n, n, n_t, 1.0, 1.0, T, 1, geo.angles_array())
    if st != 0:
        pytest.skip(f"geometry unsupported by the kernels (status {st})")
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = synth.phantom("C1", 0, n=n)[None]
    _check(_run(torch_cuda, plan, f=f)[0], O.forward(f[0].astype(np.float64), C), "A")
    gr = synth.random_data(n_t, n, 9)[None]
    _check(_run(torch_cuda, plan, g=gr)[0], O.adjoint(gr[0].astype(np.float64), C), "A*")


@pytest.mark.parametrize("name", ["T32", "C1", "C2"])
def test_adjoint_identity_gpu(torch_cuda, name):
    geo = synth.geometry(name)
    plan = _plan(geo, batch=1)
    C = O.derive_geom(geo)
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    for s in range(5):
        f = synth.random_image(geo.n, 300 + s)[None]
        g = synth.random_data(geo.n_t, geo.n_det, 400 + s)[None]
        Af = _run(torch_cuda, plan, f=f).astype(np.float64)
        Asg = _run(torch_cuda, plan, g=g).astype(np.float64)
        lhs = wY * np.sum(Af * g)
        rhs = wX * np.sum(f * Asg)
        bound = ADJ_TOL * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(g.astype(np.float64) ** 2))
        assert abs(lhs - rhs) <= bound, (lhs, rhs, bound)


def test_delta_and_rotation_gpu(torch_cuda):
    """P8 (delta at the origin) and P7 (quarter-turn equivariance) on the GPU path."""
    geo = synth.geometry("C1")
    C = O.derive_geom(geo)
    plan = _plan(geo)
    n = geo.n
    d = np.zeros((1, n, n), np.float32)
    d[0, n // 2, n // 2] = 1.0
    _check(_run(torch_cuda, plan, f=d)[0], O.forward(d[0].astype(np.float64), C), "delta")
    f = synth.phantom("C1")
    f[0, :] = 0
    f[:, 0] = 0
    frot = np.zeros_like(f)
    frot[:, 1:] = f[n - np.arange(1, n), :].T
    g = _run(torch_cuda, plan, f=f[None])[0]
    gr = _run(torch_cuda, plan, f=frot[None])[0]
    r = np.arange(C.n_ring)
    assert np.abs(gr - g[:, (r - C.n_ring // 4) % C.n_ring]).max() <= 1e-5 * np.abs(g).max()


def test_determinism(torch_cuda):
    geo = synth.geometry("C2")
    plan = _plan(geo)
    f = synth.phantom_batch("C2")
    g1 = _run(torch_cuda, plan, f=f)
    g2 = _run(torch_cuda, plan, f=f)
    assert np.array_equal(g1, g2)
    u1 = _run(torch_cuda, plan, g=g1)
    u2 = _run(torch_cuda, plan, g=g1)
    assert np.array_equal(u1, u2)


def test_zero_input_gives_zero(torch_cuda):
    geo = synth.geometry("C1")
    plan = _plan(geo)
    z = np.zeros((1, geo.n, geo.n), np.float32)
    assert np.all(_run(torch_cuda, plan, f=z) == 0)
    zg = np.zeros((1, geo.n_t, geo.n_det), np.float32)
    assert np.all(_run(torch_cuda, plan, g=zg) == 0)


@pytest.mark.parametrize("name,images", [("C3", [0, 7, 15]), ("C4", [0, 33, 63]), ("C5", [0, 3])])
def test_parity_full_size(torch_cuda, name, images):
    """Full BASELINE sizes in the launch configuration bench.py times (whole batch on the GPU),
    checked image by image against the oracle on sampled images."""
    geo = synth.geometry(name)
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = synth.phantom_batch(name)
    g_gpu = _run(torch_cuda, plan, f=f)
    gs = []
    for b in images:
        ref = O.forward(f[b].astype(np.float64), C)
        _check(g_gpu[b], ref, f"{name} A image {b}")
        gs.append(ref)
    u_gpu = _run(torch_cuda, plan, g=g_gpu)
    for b in images:
        ref = O.adjoint(g_gpu[b].astype(np.float64), C)
        _check(u_gpu[b], ref, f"{name} A* image {b}")


def test_parity_mixed_engines_and_arc_at_n256(torch_cuda):
    """n = 256 runs the two-stage K1/K2/K2T/K1T; n_t = n gives 2M = 6n, which runs the
    first-generation DCT kernels (r = 3); a 3/4 arc of the ring and an odd batch of 3."""
    n, n_det, n_t = 256, 192, 256
    geo = synth.Geometry(n, n_det, n_t, batch=3, angles=synth.ring_angles(n_det, 256, 224))
    from paper_2510_24687_b200 import derive
    info, _, st = derive(n, n_det, n_t, 1.0, 1.0, 2.0, 3, geo.angles_array())
    assert st == 0, "geometry must be supported"
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = np.stack([synth.phantom("C2", b, n=n) for b in range(3)])
    g_gpu = _run(torch_cuda, plan, f=f)
    for b in range(3):
        _check(g_gpu[b], O.forward(f[b].astype(np.float64), C), f"n256 arc A {b}")
    gr = np.stack([synth.random_data(n_t, n_det, 70 + b) for b in range(3)])
    u_gpu = _run(torch_cuda, plan, g=gr)
    for b in range(3):
        _check(u_gpu[b], O.adjoint(gr[b].astype(np.float64), C), f"n256 arc A* {b}")


def test_nan_propagates(torch_cuda):
    """NaN/Inf in the input propagate to the output (include/tat.h: no scan pass)."""
    geo = synth.geometry("C2")
    plan = _plan(geo, batch=1)
    f = synth.phantom("C2")[None].copy()
    f[0, geo.n // 2, geo.n // 3] = np.nan
    g = _run(torch_cuda, plan, f=f)
    assert np.isnan(g).any()
