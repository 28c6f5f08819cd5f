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


def _adjoint_identity(torch, plan, geo, C, f, g):
    """<A f, g>_Y = <f, A* g>_X per image (eqn:innerProducts P:L217-222, discretised as G18),
    GPU outputs, inner products in float64 on the host; bound ADJ_TOL ||A f||_Y ||g||_Y."""
    wY = C.dt * 2 * np.pi * C.R / C.n_ring
    wX = C.h * C.h
    Af = _run(torch, plan, f=f).astype(np.float64)
    Asg = _run(torch, plan, g=g).astype(np.float64)
    worst = 0.0
    for b in range(f.shape[0]):
        lhs = wY * np.sum(Af[b] * g[b].astype(np.float64))
        rhs = wX * np.sum(f[b].astype(np.float64) * Asg[b])
        bound = np.sqrt(wY * np.sum(Af[b] * Af[b])) * np.sqrt(wY * np.sum(g[b].astype(np.float64) ** 2))
        worst = max(worst, abs(lhs - rhs) / bound)
        assert abs(lhs - rhs) <= ADJ_TOL * bound, (b, lhs, rhs, bound)
    return worst


@pytest.mark.parametrize("name", ["T32", "C1", "C2"])
def test_adjoint_identity_gpu(torch_cuda, name):
    geo = synth.geometry(name)
    plan = _plan(geo, batch=1)
    C = O.derive_geom(geo)
    for s in range(5):
        f = synth.random_image(geo.n, 300 + s)[None]
        g = synth.random_data(geo.n_t, geo.n_det, 400 + s)[None]
        _adjoint_identity(torch_cuda, plan, geo, C, f, g)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_adjoint_identity_gpu_full_batch(torch_cuda, name):
    """The north star's 1e-5 adjoint test on the two-stage column engines (n = 512: C3,
    n = 256: C4, n = 1024: C5) at each configuration's own batch, a distinct random (f, g)
    per image, in the launch configuration bench.py times."""
    geo = synth.geometry(name)
    plan = _plan(geo)
    C = O.derive_geom(geo)
    f = np.stack([synth.random_image(geo.n, 600 + b) for b in range(geo.batch)])
    g = np.stack([synth.random_data(geo.n_t, geo.n_det, 700 + b) for b in range(geo.batch)])
    _adjoint_identity(torch_cuda, plan, geo, C, f, g)


def test_adjoint_identity_phantoms_c3(torch_cuda):
    """Same identity with g = A f of the C3 phantoms (structured, not white) against
    phantoms of the next seeds: the pairing bench.py's A then A* step produces."""
    geo = synth.geometry("C3")
    plan = _plan(geo)
    C = O.derive_geom(geo)
    f = synth.phantom_batch("C3")
    g = _run(torch_cuda, plan, f=np.stack([synth.phantom("C3", 16 + b) for b in range(16)]))
    _adjoint_identity(torch_cuda, plan, geo, C, f, g)


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


@pytest.mark.parametrize("name,images", [("C3", list(range(16))), ("C4", list(range(0, 64, 4))),
                                         ("C5", list(range(4)))])
def test_parity_full_size(torch_cuda, name, images):
    """Full BASELINE sizes in the launch configuration bench.py times (whole batch on the GPU),
    checked image by image against the oracle: every image of C3 and C5, 16 of C4's 64."""
    geo = synth.geometry(name)
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = synth.phantom_batch(name)
    g_gpu = _run(torch_cuda, plan, f=f)
    for b in images:
        _check(g_gpu[b], O.forward(f[b].astype(np.float64), C), f"{name} A image {b}")
    u_gpu = _run(torch_cuda, plan, g=g_gpu)
    for b in images:
        ref = O.adjoint(g_gpu[b].astype(np.float64), C)
        _check(u_gpu[b], ref, f"{name} A* image {b}")


def test_graph_replay_matches_eager_c3(torch_cuda):
    """bench.py times a CUDA-graph replay of the step (A then A*): the replayed results equal
    the eager launches bit for bit, and image 5 matches the oracle."""
    torch = torch_cuda
    geo = synth.geometry("C3")
    plan = _plan(geo)
    f = torch.from_numpy(synth.phantom_batch("C3")).cuda()
    g = torch.empty((geo.batch, geo.n_t, geo.n_det), device="cuda")
    u = torch.empty((geo.batch, geo.n, geo.n), device="cuda")
    plan.forward(f, out=g)
    plan.adjoint(g, out=u)
    torch.cuda.synchronize()
    g_eager, u_eager = g.clone(), u.clone()
    g.zero_()
    u.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        plan.forward(f, out=g)
        plan.adjoint(g, out=u)
    g.zero_()
    u.zero_()
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(g, g_eager) and torch.equal(u, u_eager)
    C = O.derive_geom(geo)
    _check(g[5].cpu().numpy(), O.forward(f[5].cpu().numpy().astype(np.float64), C), "graph A 5")
    _check(u[5].cpu().numpy(), O.adjoint(g[5].cpu().numpy().astype(np.float64), C), "graph A* 5")


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_host_buffer_abi(torch_cuda, name):
    """tat_forward_host / tat_adjoint_host (H2D + operator + D2H on the stream): the same
    kernels as the device entry points, so the results are equal bit for bit; checked against
    the oracle on one image."""
    torch = torch_cuda
    geo = synth.geometry(name)
    plan = _plan(geo)
    f = synth.phantom_batch(name)
    g_h = np.empty((geo.batch, geo.n_t, geo.n_det), np.float32)
    plan.forward_host(f, g_h)
    torch.cuda.synchronize()
    u_h = np.empty((geo.batch, geo.n, geo.n), np.float32)
    plan.adjoint_host(g_h, u_h)
    torch.cuda.synchronize()
    g_d = _run(torch, plan, f=f)
    u_d = _run(torch, plan, g=g_h)
    assert np.array_equal(g_h, g_d) and np.array_equal(u_h, u_d)
    C = O.derive_geom(geo)
    _check(g_h[-1], O.forward(f[-1].astype(np.float64), C), f"{name} host A")
    _check(u_h[-1], O.adjoint(g_h[-1].astype(np.float64), C), f"{name} host A*")


@pytest.mark.parametrize("n,n_det,n_ring,dense", [(32, 16, 16, False), (32, 8, 8, False),
                                                  (32, 12, 16, False), (32, 6, None, True),
                                                  (32, 14, None, True)])
def test_small_rings_generic_kernels(torch_cuda, n, n_det, n_ring, dense):
    """n_ring < 32 runs the generic ring kernels (kernels.cu k3_angular_mult, k5_synth_restrict,
    k5t_analysis, k3t_angular): canonical rings of 8 and 16 positions (full and partial) and
    dense-mode geometries whose polar grid has n_phi = 8 or 16, with batch 2."""
    if dense:
        ang = np.sort(np.random.default_rng(n_det).uniform(0.0, 2 * np.pi, n_det))
    else:
        ang = np.asarray(synth.ring_angles(n_det, n_ring, 3))
    geo = synth.Geometry(n, n_det, 2 * n, batch=2, angles=tuple(ang))
    C = O.derive(n, n_det, 2 * n, 1.0, 1.0, 2.0, ang)
    assert bool(C.dense) == dense and C.n_ring < 32
    plan = _plan(geo)
    f = np.stack([synth.phantom("C1", b, n=n) for b in range(2)])
    g_gpu = _run(torch_cuda, plan, f=f)
    gr = np.stack([synth.random_data(2 * n, n_det, 90 + b) for b in range(2)])
    u_gpu = _run(torch_cuda, plan, g=gr)
    for b in range(2):
        _check(g_gpu[b], O.forward(f[b].astype(np.float64), C), f"small ring A {b}")
        _check(u_gpu[b], O.adjoint(gr[b].astype(np.float64), C), f"small ring A* {b}")
    _adjoint_identity(torch_cuda, plan, geo, C, f, gr)


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


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fused_adjoint_column_stage(torch_cuda, monkeypatch, name):
    """The adjoint column stage variants: fused (TAT_K2F=1, k2c_adjf: target sums inside the
    column kernel) and the default multi-image target sums (k2t_sumf) + k2c_adj, both on the
    window-relative records.  Fused k2c_adjf: records
    staged once per column, origin columns from global memory, targets with > 2 entries summed
    by a warp in a fixed lane/butterfly order) against the two-kernel path (TAT_K2F=0:
    k2t_sum + k2c_adj, sequential sums): equal up to the summation order of those few targets
    (<= 1e-6 of max|A* g|), and bitwise reproducible run to run."""
    torch = torch_cuda
    geo = synth.geometry(name)
    plan = _plan(geo)
    monkeypatch.setenv("TAT_K2F", "0")
    plan0 = _plan(geo)
    monkeypatch.setenv("TAT_K2F", "1")
    plan1 = _plan(geo)
    monkeypatch.setenv("TAT_K2F", "2")
    plan2 = _plan(geo)
    monkeypatch.delenv("TAT_K2F")
    assert plan1.info["launches_adjoint"] == plan0.info["launches_adjoint"] - 1
    g = torch.from_numpy(np.stack([synth.random_data(geo.n_t, geo.n_det, 800 + b)
                                   for b in range(geo.batch)])).cuda()
    u0 = plan0.adjoint(g)
    for p in (plan, plan1, plan2):
        u = p.adjoint(g)
        u1 = p.adjoint(g)
        torch.cuda.synchronize()
        assert torch.equal(u, u1)
        assert (u - u0).abs().max().item() <= 1e-6 * u0.abs().max().item()


@pytest.mark.parametrize("name", ["C3", "C4", "C2", "C5"])
def test_ring_engines_agree(torch_cuda, monkeypatch, name):
    """n_phi = 512 / 256 / 1024 (C5: a 270-degree arc): the two-stage ring kernels (kernels_ring2.cu: K3 / K3T / K5 / K5T,
    TAT_RING2 bit mask; default auto) against the radix-8 Stockham ring kernels (TAT_RING2=0):
    the same transforms in a different summation order, so A f and A* g agree to fp32 rounding
    (<= 2e-6 of the maximum); the default path is the one the full-size oracle parity tests
    check."""
    torch = torch_cuda
    geo = synth.geometry(name)
    plans = {}
    for r in ("0", "15"):
        monkeypatch.setenv("TAT_RING2", r)
        plans[r] = _plan(geo)
    monkeypatch.delenv("TAT_RING2")
    plans["default"] = _plan(geo)
    f = torch.from_numpy(synth.phantom_batch(name)).cuda()
    g = torch.from_numpy(np.stack([synth.random_data(geo.n_t, geo.n_det, 900 + b)
                                   for b in range(geo.batch)])).cuda()
    a0, u0 = plans["0"].forward(f), plans["0"].adjoint(g)
    for key in ("15", "default"):
        a, u = plans[key].forward(f), plans[key].adjoint(g)
        torch.cuda.synchronize()
        assert (a - a0).abs().max().item() <= 2e-6 * a0.abs().max().item(), key
        assert (u - u0).abs().max().item() <= 2e-6 * u0.abs().max().item(), key


def test_full_ring_at_the_largest_n(torch_cuda):
    """The largest supported grid with a full detector ring: n = 1024, 1024 detectors (n_phi =
    1024, every ring position occupied: the two-stage K5T without its zero fill), n_t = 2048,
    batch 2 (the second image checks the batch stride): A and A* of image 0 against the oracle,
    the 1e-5 adjoint identity on both images."""
    import dataclasses
    geo = dataclasses.replace(synth.geometry("C5"), n_det=1024, batch=2, angles=synth.ring_angles(1024))
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = np.stack([synth.phantom("C5", b) for b in range(2)])
    g_gpu = _run(torch_cuda, plan, f=f)
    _check(g_gpu[0], O.forward(f[0].astype(np.float64), C), "n=1024 full ring A")
    u_gpu = _run(torch_cuda, plan, g=g_gpu)
    _check(u_gpu[0], O.adjoint(g_gpu[0].astype(np.float64), C), "n=1024 full ring A*")
    gr = np.stack([synth.random_data(geo.n_t, geo.n_det, 510 + b) for b in range(2)])
    _adjoint_identity(torch_cuda, plan, geo, C, f, gr)


@pytest.mark.parametrize("n,n_det,n_t,batch", [(128, 256, 216, 3), (256, 512, 432, 2), (256, 1024, 486, 1)])
def test_ring2_ragged_time_tiles(torch_cuda, n, n_det, n_t, batch):
    """The two-stage ring kernels (n_phi = n_det = 256 / 512 / 1024) with n_t not a multiple of
    their 2G time samples per CTA (ragged last K5 / K5T tile; n_t = 2^a 3^b as 2M = 6 n_t must be)
    and an odd batch: A and A* of every image against the oracle."""
    geo = synth.Geometry(n, n_det, n_t, T=2.0, batch=batch, angles=synth.ring_angles(n_det))
    from paper_2510_24687_b200 import derive
    info, _, st = derive(n, n_det, n_t, 1.0, 1.0, 2.0, batch, geo.angles_array())
    if st != 0:
        pytest.skip(f"geometry unsupported by the kernels (status {st})")
    C = O.derive_geom(geo)
    plan = _plan(geo)
    f = np.stack([synth.phantom("C2", b, n=n) for b in range(batch)])
    gg = _run(torch_cuda, plan, f=f)
    gr = np.stack([synth.random_data(n_t, n_det, 40 + b) for b in range(batch)])
    uu = _run(torch_cuda, plan, g=gr)
    for b in range(batch):
        _check(gg[b], O.forward(f[b].astype(np.float64), C), f"A image {b}")
        _check(uu[b], O.adjoint(gr[b].astype(np.float64), C), f"A* image {b}")
