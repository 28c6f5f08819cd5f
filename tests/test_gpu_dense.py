"""GPU dense mode (reading G24): detectors at irregular angles off any
canonical ring, K5/K5T as dense sums on the GPU, against the float64 oracle's dense mode."""
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


# K5 on tcgen05 (3xTF32 GEMM; 288 leaves a ragged 32-row time tile and a 3-tile multicast
# cluster falls back to 1 CTA, 81 an odd ragged one, 200 / 100 a ragged detector tile);
# TAT_DENSE_TC=0: the SIMT synthesis / analysis kernels, =2 SIMT analysis only
@pytest.mark.parametrize("n,n_det,n_t,batch,tc", [(64, 48, 128, 2, "1"), (256, 200, 512, 2, "1"),
                                                  (128, 100, 288, 3, "1"), (64, 48, 81, 2, "1"),
                                                  (64, 48, 128, 2, "0"), (256, 200, 512, 2, "2")])
def test_dense_parity_and_adjoint(torch_cuda, monkeypatch, n, n_det, n_t, batch, tc):
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    monkeypatch.setenv("TAT_DENSE_TC", tc)
    ang = np.sort(np.random.default_rng(n).uniform(0.0, 2 * np.pi, n_det))
    C = O.derive(n, n_det, n_t, 1.0, 1.0, 2.0, ang)
    assert C.dense
    plan = Plan(n, n_det, n_t, batch=batch, angles=ang)
    assert plan.info["n_ring"] == C.n_ring and (plan.info["ring"] == -1).all()
    f = np.stack([synth.phantom("C2", b, n=n) for b in range(batch)])
    g = plan.forward(torch.from_numpy(f).cuda())
    gd = np.stack([synth.random_data(n_t, n_det, 80 + b) for b in range(batch)])
    u = plan.adjoint(torch.from_numpy(gd).cuda())
    torch.cuda.synchronize()
    gh, uh = g.cpu().numpy(), u.cpu().numpy()
    for b in range(batch):
        _check(gh[b], O.forward(f[b].astype(np.float64), C), f"dense A {b}")
        _check(uh[b], O.adjoint(gd[b].astype(np.float64), C), f"dense A* {b}")
    wY, wX = C.dt * 2 * np.pi / C.n_ring, C.h * C.h
    Af = gh.astype(np.float64)
    lhs = wY * np.sum(Af * gd)
    rhs = wX * np.sum(f.astype(np.float64) * uh)
    assert abs(lhs - rhs) <= 1e-5 * np.sqrt(wY * np.sum(Af * Af)) * np.sqrt(wY * np.sum(gd.astype(np.float64) ** 2))


def test_dense_full_size_c3(torch_cuda):
    """C3 sizes (n = 512, 512 detectors at irregular angles, n_t = 1024, batch 16, the launch
    configuration the dense timing uses): images 0 and 15 against the oracle in full."""
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    n, n_det, n_t, batch = 512, 512, 1024, 16
    ang = np.sort(np.random.default_rng(1).uniform(0.0, 2 * np.pi, n_det))
    C = O.derive(n, n_det, n_t, 1.0, 1.0, 2.0, ang)
    plan = Plan(n, n_det, n_t, batch=batch, angles=ang)
    f = synth.phantom_batch("C3")
    gd = np.stack([synth.random_data(n_t, n_det, 500 + b) for b in range(batch)])
    g = plan.forward(torch.from_numpy(f).cuda()).cpu().numpy()
    u = plan.adjoint(torch.from_numpy(gd).cuda()).cpu().numpy()
    for b in (0, batch - 1):
        _check(g[b], O.forward(f[b].astype(np.float64), C), f"dense C3 A {b}")
        _check(u[b], O.adjoint(gd[b].astype(np.float64), C), f"dense C3 A* {b}")
