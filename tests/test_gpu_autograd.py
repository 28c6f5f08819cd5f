"""Reverse-mode autodiff through A and A* on the GPU, against the float64
oracle: backward(A) = A^T = A*/omega and backward(A*) = omega A (reading G20), the LPD-shaped
use of PAPER.md §4.3 (L870-891) in miniature (a loss through A* A)."""
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


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_backward_of_A_and_Astar(torch_cuda, name):
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    geo = synth.geometry(name)
    C = O.derive_geom(geo)
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, 1, geo.angles_array())
    f0 = synth.random_image(geo.n, 21)[None]
    w = synth.random_data(geo.n_t, geo.n_det, 22)[None]
    f = torch.from_numpy(f0).cuda().requires_grad_(True)
    loss = (plan.A(f) * torch.from_numpy(w).cuda()).sum()          # <A f, w>
    loss.backward()
    ref = O.adjoint(w[0].astype(np.float64), C) / C.omega            # A^T w
    assert _rel(f.grad.cpu().numpy()[0], ref) <= 1e-4

    g = torch.from_numpy(w).cuda().requires_grad_(True)
    v = synth.random_image(geo.n, 23)[None]
    loss2 = (plan.Astar(g) * torch.from_numpy(v).cuda()).sum()      # <A* g, v>
    loss2.backward()
    ref2 = C.omega * O.forward(v[0].astype(np.float64), C)          # omega A v
    assert _rel(g.grad.cpu().numpy()[0], ref2) <= 1e-4


def test_gradient_of_data_fidelity(torch_cuda):
    """d/df 1/2 ||A f - g||^2 (Euclidean) = A^T (A f - g) through two autograd nodes, and the
    Euclidean transpose identity <A f, w> = <f, A^T w> in float64 on the host."""
    torch = torch_cuda
    from paper_2510_24687_b200 import Plan
    geo = synth.geometry("C1")
    C = O.derive_geom(geo)
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, 1, geo.angles_array())
    f0 = synth.phantom("C1", 3)[None]
    gobs = synth.random_data(geo.n_t, geo.n_det, 24)[None]
    f = torch.from_numpy(f0).cuda().requires_grad_(True)
    loss = 0.5 * ((plan.A(f) - torch.from_numpy(gobs).cuda()) ** 2).sum()
    loss.backward()
    r = O.forward(f0[0].astype(np.float64), C) - gobs[0]
    ref = O.adjoint(r, C) / C.omega
    assert _rel(f.grad.cpu().numpy()[0], ref) <= 1e-4
    w = torch.from_numpy(gobs).cuda()
    Af = plan.forward(torch.from_numpy(f0).cuda()).cpu().numpy().astype(np.float64)
    ATw = plan.transpose(w).cpu().numpy().astype(np.float64)
    lhs, rhs = np.sum(Af * gobs), np.sum(f0.astype(np.float64) * ATw)
    assert abs(lhs - rhs) <= 1e-5 * np.linalg.norm(Af) * np.linalg.norm(gobs)
