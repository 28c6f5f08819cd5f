"""Time A + A* at C3 with the f4 variants (G25 low-k quadrature, G26 de-apodised bilinear) and
the inverse, on the step's CUDA graph like bench.py (device time, L2 not flushed)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24687_b200 import Plan
import synth

geo = synth.geometry("C3")
f = torch.from_numpy(synth.phantom_batch("C3")).cuda()
g = torch.empty((geo.batch, geo.n_t, geo.n_det), device="cuda")
u = torch.empty_like(f)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gr.replay()
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for quad, interp in [("trapezoid", "bilinear"), ("lowk", "bilinear"), ("trapezoid", "deapod"), ("lowk", "deapod")]:
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
    plan.set_quadrature(quad)
    plan.set_interpolation(interp)
    ms = timed(lambda: (plan.forward(f, out=g), plan.adjoint(g, out=u)))
    print(f"{quad:9s} {interp:8s}  A+A* {ms * 1000:7.1f} us per 16-image pair")
plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
plan.forward(f, out=g)
plan.inverse(g, r0=0.95, out=u)
ms = timed(lambda: plan.inverse(g, r0=0.95, out=u))
print(f"inverse (Alg. 3)     {ms * 1000:7.1f} us per 16 images")
