"""Time A and A* at C3 sizes with irregular detector angles (dense mode) vs the ring geometry."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24687_b200 import Plan
import synth

def t(plan, f, g, reps=10):
    for _ in range(3):
        plan.forward(f, out=g); plan.adjoint(g, out=f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.forward(f, out=g); plan.adjoint(g, out=f)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n, nd, nt, B = 512, 512, 1024, 16
f = torch.from_numpy(synth.phantom_batch("C3")).cuda()
g = torch.empty((B, nt, nd), device="cuda")
ring = Plan(n, nd, nt, batch=B, angles=synth.ring_angles(nd))
ang = np.sort(np.random.default_rng(1).uniform(0, 2 * np.pi, nd))
dense = Plan(n, nd, nt, batch=B, angles=ang)
print("ring  ms/pair-batch", t(ring, f.clone(), g))
print("dense ms/pair-batch", t(dense, f.clone(), g), "n_ring", dense.info["n_ring"])
dense.profile_begin(4)
for _ in range(2):
    dense.forward(f, out=g); dense.adjoint(g, out=f)
torch.cuda.synchronize()
ms, nf, na = dense.profile_end()
print("dense stages us", [round(1000 * x / 2, 1) for x in ms])
