"""NNLS (projected Landweber) at C3, a few iterations: for an ncu launch list of its kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2510_24687_b200 import Plan
geo = synth.geometry("C3")
plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
f = torch.from_numpy(synth.phantom_batch("C3")).cuda()
g = plan.forward(f)
x = torch.zeros_like(f)
r = torch.empty_like(g)
plan.nnls(g, x, 0.1, 3, r_work=r)
torch.cuda.synchronize()
