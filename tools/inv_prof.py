"""Inverse (Alg. 3) at C3, three calls: for an ncu launch list of its kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2510_24687_b200 import Plan
geo = synth.geometry("C3")
plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
g = torch.from_numpy(np.stack([synth.random_data(geo.n_t, geo.n_det, 700 + b) for b in range(geo.batch)])).cuda()
u = torch.empty(geo.batch, geo.n, geo.n, device="cuda")
for _ in range(3): plan.inverse(g, 0.95, out=u)
torch.cuda.synchronize()
