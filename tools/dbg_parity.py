import sys, numpy as np, torch
sys.path.insert(0,'.')
import synth
from oracle import tat_oracle as O
from paper_2510_24687_b200 import Plan
for name in ['T32','C1','C2']:
    geo=synth.geometry(name); C=O.derive_geom(geo)
    plan=Plan(geo.n,geo.n_det,geo.n_t,1.,1.,2.,1,geo.angles_array())
    f=synth.phantom(name)[None]
    g=plan.forward(torch.from_numpy(f).cuda()).cpu().numpy()[0]
    ref=O.forward(f[0].astype(float),C)
    gg=synth.random_data(geo.n_t,geo.n_det,5)[None]
    u=plan.adjoint(torch.from_numpy(gg).cuda()).cpu().numpy()[0]
    uref=O.adjoint(gg[0].astype(float),C)
    print(name, 'fwd', np.linalg.norm(g-ref)/np.linalg.norm(ref), 'adj', np.linalg.norm(u-uref)/np.linalg.norm(uref))
