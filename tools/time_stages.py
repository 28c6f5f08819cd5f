"""Per-stage device times (µs) of one configuration through the in-library events, and the
graph-replayed step time (L2 flushed between replays).  Tuning helper, not a bench line.
    python tools/time_stages.py [C3] [reps]      (TAT_LIB selects a variant build)"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2510_24687_b200 import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
geo = synth.geometry(name)
plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
f = torch.from_numpy(synth.phantom_batch(name)).cuda()
g = torch.empty((geo.batch, geo.n_t, geo.n_det), device="cuda")
u = torch.empty((geo.batch, geo.n, geo.n), device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(3):
    plan.forward(f, out=g)
    plan.adjoint(g, out=u)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    plan.forward(f, out=g)
    plan.adjoint(g, out=u)
ts = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
plan.profile_begin(2 * 5)
for _ in range(5):
    flush.zero_()
    plan.forward(f, out=g)
    plan.adjoint(g, out=u)
torch.cuda.synchronize()
ms, nf, na = plan.profile_end()
names = ["K1", "K2", "K3", "K4", "K5", "K5T", "K4T", "K3T", "K2Ta", "K2Tb", "K1T"]
st = {k: round(1000 * v / (nf if i < 5 else na), 1) for i, (k, v) in enumerate(zip(names, ms))}
print(f"{os.environ.get('TAT_LIB', 'default')} {name} step_us {1000 * statistics.median(ts):.1f} "
      + " ".join(f"{k}={v}" for k, v in st.items()), flush=True)
