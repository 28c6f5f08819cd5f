#!/usr/bin/env python
"""Benchmark: A + A* pairs per second at n=512, batch 16 (BASELINE.json metric, config C3).

One step = one forward A and one adjoint A* over the whole batch (all SURVEY §8(a) rows),
through libtat's C ABI (ctypes binding), inputs resident in HBM.  L2 (126 MB) is flushed
between timed steps (outside the per-step CUDA events); the step's own working set (~300 MB
at C3) exceeds L2 as well.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

--impl reference times the float64 oracle (tests' reference; a deliberately slow CPU program)
on bounded samples of the same workload.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "A+A* pairs/sec at n=512, batch 16 (fp32); achieved % of HBM roofline"
UNIT = "image-pairs/s"
STAGES = ["K1", "K2", "K3", "K4", "K5", "K5T", "K4T", "K3T", "K2Ta", "K2Tb", "K1T"]


def workload_desc(name: str) -> str:
    g = synth.geometry(name)
    kind = {"C1": "8 Gaussians", "C2": "20 ellipses", "C3": "20 random ellipses",
            "C4": "8 Gaussians + 20 ellipses", "C5": "20 ellipses, 270-degree arc"}[name]
    return (f"{name}: n={g.n}, {g.n_det} detectors (R=1, c=1), n_t={g.n_t} on (0,{g.T:g}], "
            f"batch {g.batch}, {kind}")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- models
def model(info: dict) -> dict:
    """SURVEY §8(d) "Algorithmic bytes" and flops per launch (whole batch), DESIGN.md §7.
    Bytes: every transposed intermediate (S1..S4) written once and read once at its minimal
    size (complex64, Hermitian-reduced), inputs / outputs once, plan tables once per call:
      per image per A (= per A*): 4n^2 + 4 n_t n_det + 16 [n (N/2+1) + 2 N_lam (K+1) + n_t (K+1)],
      per call: 16 N_lam (K+1) + 4 n_det.
    Split over the stages as the survey does (K1 = f + S1, K2 = S1 + S2 + tables, K3 = S2 + S3,
    K4 = S3 + S4, K5 = S4 + g + ring map; the adjoint stages mirror them).
    Flops: 5 m log2 m per m-point complex FFT (K2: N-point per column, SURVEY §8(d)'s 8.1 GFLOP
    at C3), the same convention for every stage."""
    n, N, B = info["n"], info["N"], info["batch"]
    ncols = N // 2 + 1
    NL = info["J"] + 1
    Kp = info["K"] + 1
    nphi = info["n_ring"]
    n_t, n_det = info["n_t"], info["n_det"]
    M2 = 2 * info["M"]
    f_b, g_b = 4 * n * n, 4 * n_t * n_det
    S1, S2, S3, S4 = 8 * n * ncols, 8 * NL * Kp, 8 * NL * Kp, 8 * n_t * Kp
    tables = 16 * NL * Kp
    lg = math.log2
    fft = lambda m: 5 * m * lg(m)
    fwd = {"K1": B * (f_b + S1), "K2": B * (S1 + S2) + tables, "K3": B * (S2 + S3),
           "K4": B * (S3 + S4), "K5": B * (S4 + g_b) + 4 * n_det}
    adj = {"K5T": fwd["K5"], "K4T": fwd["K4"], "K3T": fwd["K3"], "K2T": fwd["K2"], "K1T": fwd["K1"]}
    by = {**fwd, **adj}
    fl = {"K1": B * n * fft(N) / 2,            # n/2 complex row-pair transforms of length N
          "K2": B * ncols * fft(N),
          "K3": B * NL * fft(nphi),
          "K4": B * Kp * fft(M2),
          "K5": B * n_t * fft(nphi) / 2}         # two real time samples per complex transform
    fl.update({"K5T": fl["K5"], "K4T": fl["K4"], "K3T": fl["K3"], "K2T": fl["K2"], "K1T": fl["K1"]})
    # the two kernels of the A*-4 stage: K2Ta (target sums: reads S2, writes the targets Rc,
    # 8 bytes per Cartesian target, + 12-byte records) and K2Tb (reads Rc, writes S1; K2's flops)
    Rc = 8 * info.get("n_targets", 0)
    by.update({"K2Ta": B * (S2 + Rc) + 12 * info.get("n_targets", 0), "K2Tb": B * (Rc + S1)})
    fl.update({"K2Ta": B * info.get("n_targets", 0) * 6, "K2Tb": fl["K2"]})
    per_op = B * (f_b + g_b + 16 * (n * ncols + 2 * NL * Kp + n_t * Kp)) + tables + 4 * n_det
    return {"bytes": by, "flops": fl, "pair_bytes": 2 * per_op, "op_bytes": per_op}


BOUND = {"K1": "hbm", "K2": "alu", "K3": "hbm", "K4": "alu", "K5": "hbm",
         "K5T": "hbm", "K4T": "alu", "K3T": "hbm", "K2T": "alu", "K1T": "hbm",
         "K2Ta": "hbm", "K2Tb": "alu"}


def measured_traffic(name: str, stage: str):
    """DRAM bytes per launch of `stage` from the committed ncu --set full capture
    (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t[name][stage]
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle arm
def oracle_sample(name: str, budget_s: float, min_pairs: int = 1, max_pairs: int = 64):
    """Time the float64 oracle (as it stands) on images of the workload until budget_s."""
    from oracle import tat_oracle as O
    geo = synth.geometry(name)
    C = O.derive_geom(geo)
    t0 = time.perf_counter()
    O.forward(np.zeros((geo.n, geo.n)), C)          # untimed warm-up (table caches)
    setup = time.perf_counter() - t0
    done, t_work = 0, 0.0
    while done < max_pairs and (done < min_pairs or t_work < budget_s):
        f = synth.phantom(name, done % geo.batch).astype(np.float64)
        t1 = time.perf_counter()
        g = O.forward(f, C)
        O.adjoint(g, C)
        t_work += time.perf_counter() - t1
        done += 1
    return done, t_work, setup


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        th = [d.get("num_threads", 0) for d in threadpool_info() if d.get("user_api") == "blas"]
        return max(th) if th else os.cpu_count()
    except Exception:
        return os.cpu_count()


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    name = args.config
    budget = float(os.environ.get("TAT_ORACLE_STEP_S", "2.0"))
    oracle_sample(name, 0.0, min_pairs=1, max_pairs=1) if args.warmup > 0 else None
    times, pairs = [], 0
    for _ in range(args.steps):
        done, t, _ = oracle_sample(name, budget, min_pairs=1, max_pairs=4)
        times.append(t)
        pairs += done
    total = sum(times)
    value = pairs / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_desc(name), "parallelism": "cpu (float64 oracle)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
                         "sample": f"{pairs} image pairs (A then A*) of {name}, float64 direct sums"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- multi-GPU host logic
def rank_images(name: str, rank: int) -> np.ndarray:
    """The batch of rank `rank` (replicas): images rank*B .. rank*B + B - 1 of
    the workload's seeded phantom family, so every rank processes distinct images."""
    B = synth.geometry(name).batch
    return np.stack([synth.phantom(name, rank * B + b) for b in range(B)]).astype(np.float32)


def reduce_timing(total_ms: float, units: float, world: int, device=None):
    """(max over ranks of the timed region in ms, sum over ranks of the units processed)."""
    if world <= 1:
        return total_ms, units
    import torch
    import torch.distributed as dist
    t = torch.tensor([total_ms], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


# ----------------------------------------------------------------------------- GPU arm
def landweber(plan, f, f_host, geo, name, dev, stream, iters: int = 50, reps: int = 3):
    """BASELINE configs[2] workload: projected-Landweber / NNLS (§4.2) on
    g = A f + Gaussian noise at 2% of max|g| per image, f0 = 0, step 1/lambda_max(A*A) from
    20 power iterations; `iters` iterations = 2*iters operator applications, captured once
    as a CUDA graph (fused residual / update epilogues) and replayed."""
    import torch
    B = geo.batch
    g = plan.forward(f)
    torch.cuda.synchronize()
    gh = g.cpu().numpy()
    for b in range(B):
        gh[b] += 0.02 * np.abs(gh[b]).max() * synth.random_data(geo.n_t, geo.n_det, 3100 + b)
    g_obs = torch.from_numpy(gh).to(dev)
    lam_max = plan.power_norm(20, seed=3000)
    lam = 1.0 / lam_max
    fl = torch.zeros_like(f)
    r = torch.empty_like(g_obs)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        plan.nnls(g_obs, fl, lam, iters, r_work=r, stream=s)
    fl.zero_()
    graph.replay()                       # warm-up
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res = plan.residual(fl, g_obs)
    torch.cuda.synchronize()
    rel_res = float(torch.linalg.vector_norm(res) / torch.linalg.vector_norm(g_obs))
    return {"workload": f"{name}: NNLS (projected Landweber) {iters} iterations = {2 * iters} "
                        f"applications, batch {B}, noise 2% of max|g|, f0 = 0, CUDA graph",
            "lambda_max": lam_max, "step": lam, "ms_per_loop": ms,
            "image_pairs_per_s": B * iters / (ms / 1000.0), "final_rel_residual": rel_res}


def step_graph(plan, f, g, u):
    """A CUDA graph of one step (A then A* over the batch) on the current stream."""
    import torch
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        plan.forward(f, out=g)
        plan.adjoint(g, out=u)
    return graph


def time_replays(graph, flush, stream, reps: int) -> list:
    """Per-replay device times (ms) with CUDA events, L2 flushed before each (outside)."""
    import torch
    st = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for i in range(reps):
        flush.zero_()
        st[i].record(stream)
        graph.replay()
        en[i].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in zip(st, en)]


def other_configs(names, flush, stream, pk) -> dict:
    """SURVEY §8(d) per-config numbers: µs per batch A + A* pair (graph replay, median of 20),
    image-pairs/s and the effective HBM fraction by the §8(d) model bytes."""
    import torch
    from paper_2510_24687_b200 import Plan
    out = {}
    for name in names:
        geo = synth.geometry(name)
        plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, geo.batch, geo.angles_array())
        f = torch.from_numpy(synth.phantom_batch(name)).cuda()
        g = torch.empty((geo.batch, geo.n_t, geo.n_det), device="cuda")
        u = torch.empty((geo.batch, geo.n, geo.n), device="cuda")
        for _ in range(3):
            plan.forward(f, out=g)
            plan.adjoint(g, out=u)
        graph = step_graph(plan, f, g, u)
        graph.replay()
        torch.cuda.synchronize()
        ms = statistics.median(time_replays(graph, flush, stream, 20))
        mdl = model(plan.info)
        out[name] = {"us_per_pair": round(1000 * ms, 2),
                     "image_pairs_per_s": round(geo.batch / (ms / 1000.0), 1),
                     "hbm_frac": round(mdl["pair_bytes"] / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], 4),
                     "batch": geo.batch}
        del graph, plan
    return out


def lpd_step_bench(name: str, steps: int, warmup: int, flush, stream, K: int = 5) -> dict:
    """LPD-shaped training step (§4.2; §8(f) f3): K
    unrolled primal-dual iterations q <- Gamma(q, A f, y), f <- Lambda(f, A* q) (eq:LPD_dual,
    eq:LPD_primal) with the CNNs replaced by elementwise maps with learnable scalars (no
    networks), f0 = q0 = 0, loss ||f_K - f_true||^2, torch.autograd backward through
    Plan.A / Plan.Astar (backward of A = A^T, of A* = omega A: libtat kernels), then an SGD
    update.  y = A f_true + 5 % noise.  Eager (autograd), CUDA events per step."""
    import torch
    from paper_2510_24687_b200 import Plan
    geo = synth.geometry(name)
    B = geo.batch
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, B, geo.angles_array())
    f_true = torch.from_numpy(synth.phantom_batch(name)).cuda()
    y = plan.forward(f_true)
    noise = torch.from_numpy(np.stack([synth.random_data(geo.n_t, geo.n_det, 4100 + b)
                                       for b in range(B)])).cuda()
    y = y + 0.05 * y.abs().amax(dim=(1, 2), keepdim=True) * noise
    lam = 1.0 / plan.power_norm(10, seed=4000)
    a = torch.tensor([1.0, 0.0], device="cuda", requires_grad=True)          # Gamma
    b = torch.tensor([lam, 0.0], device="cuda", requires_grad=True)          # Lambda
    opt = torch.optim.SGD([a, b], lr=1e-6)
    calls = {"forward": 0, "adjoint": 0, "transpose": 0, "forward_scaled": 0}
    for nm in calls:
        fn = getattr(plan, nm)

        def wrap(*args, _fn=fn, _nm=nm, **kw):
            calls[_nm] += 1
            return _fn(*args, **kw)
        setattr(plan, nm, wrap)

    def train_step():
        f = torch.zeros_like(f_true)
        q = torch.zeros_like(y)
        for _ in range(K):
            q = q + a[0] * (plan.A(f) - y) + a[1] * q                       # Gamma stand-in
            f = torch.relu(f - b[0] * plan.Astar(q) + b[1] * f)              # Lambda stand-in
        loss = ((f - f_true) ** 2).mean()
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        return loss

    for _ in range(warmup):
        train_step()
    torch.cuda.synchronize()
    for k in calls:
        calls[k] = 0
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        st[i].record(stream)
        loss = train_step()
        en[i].record(stream)
    torch.cuda.synchronize()
    ms = statistics.median([x.elapsed_time(z) for x, z in zip(st, en)])
    per = {k: v // steps for k, v in calls.items()}
    n_a = per["forward"] + per["forward_scaled"]
    n_as = per["adjoint"] + per["transpose"]
    return {"workload": f"{name}: LPD-shaped training step, K = {K} unrolled iterations, batch {B}, "
                        "5% noise, elementwise CNN stand-ins, autograd through Plan.A / Plan.Astar, SGD",
            "ms_per_step": ms, "steps_per_s": 1000.0 / ms,
            "operator_evals_per_step": {"A (forward + omega A in backward)": n_a,
                                        "A* (adjoint + A^T in backward)": n_as},
            "image_operator_pairs_per_s": B * 0.5 * (n_a + n_as) / (ms / 1000.0),
            "final_loss": float(loss.item())}


def run_gpu(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    from paper_2510_24687_b200 import Plan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    name = args.config
    geo = synth.geometry(name)
    B = geo.batch
    plan = Plan(geo.n, geo.n_det, geo.n_t, geo.R, geo.c, geo.T, B, geo.angles_array())
    info = plan.info
    f_host = rank_images(name, rank)                        # distinct images per rank
    f = torch.from_numpy(f_host).to(dev)
    g = torch.empty((B, geo.n_t, geo.n_det), device=dev)
    u = torch.empty((B, geo.n, geo.n), device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step():
        plan.forward(f, out=g)
        plan.adjoint(g, out=u)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # the timed steps replay one CUDA graph of the step's launches (enqueue-only API, PDL edges
    # kept), so small configurations are not bound by host launch overhead
    graph = None
    if not args.no_graph:
        graph = step_graph(plan, f, g, u)
        graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        if graph is not None:
            graph.replay()
        else:
            step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    # per-stage device times from in-library events, in a separate (untimed) pass
    prof_steps = min(args.steps, 5)
    plan.profile_begin(2 * prof_steps)
    for _ in range(prof_steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    stage_ms, nf, na = plan.profile_end()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms, units = reduce_timing(sum(step_ms), B * args.steps, world, dev)
    ms_per_step = total_ms / args.steps
    value = units / (total_ms / 1000.0)

    # ---- end to end through the C ABI with HOST buffers: every step tat_pair_host copies its
    # batch from pinned host memory (H2D), runs A and A*, copies A* g back (D2H); the plan
    # pipelines the copies of neighbouring steps on its own streams (include/tat.h)
    f_pin = torch.from_numpy(f_host).pin_memory()
    u_pin = [torch.empty((B, geo.n, geo.n), dtype=torch.float32).pin_memory() for _ in range(2)]
    fp_np, up_np = f_pin.numpy(), [t.numpy() for t in u_pin]
    for i in range(4):
        plan.pair_host(fp_np, up_np[i & 1], stream=stream)
    plan.join_host(stream)
    torch.cuda.synchronize()
    e2e_steps = max(3, args.steps)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_steps):
        plan.pair_host(fp_np, up_np[i & 1], stream=stream)
    plan.join_host(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms, e2e_units = reduce_timing(e0.elapsed_time(e1), B * e2e_steps, world, dev)
    e2e_value = e2e_units / (e2e_ms / 1000.0)

    lw = landweber(plan, f, f_host, geo, name, dev, stream) if not args.no_loop else None
    inv = None
    if not args.no_loop:   # A^{-1} (Algorithm 3) over the batch, tables built before timing
        try:
            plan.inverse(g, 0.95, out=u)
            torch.cuda.synchronize()
            i0 = torch.cuda.Event(enable_timing=True)
            i1 = torch.cuda.Event(enable_timing=True)
            i0.record(stream)
            for _ in range(3):
                plan.inverse(g, 0.95, out=u)
            i1.record(stream)
            torch.cuda.synchronize()
            inv_ms = i0.elapsed_time(i1) / 3
            inv = {"ms_per_call": inv_ms, "images_per_s": B / (inv_ms / 1000.0), "r0": 0.95}
        except Exception as exc:   # geometry outside the inverse's support
            inv = {"unavailable": str(exc)}

    pk, pk_kind = peaks()
    extras = lpd = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = other_configs([c for c in ("C1", "C2", "C4", "C5") if c != name], flush, stream, pk)
        lpd = lpd_step_bench("C4", 5, 3, flush, stream)

    if rank != 0:
        return 0

    mdl = model(info)
    raw = {s: 1000.0 * stage_ms[i] / max(1, (nf if i < 5 else na)) for i, s in enumerate(STAGES)}
    per_stage_us = {k: v for k, v in raw.items() if k not in ("K2Ta", "K2Tb")}
    per_stage_us["K2T"] = raw["K2Ta"] + raw["K2Tb"]     # the adjoint column stage (A*-4)
    # the roofline names the dominant single KERNEL (the A*-4 stage is two launches: the
    # transposed-bilinear target sums K2Ta, HBM/latency, and the inverse column DFT K2Tb, whose
    # flops are K2's); per-stage floors below use the §8(d) stages
    per_kernel_us = {k: v for k, v in raw.items() if v > 0}
    dom = max(per_kernel_us, key=per_kernel_us.get)
    dur_s = per_kernel_us[dom] * 1e-6
    # FP32 FFMA peak MEASURED on this pool's B200 (tools/ubench_fp32.cu, profiles/
    # r2_ubench_fp32.txt: 3.553e13 lane-ops/s = 71.1 TFLOP/s at 1965 MHz; 95 % of the 74.4
    # TFLOP/s that 148 SM x 128 lanes x 2 x 1965 MHz gives), scaled to the run's max clock
    alu_peak = 2 * 3.553e13 / 1e12 * pk.get("sm_max_mhz", 1965.0) / 1965.0    # TFLOP/s
    if BOUND[dom] == "alu":
        ach = mdl["flops"][dom] / dur_s / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": ach / alu_peak, "traffic": measured_traffic(name, dom),
                "kernel": dom, "algorithmic_flops": mdl["flops"][dom],
                "flops_model": "SURVEY §8(d): 5 N log2 N per N-point column transform",
                "hbm_achieved_gbs": mdl["bytes"][dom] / dur_s / 1e9,
                "peak_source": "measured FFMA rate (tools/ubench_fp32.cu, profiles/r2_ubench_fp32.txt)"}
    else:
        ach = mdl["bytes"][dom] / dur_s / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach / pk["hbm_gbs"], "traffic": measured_traffic(name, dom), "kernel": dom,
                "algorithmic_bytes": mdl["bytes"][dom], "peak_source": pk_kind}
    # attained fraction of each stage's max(HBM, FP32) floor from the model
    # bytes / flops at the measured HBM peak and the derived ALU peak
    floors = {}
    for st, us in per_stage_us.items():
        f_us = max(mdl["bytes"][st] / (pk["hbm_gbs"] * 1e9), mdl["flops"][st] / (alu_peak * 1e12)) * 1e6
        floors[st] = {"floor_us": round(f_us, 2), "frac": round(f_us / us, 3) if us > 0 else None}
    floor_tot = sum(v["floor_us"] for v in floors.values())
    stage_floor = {"per_stage": floors, "sum_floor_us": round(floor_tot, 1),
                   "frac": round(floor_tot / sum(per_stage_us.values()), 3),
                   "model": "max(§8(d) model bytes / measured HBM peak, model flops / measured FP32 peak)"}
    eff_hbm = mdl["pair_bytes"] / (ms_per_step * 1e-3) / 1e9     # GB/s, whole batch
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline_leg(name, plan, f, g, u, geo)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(name), "batch_per_gpu": B,
                   "parallelism": f"replicas x{world} (batch-sharded, no collective)",
                   "l2": "flushed (256 MB write) between timed steps, outside the step events",
                   "launch": "CUDA graph replay per step" if graph is not None else "eager"},
        "hbm_roofline_effective": {"model_bytes_per_step": mdl["pair_bytes"],
                                   "model": "SURVEY §8(d) algorithmic bytes (2 x per-operator)",
                                   "achieved_gbs": eff_hbm, "peak_gbs": pk["hbm_gbs"],
                                   "frac": eff_hbm / pk["hbm_gbs"]},
        "roofline": roof,
        "stage_us": {k: round(v, 2) for k, v in per_stage_us.items()},
        "kernel_us": {k: round(v, 2) for k, v in per_kernel_us.items()},
        "stage_floor": stage_floor,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(f_host.nbytes),
                "d2h_bytes_per_step": int(u_pin[0].numel() * 4),
                "path": "tat_pair_host (C ABI, pinned host buffers, copies pipelined on the "
                        "plan's streams), device-timed over the whole run"},
        "gpu_launches": (info["launches_forward"] + info["launches_adjoint"]) * args.steps,
        "clocks": clocks,
        "landweber": lw,
        "inverse": inv,
        "other_configs": extras,
        "lpd_step": lpd,
        "paper_context": "A alone: 0.0055 s at 257^2, 360x513, batch 1 on an Nvidia A2000 "
                         "(PAPER.md L822-825); not this workload",
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(name, plan, f, g, u, geo) -> dict:
    """The float64 oracle as it stands, timed on the host cores on a bounded sample of the
    workload (SURVEY §8(d) "Oracle timing"); the sampled images' oracle outputs are also
    compared with the GPU's outputs for the same images (rel-L2, the parity bar 1e-4)."""
    from oracle import tat_oracle as O
    import torch
    budget = float(os.environ.get("TAT_ORACLE_BUDGET_S", "10"))
    C = O.derive_geom(geo)
    t0 = time.perf_counter()
    O.forward(np.zeros((geo.n, geo.n)), C)          # untimed warm-up (table caches)
    setup = time.perf_counter() - t0
    plan.forward(f, out=g)
    plan.adjoint(g, out=u)
    torch.cuda.synchronize()
    fh, gh, uh = f.cpu().numpy(), g.cpu().numpy(), u.cpu().numpy()
    done, t_work, worst_a, worst_as = 0, 0.0, 0.0, 0.0
    while done < 64 and (done < 1 or t_work < budget):
        b = done % geo.batch
        t1 = time.perf_counter()
        ga = O.forward(fh[b].astype(np.float64), C)
        ua = O.adjoint(gh[b].astype(np.float64), C)
        t_work += time.perf_counter() - t1
        worst_a = max(worst_a, float(np.linalg.norm(gh[b] - ga) / np.linalg.norm(ga)))
        worst_as = max(worst_as, float(np.linalg.norm(uh[b] - ua) / np.linalg.norm(ua)))
        done += 1
    return {"value": done / t_work, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
            "sample": f"{done} image pair(s) (A then A*) of {name} in float64 direct sums; "
                      f"table setup {setup:.1f}s excluded",
            "parity_on_sample": {"A_rel_l2_max": worst_a, "Astar_rel_l2_max": worst_as,
                                 "bar": 1e-4}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=list(synth.CONFIGS))
    ap.add_argument("--impl", default="tat", choices=["tat", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-loop", action="store_true", help="skip the NNLS loop measurement")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a graph")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the other-config and LPD-step measurements")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        return run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
