"""Throughput of every SURVEY.md §8(d) config on one GPU (forward + gradient).

Device-timed with CUDA events (inputs resident), warm-up excluded.  Prints one
JSON line per config; used to fill profiles/ and DESIGN.md.
"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl
from paper_2301_03251_b200 import templates as T

def run(cfg, prec, batch=None, steps=5, warmup=2):
    n, d, P, B0, _ = wl.CONFIGS[cfg]
    B = batch or B0
    b = wl.make_builder(cfg, qsim, T)
    x = wl.inputs_for(cfg, B); th = wl.params_for(cfg)
    want_x = cfg in ("cfg1", "cfg2")
    tape, ok = tr.trace(b, x, th)
    grad = tr.classify(tape, d + P, [want_x] * d + [True] * P, math.pi / 2, 0.5)
    plan = engine.Plan(tape, d, P, prec, grad)
    xd = torch.tensor(x if d else np.zeros((B, 1)), device="cuda"); td = torch.tensor(th, device="cuda")
    up = torch.ones(B, dtype=torch.float64, device="cuda")
    def step():
        out, jac = plan.forward(xd, td, True)
        plan.vjp(jac, up, want_x, True)
    for _ in range(warmup): step()
    torch.cuda.synchronize()
    # latency-bound configs (host launch path in every step): many steps, median of 5 repeats
    small = n <= 12
    reps = 5 if small else 1
    steps = 100 if small else steps
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps): step()
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / steps)
    ms = sorted(times)[len(times) // 2]
    return {"config": cfg, "precision": prec, "batch": B, "ms_per_step": ms, "samples_per_s": B / (ms / 1e3),
            "steps": steps, "repeats": reps, "plan": plan.description.split(" [")[0]}

if __name__ == "__main__":
    jobs = [("cfg1", "c128", None), ("cfg1", "c64", None), ("cfg2", "c64", None), ("cfg2", "c128", None),
            ("cfg3", "c128", None), ("cfg3", "c64", None), ("cfg4", "c64", 1024), ("cfg4", "c128", 512)]
    for cfg, prec, B in jobs:
        print(json.dumps(run(cfg, prec, B)), flush=True)
