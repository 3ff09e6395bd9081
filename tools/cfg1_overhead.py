import sys, math, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl, templates as T
cfg = "cfg1"; n, d, P, B, _ = wl.CONFIGS[cfg]
b = wl.make_builder(cfg, qsim, T); x = wl.inputs_for(cfg, B); th = wl.params_for(cfg)
tape, ok = tr.trace(b, x, th)
grad = tr.classify(tape, d + P, [True] * (d + P), math.pi / 2, 0.5)
plan = engine.Plan(tape, d, P, "c128", grad)
xd = torch.tensor(x, device="cuda"); td = torch.tensor(th, device="cuda"); up = torch.ones(B, dtype=torch.float64, device="cuda")
def step():
    out, jac = plan.forward(xd, td, True)
    return plan.vjp(jac, up, True, True)
for _ in range(20): step()
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N): step()
torch.cuda.synchronize()
print("wall us/step", (time.perf_counter() - t0) / N * 1e6)
plan.profile(True)
for _ in range(N): step()
torch.cuda.synchronize()
print({k: round(v["ms"] / N * 1e3, 2) for k, v in plan.profile_read().items()}, "us per step (device)")
plan.profile(False)
# host-side cost only: time the python calls without sync
t0 = time.perf_counter()
for _ in range(N): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host enqueue us/step", (t1 - t0) / N * 1e6)
