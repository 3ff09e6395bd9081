"""cfg5 (32 qubits, depth 20, complex128 — a 64 GiB state) on ONE B200.

ψ and λ (128 GiB together) fit in one B200's HBM, so the full forward AND the
400... 1280-parameter adjoint run without sharding.  Prints one JSON line.
"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl
from paper_2301_03251_b200 import templates as T

grad = "--grad" in sys.argv
cfg = "cfg5"
n, d, P, _, _ = wl.CONFIGS[cfg]
b = wl.make_builder(cfg, qsim, T)
x = np.zeros((1, 0)); th = wl.params_for(cfg)
tape, ok = tr.trace(b, x, th)
spec = tr.classify(tape, P, [True] * P, math.pi / 2, 0.5) if grad else None
t0 = time.time()
plan = engine.Plan(tape, 0, P, "c128", spec)
t_plan = time.time() - t0
xd = torch.zeros((1, 1), dtype=torch.float64, device="cuda"); td = torch.tensor(th, device="cuda")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
plan.profile(True)
ev0.record()
out, jac = plan.forward(xd, td, grad)
ev1.record(); torch.cuda.synchronize()
prof = plan.profile_read()
ms = ev0.elapsed_time(ev1)
st = plan.stats(1, grad)
amp = 16 * 2 ** n
alg = amp * st["n_passes"] * (2 + (4 if grad else 0))
line = {"workload": "cfg5: 32-qubit HEA depth 20 (1900 gates), complex128, 1 GPU (no sharding)",
        "grad": grad, "E": float(out.item()), "ms": ms, "plan_s": t_plan, "passes": st["n_passes"],
        "algorithmic_GB": alg / 1e9, "achieved_GBps": alg / (ms / 1e3) / 1e9,
        "kernels_ms": {k: v["ms"] for k, v in prof.items()},
        "grad_norm": float(jac.norm().item()) if grad else None, "plan": plan.description}
print(json.dumps(line))
