"""cfg4 with the opt-in light-cone pruning (HQ_LIGHTCONE=1): the readout of
qubit 0 depends on 10 qubits and 164 of the 610 gates.  Device-timed forward +
gradient, same inputs as bench.py (B=4096, complex64)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl, templates as T

cfg = "cfg4"; n, d, P, B, prec = wl.CONFIGS[cfg]
b = wl.make_builder(cfg, qsim, T)
x = wl.inputs_for(cfg, B); th = wl.params_for(cfg)
tape, ok = tr.trace(b, x, th)
lc = tr.light_cone(tape)
grad = tr.classify(lc, d + P, [False] * d + [True] * P, math.pi / 2, 0.5)
plan = engine.Plan(lc, d, P, prec, grad)
xd = torch.tensor(x, device="cuda"); td = torch.tensor(th, device="cuda")
up = torch.ones(B, dtype=torch.float64, device="cuda")
def step():
    out, jac = plan.forward(xd, td, True)
    return plan.vjp(jac, up, False, True)
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"workload": "cfg4 + light cone (opt-in)", "reduced": f"{lc.n_qubits} qubits, {len(lc.ops)} gates",
                  "batch": B, "ms_per_step": ms, "samples_per_s": B / (ms / 1e3), "plan": plan.description}))
