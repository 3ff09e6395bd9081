"""Per-launch timing of one plan (HQ_PROFILE_DUMP=1 prints every launch)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl
from paper_2301_03251_b200 import templates as T
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
prec = sys.argv[3] if len(sys.argv) > 3 else "c64"
n, d, P, _, _ = wl.CONFIGS[cfg]
b = wl.make_builder(cfg, qsim, T)
x = wl.inputs_for(cfg, B); th = wl.params_for(cfg)
tape, ok = tr.trace(b, x, th)
grad = tr.classify(tape, d + P, [False] * d + [True] * P, math.pi / 2, 0.5)
plan = engine.Plan(tape, d, P, prec, grad)
print(plan.description)
xd = torch.tensor(x, device="cuda"); td = torch.tensor(th, device="cuda")
for _ in range(2):
    plan.forward(xd, td, True)
torch.cuda.synchronize()
plan.profile(True)
plan.forward(xd, td, True)
print(plan.profile_read())
