"""Interleaved A/B timing of plan variants (JIT environment knobs) in ONE
process: every variant's plan is built first (its env applied while the
kernels are generated), then forward+adjoint steps alternate A, B, A, B, ...
so clock / power drift hits all variants alike; medians of the device times.
Each plan's kernels keep the launch geometry they were generated with, so
knobs read at launch time (HQ_PINGPONG, HQ_DOT_GROUP) vary per plan too.

  python tools/ab_probe.py cfg4 1024 c64 "HQ_WARP_SYNC=0" "HQ_WARP_SYNC=1" [rounds]
"""
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl  # noqa: E402
from paper_2301_03251_b200 import templates as T  # noqa: E402


def main():
    cfg, B, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    variants = [v for v in sys.argv[4:] if "=" in v or v == "-"]
    rounds = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 5
    n, d, P, _, _ = wl.CONFIGS[cfg]
    b = wl.make_builder(cfg, qsim, T)
    x = wl.inputs_for(cfg, B)
    th = wl.params_for(cfg)
    tape, ok = tr.trace(b, x, th)
    grad = tr.classify(tape, d + P, [False] * d + [True] * P, math.pi / 2, 0.5)
    plans = []
    for v in variants:
        saved = dict(os.environ)
        for kv in v.split(","):
            if "=" in kv:
                k, val = kv.split("=", 1)
                os.environ[k] = val
        plans.append(engine.Plan(tape, d, P, prec, grad))
        os.environ.clear()
        os.environ.update(saved)
    xd = torch.tensor(x, device="cuda")
    td = torch.tensor(th, device="cuda")
    for p in plans:
        p.forward(xd, td, True)
    torch.cuda.synchronize()
    times = [[] for _ in plans]
    for _ in range(rounds):
        for i, p in enumerate(plans):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.forward(xd, td, True)
            e1.record()
            torch.cuda.synchronize()
            times[i].append(e0.elapsed_time(e1))
    for v, p, t in zip(variants, plans, times):
        print(f"{cfg} B={B} {prec} [{v}] median {statistics.median(t):.2f} ms  min {min(t):.2f}  "
              f"all {' '.join(f'{x:.1f}' for x in t)}  plan {p.description[-80:]}", flush=True)


if __name__ == "__main__":
    main()
