"""Precompile (NVRTC, sm_100a) the specialised pass kernels of known plans on
the build host, so GPU runs find their cubins in paper_2301_03251_b200/_jit_cache.

No GPU needed: plan creation compiles first and only then fails at device upload.
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HQ_JIT_COMPILE_ONLY", "1")

from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl  # noqa: E402
from paper_2301_03251_b200 import templates as T  # noqa: E402


class _FakeCuda:
    @staticmethod
    def current_device():
        return 0


class _FakeTorch:
    cuda = _FakeCuda


def plan_for(cfg, prec, want_x=False, want_p=True):
    n, d, P, _, _ = wl.CONFIGS[cfg]
    b = wl.make_builder(cfg, qsim, T)
    tape, ok = tr.trace(b, wl.inputs_for(cfg, 2), wl.params_for(cfg))
    grad = tr.classify(tape, d + P, [want_x] * d + [want_p] * P, math.pi / 2, 0.5)
    try:
        engine.Plan(tape, d, P, prec, grad)
    except Exception:
        pass  # expected without a GPU: the cubins are already on disk


def cfg5_segments(prec="c128"):
    """Segment plans of the amplitude-sharded cfg5 schedule (n=32, g=3): every
    distinct per-rank resolved segment (shard.py)."""
    from paper_2301_03251_b200 import shard as S
    n, depth = 32, 20

    def b(inputs, params):
        c = qsim.Circuit(n)
        k = 0
        for _ in range(depth):
            for q in range(n):
                c.ry(q, params[k]); c.rz(q, params[k + 1]); k += 2
            for q in range(n - 1):
                c.cnot(q, q + 1)
        c.measure(0)
        return c
    P = 2 * n * depth
    theta = wl.params_for("cfg5")
    tape, ok = tr.trace(b, wl.inputs_for("cfg5", 1), theta)
    sc = S.ShardedCircuit(tape, 0, P, 3, prec)
    seen = set()
    for i in range(len(sc.sched.segments)):
        for r in range(sc.world):
            t, grad = sc.segment(i, r)
            key = engine.tape_key(t)
            if key in seen:
                continue
            seen.add(key)
            try:
                engine.Plan(t, 0, P, prec, grad, segment=True)
            except Exception:
                pass


if __name__ == "__main__":
    engine._torch = lambda: _FakeTorch
    # cfg:prec[:x] (x: input gradients too, as cfg1/cfg2 train them)
    jobs = sys.argv[1:] or ["cfg4:c64", "cfg4:c128", "cfg3:c128", "cfg2:c64:x", "cfg1:c128:x", "cfg1:c64:x", "cfg5seg"]
    for job in jobs:
        if job == "cfg5seg":
            cfg5_segments()
            print("precompiled", job)
            continue
        parts = job.split(":")
        plan_for(parts[0], parts[1], want_x=len(parts) > 2 and parts[2] == "x")
        print("precompiled", job)
