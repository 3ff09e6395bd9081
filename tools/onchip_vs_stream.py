"""On-chip interpreter vs specialised streaming kernels for small circuits
(HEA: RY/RZ layers + CNOT chain, θ gradient), device-timed, B=1024."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, tracer as tr


def hea(n, depth):
    def b(inputs, params):
        c = qsim.Circuit(n)
        for q in range(n):
            c.ry(q, inputs[q])
        k = 0
        for _ in range(depth):
            for q in range(n):
                c.ry(q, params[k]); c.rz(q, params[k + 1]); k += 2
            for q in range(n - 1):
                c.cnot(q, q + 1)
        c.measure(0)
        return c
    return b


def run(n, prec, B=1024, depth=6, steps=10):
    P = 2 * n * depth
    b = hea(n, depth)
    rng = np.random.default_rng(n)
    x = rng.uniform(-3, 3, (B, n)); th = rng.uniform(0, 6, P)
    tape, ok = tr.trace(b, x, th)
    grad = tr.classify(tape, n + P, [False] * n + [True] * P, math.pi / 2, 0.5)
    plan = engine.Plan(tape, n, P, prec, grad)
    xd = torch.tensor(x, device="cuda"); td = torch.tensor(th, device="cuda")
    up = torch.ones(B, dtype=torch.float64, device="cuda")
    def step():
        out, jac = plan.forward(xd, td, True)
        return out, plan.vjp(jac, up, False, True)[1]
    for _ in range(3): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): o, g = step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return ms, o.cpu().numpy(), g.cpu().numpy(), plan.description.split(" [")[0]


if __name__ == "__main__":
    for prec in ("c64", "c128"):
        for n in range(7, 14):
            os.environ.pop("HQ_ONCHIP_MAX", None)
            a = run(n, prec)
            os.environ["HQ_ONCHIP_MAX"] = "0"
            try:
                s = run(n, prec)
            except Exception as e:
                print(json.dumps({"n": n, "prec": prec, "onchip_ms": a[0], "stream": str(e)[:80]}), flush=True)
                continue
            print(json.dumps({"n": n, "prec": prec, "onchip_ms": round(a[0], 4), "stream_ms": round(s[0], 4),
                              "max_out_diff": float(np.abs(a[1] - s[1]).max()),
                              "max_grad_diff": float(np.abs(a[2] - s[2]).max()), "stream_plan": s[3][-60:]}), flush=True)
