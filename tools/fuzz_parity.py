"""Randomised parity sweep (not part of the suite): random circuits through the
streaming kernels at several tile sizes vs the oracle, values and gradients."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import hq_oracle as O
from paper_2301_03251_b200 import engine, Circuit

KINDS = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
if os.environ.get("FUZZ_KINDS"):   # e.g. a diagonal-heavy mix: RZ,RZ,RZ,CR,CR,RY,CNOT,CZ
    KINDS = os.environ["FUZZ_KINDS"].split(",")


def builder_for(n, depth, rng):
    plan = []
    for _ in range(depth):
        k = KINDS[rng.integers(len(KINDS))]
        two = k in ("CNOT", "CZ", "CR", "SWAP")
        tg = tuple(int(q) for q in rng.choice(n, 2 if two else 1, replace=False))
        plan.append((k, tg, int(rng.integers(0, 6))))
    if rng.random() < 0.5:   # trailing diagonal / monomial gates (readout-invariant diagonals are dropped)
        for _ in range(int(rng.integers(1, 8))):
            k = ["RZ", "CZ", "CR", "Z", "X", "CNOT", "SWAP", "Y"][rng.integers(8)]
            two = k in ("CNOT", "CZ", "CR", "SWAP")
            tg = tuple(int(q) for q in rng.choice(n, 2 if two else 1, replace=False))
            plan.append((k, tg, int(rng.integers(0, 6))))
    if rng.random() < 0.5:   # trailing permutation layer
        for q in range(n - 1):
            plan.append(("CNOT", (q, q + 1), 0))
    meas = [int(q) for q in rng.choice(n, int(rng.integers(1, 4)), replace=False)]

    def b(inputs, params, Circ=Circuit):
        c = Circ(n)
        for k, tg, v in plan:
            ang = (inputs[v] if v < 2 else params[v - 2]) if k in ("RX", "RY", "RZ", "CR") else None
            getattr(c, k.lower())(*tg) if ang is None else getattr(c, k.lower())(*tg, ang)
        c.measure(*meas)
        return c
    return b


def main(count=40, seed=2024):
    rng = np.random.default_rng(seed)
    worst = {"c64": 0.0, "c128": 0.0}
    for t in range(count):
        n = int(rng.integers(9, 16))
        tile = int(rng.integers(9, min(n, 12) + 1))
        os.environ["HQ_FORCE_STREAM"] = "1"
        os.environ["HQ_TILE_BITS"] = str(tile)
        b = builder_for(n, int(rng.integers(20, 90)), rng)
        x = rng.uniform(-3, 3, (2, 2)); th = rng.uniform(0, 6, 4)
        out, jx, jp, _, _ = O.layer(lambda i, p: b(i, p, Circ=O.Circuit), x, th)
        ref = np.concatenate([out, jx.ravel(), jp.ravel()])
        for prec in ("c128", "c64"):
            try:
                res, jac, info = engine.run_batch(b, x, th, True, True, prec, cache=engine.PlanCache(2))
            except Exception as exc:
                import paper_2301_03251_b200.tracer as tr
                tape, _ = tr.trace(b, x, th)
                print("FAILED", t, n, tile, prec, len(tape.ops), repr(exc)[:200], flush=True)
                os.environ["HQ_PLAN_WINDOWS"] = "1"
                try:
                    engine.Plan(tape, 2, 4, prec, tr.classify(tape, 6, [True] * 6, math.pi / 2, 0.5))
                except Exception:
                    pass
                os.environ.pop("HQ_PLAN_WINDOWS")
                continue
            got = np.concatenate([res, jac.cpu().numpy()[:, :2].ravel(), jac.cpu().numpy()[:, 2:].ravel()])
            err = float(np.max(np.abs(got - ref)) / max(1.0, np.max(np.abs(ref))))
            worst[prec] = max(worst[prec], err)
            lim = 1e-10 if prec == "c128" else 1e-4
            if err > lim:
                print("MISMATCH", t, n, tile, prec, err, info["plan"].description[:200], flush=True)
    print("worst", worst, "circuits", count, "seed", seed, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 40, int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
