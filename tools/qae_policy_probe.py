"""Debug probe: per-step timings and run_batch calls of QAELayer (2,12) under
the auto / eager jacobian policies."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import QAELayer, Tensor, backward, tsum, engine, workloads as wl
orig = engine.run_batch
calls = []
def rb(builder, xd, pd, want_x, want_p, *a, **k):
    t0 = time.perf_counter(); r = orig(builder, xd, pd, want_x, want_p, *a, **k); torch.cuda.synchronize()
    calls.append((want_p, round(1e3 * (time.perf_counter() - t0), 2)))
    return r
engine.run_batch = rb
x = wl.qae_vectors(64, 512, 128, seed=0)
for mode in ("auto", "eager"):
    layer = QAELayer(2, 12, machine_type="exact_prob", jacobian=mode)
    for s in range(4):
        t0 = time.perf_counter()
        out = layer(Tensor(x, dtype=np.float64)); backward(tsum(out)); layer.params.zero_grad()
        torch.cuda.synchronize()
        print(mode, s, round(1e3 * (time.perf_counter() - t0), 2), "ms", calls, flush=True); calls.clear()
