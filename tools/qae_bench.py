"""QAELayer (the reference's own autoencoder) forward +
parameter gradient throughput on one GPU, EXACT_PROB, complex128."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import QAELayer, Tensor, backward, tsum, workloads as wl

for trash, total, B in ((2, 7, 256), (2, 12, 64)):
    layer = QAELayer(trash, total, machine_type="exact_prob")
    dim = 1 << (total - 1 - trash)
    x = wl.qae_vectors(B, dim, min(dim, 128), seed=0)
    def step():
        out = layer(Tensor(x, dtype=np.float64))
        backward(tsum(out))
        layer.params.zero_grad()
    step(); step(); torch.cuda.synchronize()       # the first call runs lazily, the second eagerly
    ts = []
    for _ in range(7):
        t0 = time.perf_counter(); step(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    dt = float(np.median(ts))
    info = getattr(layer, "last_info", None)
    print(json.dumps({"trash": trash, "total": total, "batch": B, "params": int(layer.params.data.size),
                      "s_per_step": dt, "samples_per_s": B / dt, "stat": "median of 7 steps",
                      "plan": (info["plan"].description[:160] if info and "plan" in info else None)}), flush=True)
