# A/B: QAE (2,12) throughput with the round-1 tree vs the current tree (same box)
echo "== r01"; (cd scratch_r01 && timeout 900 python tools/qae_bench.py 2>&1 | cut -c1-160)
echo "== r02"; timeout 900 python tools/qae_bench.py 2>&1 | cut -c1-160
echo "== r02 jacobian=eager"; timeout 900 python - <<'PY' 2>&1 | cut -c1-200
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2301_03251_b200 import QAELayer, Tensor, backward, tsum, workloads as wl
layer = QAELayer(2, 12, machine_type="exact_prob", jacobian="eager")
x = wl.qae_vectors(64, 512, 128, seed=0)
def step():
    out = layer(Tensor(x, dtype=np.float64)); backward(tsum(out)); layer.params.zero_grad()
step(); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3): step()
torch.cuda.synchronize(); print("eager s/step", (time.perf_counter() - t0) / 3)
PY
