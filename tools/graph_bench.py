"""Launch-bound configs through TorchQuantumLayer captured in a CUDA graph
(forward + backward per replay, no host work per step) vs eager calls."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_03251_b200 import qsim, workloads as wl, templates as T
from paper_2301_03251_b200.torch_layer import TorchQuantumLayer


def run(cfg, prec, B):
    n, d, P, _, _ = wl.CONFIGS[cfg]
    layer = TorchQuantumLayer(wl.make_builder(cfg, qsim, T), P, precision=prec,
                              param_init=wl.params_for(cfg), device="cuda")
    x = torch.tensor(wl.inputs_for(cfg, B), device="cuda", requires_grad=True)

    def step():
        layer(x).sum().backward()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N = 200
    e0.record()
    for _ in range(N):
        step()
    e1.record(); torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / N
    layer.params.grad = None
    x.grad = None
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(N):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    gms = e0.elapsed_time(e1) / N
    return {"config": cfg, "precision": prec, "batch": B, "eager_us_per_step": eager * 1e3,
            "graph_us_per_step": gms * 1e3, "graph_samples_per_s": B / (gms / 1e3)}


if __name__ == "__main__":
    for cfg, prec, B in (("cfg1", "c128", 64), ("cfg2", "c64", 256)):
        print(json.dumps(run(cfg, prec, B)), flush=True)
