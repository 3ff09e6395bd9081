"""cfg2 end to end (SURVEY.md §8(d) cfg 2): hybrid CNN + 10-qubit VQC on
synthetic 28x28 images, one training step = forward + backward + Adam, all on
the device.  The classical layers are plain PyTorch (out of scope here); the
quantum head is TorchQuantumLayer (hq_forward / hq_vjp, no host round trip),
so the whole step captures into one CUDA graph.  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_03251_b200 import qsim, workloads as wl, templates as T
from paper_2301_03251_b200.torch_layer import TorchQuantumLayer


class Hybrid(torch.nn.Module):
    def __init__(self, precision="c64"):
        super().__init__()
        n, d, P, _, _ = wl.CONFIGS["cfg2"]
        self.features = torch.nn.Sequential(
            torch.nn.Conv2d(1, 6, 5), torch.nn.ReLU(), torch.nn.MaxPool2d(2),
            torch.nn.Conv2d(6, 16, 5), torch.nn.ReLU(), torch.nn.MaxPool2d(2), torch.nn.Flatten(),
            torch.nn.Linear(256, d))
        self.q = TorchQuantumLayer(wl.make_builder("cfg2", qsim, T), P, precision=precision,
                                   param_init=wl.params_for("cfg2"), device="cuda")
        self.head = torch.nn.Linear(1, 2)

    def forward(self, img):
        return self.head(self.q(self.features(img)))


def main(B=256, steps=50):
    torch.manual_seed(0)
    model = Hybrid().cuda()
    opt = torch.optim.Adam(model.parameters(), lr=1e-3, capturable=True)
    img = torch.rand(B, 1, 28, 28, device="cuda")
    y = torch.randint(0, 2, (B,), device="cuda")
    lossf = torch.nn.CrossEntropyLoss()

    def step():
        opt.zero_grad(set_to_none=False)
        loss = lossf(model(img), y)
        loss.backward()
        opt.step()
        return loss

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):          # warm-up and eager timing on the side stream (capture recipe)
        for _ in range(3):
            step()
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / steps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        loss = step()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / steps
    print(json.dumps({"workload": "cfg2 hybrid CNN + 10-qubit VQC (complex64), B=256, forward+backward+Adam",
                      "data": "synthetic 28x28 images", "eager_ms_per_step": eager, "graph_ms_per_step": graph,
                      "graph_samples_per_s": B / (graph / 1e3), "loss": float(loss.item()),
                      "q_params_grad_norm": float(model.q.params.grad.norm().item())}))


if __name__ == "__main__":
    main()
