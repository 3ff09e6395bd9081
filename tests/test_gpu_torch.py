"""Device-resident torch boundary (TorchQuantumLayer) vs the oracle, plus a
hybrid Linear -> quantum -> Linear training step and CUDA-graph capture."""

import numpy as np
import pytest

from oracle import hq_oracle as O
from paper_2301_03251_b200 import qsim, workloads as wl
from paper_2301_03251_b200 import templates as T

pytestmark = pytest.mark.gpu


def test_torch_layer_matches_oracle_gradients():
    import torch
    from paper_2301_03251_b200.torch_layer import TorchQuantumLayer
    x_np, th = wl.inputs_for("cfg1", 12), wl.params_for("cfg1")
    layer = TorchQuantumLayer(wl.make_builder("cfg1", qsim, T), 24, param_init=th, device="cuda")
    x = torch.tensor(x_np, device="cuda", requires_grad=True)
    g = torch.linspace(0.5, 1.5, 12, dtype=torch.float64, device="cuda")
    out = layer(x)
    (out[:, 0] * g).sum().backward()
    o, _, _, gx, gp = O.layer(wl.make_builder("cfg1", O, O), x_np, th, upstream=g.cpu().numpy())
    np.testing.assert_allclose(out[:, 0].detach().cpu().numpy(), o, atol=1e-12)
    np.testing.assert_allclose(x.grad.cpu().numpy(), gx, atol=1e-12)
    np.testing.assert_allclose(layer.params.grad.cpu().numpy(), gp, atol=1e-12)


def test_hybrid_model_step_and_graph_capture():
    import torch
    from paper_2301_03251_b200.torch_layer import TorchQuantumLayer
    torch.manual_seed(0)
    qlayer = TorchQuantumLayer(wl.make_builder("cfg2", qsim, T), 60, precision="c64",
                               param_init=wl.params_for("cfg2"), device="cuda")
    model = torch.nn.Sequential(torch.nn.Linear(16, 10), qlayer, torch.nn.Linear(1, 2)).cuda()
    opt = torch.optim.SGD(model.parameters(), lr=0.1)
    x = torch.randn(64, 16, device="cuda")
    y = torch.randint(0, 2, (64,), device="cuda")
    losses = []
    for _ in range(15):
        opt.zero_grad()
        loss = torch.nn.functional.cross_entropy(model(x), y)
        loss.backward()
        opt.step()
        losses.append(loss.item())
    assert qlayer.params.grad is not None and torch.isfinite(qlayer.params.grad).all()
    assert qlayer.params.grad.abs().max().item() > 0.0
    # full-batch SGD on a fixed batch descends
    assert losses[-1] < losses[0], losses
    del loss
    # forward + backward of a quantum layer inside a CUDA graph (no host syncs
    # after the first call); a fresh layer so no autograd node predates capture
    qlayer = TorchQuantumLayer(wl.make_builder("cfg2", qsim, T), 60, precision="c64",
                               param_init=wl.params_for("cfg2"), device="cuda")
    xs = torch.randn(64, 10, device="cuda", requires_grad=True)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            qlayer(xs).sum().backward()
    torch.cuda.current_stream().wait_stream(s)
    qlayer.params.grad = None
    xs.grad = None
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = qlayer(xs)
        out.sum().backward()
    graph.replay()
    torch.cuda.synchronize()
    ref = qlayer(xs.detach()).detach()
    torch.testing.assert_close(out.detach(), ref)


def test_torch_layer_width_change_retraces():
    """The tape's variable ids depend on the input width: a new width retraces."""
    import torch
    from paper_2301_03251_b200.torch_layer import TorchQuantumLayer

    def b(inputs, params):
        c = qsim.Circuit(3)
        for q, v in enumerate(inputs):
            c.ry(q % 3, v)
        c.rx(0, params[0]); c.cnot(0, 1); c.rz(1, params[1]); c.cnot(1, 2); c.measure(0, 2)
        return c

    def bo(inputs, params):
        c = O.Circuit(3)
        for q, v in enumerate(inputs):
            c.ry(q % 3, v)
        c.rx(0, params[0]); c.cnot(0, 1); c.rz(1, params[1]); c.cnot(1, 2); c.measure(0, 2)
        return c
    th = np.array([0.3, -1.1])
    layer = TorchQuantumLayer(b, 2, param_init=th, device="cuda")
    for d in (3, 5):
        x_np = np.random.default_rng(d).uniform(-2, 2, (6, d))
        x = torch.tensor(x_np, device="cuda", requires_grad=True)
        layer.params.grad = None
        out = layer(x)
        out.sum().backward()
        o, _, _, gx, gp = O.layer(bo, x_np, th)
        np.testing.assert_allclose(out[:, 0].detach().cpu().numpy(), o, atol=1e-12)
        np.testing.assert_allclose(x.grad.cpu().numpy(), gx, atol=1e-12)
        np.testing.assert_allclose(layer.params.grad.cpu().numpy(), gp, atol=1e-12)


def test_torch_layer_structure_change_raises():
    """A builder whose circuit changes between batches (here through outside
    state) is caught by the per-batch re-check instead of silently reusing the
    first batch's tape."""
    import torch
    from paper_2301_03251_b200 import CircuitError
    from paper_2301_03251_b200.torch_layer import TorchQuantumLayer
    calls = {"n": 0}

    def b(inputs, params):
        calls["n"] += 1
        c = qsim.Circuit(2)
        c.ry(0, inputs[0])
        if calls["n"] > 3:          # after the first batch's trace
            c.x(1)
        c.rz(1, params[0]); c.cnot(0, 1); c.measure(0)
        return c
    layer = TorchQuantumLayer(b, 1, param_init=[0.2], device="cuda")
    x = torch.tensor([[0.1], [0.4]], dtype=torch.float64, device="cuda")
    layer(x)
    with pytest.raises(CircuitError):
        layer(x)
