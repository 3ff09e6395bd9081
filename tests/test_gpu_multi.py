"""GPU side of the multi-GPU layer on ONE device: amplitude sharding with
virtual ranks whose local segments run through the sm_100a plans (the
exchange is the host permutation of shard.swap_exchange), checked against
the oracle; batch sharding through the same evaluator the ranks use."""

import numpy as np
import pytest

from oracle import hq_oracle as O
from paper_2301_03251_b200 import dist as D
from paper_2301_03251_b200 import shard as S
from paper_2301_03251_b200 import workloads as wl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,g", [(8, 2), (11, 3), (15, 1)])
def test_amplitude_sharding_gpu_local_segments(n, g):
    rng = np.random.default_rng(n)
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
    ops = []
    for _ in range(60):
        k = kinds[rng.integers(len(kinds))]
        if k in ("CNOT", "CZ", "CR", "SWAP"):
            a, b = rng.choice(n, 2, replace=False)
            ops.append((k, (int(a), int(b)), float(rng.uniform(-6, 6)) if k == "CR" else None))
        else:
            ops.append((k, (int(rng.integers(n)),), float(rng.uniform(-6, 6)) if k[0] == "R" else None))
    sch = S.schedule(n, g, ops, [0, n - 1])
    shards, E = S.run_virtual(sch, S.gpu_apply_local(n - g))
    full = O.Circuit(n)
    for kind, t, a in ops:
        full.add(O.Op(kind, t, a))
    full.measure(0, n - 1)
    np.testing.assert_allclose(S.gather_state(shards, n - g, sch.final_layout), O.simulate(full), atol=1e-11)
    assert E == pytest.approx(O.expectation(full), abs=1e-11)


def test_batch_sharding_evaluator_on_gpu():
    import math
    import torch
    from paper_2301_03251_b200 import engine, qsim, templates as T, tracer as tr
    b = wl.make_builder("cfg1", qsim, T)
    x, th = wl.inputs_for("cfg1", 10), wl.params_for("cfg1")
    tape, ok = tr.trace(b, x, th)
    plan = engine.Plan(tape, 4, 24, "c128", tr.classify(tape, 28, [True] * 28, math.pi / 2, 0.5))
    g = np.linspace(0.5, 1.5, 10)
    span, out, gx, gp = D.dp_forward_grad(D.plan_evaluator(plan, torch.device("cuda")), x, th, g)
    o, _, _, gxo, gpo = O.layer(wl.make_builder("cfg1", O, O), x, th, upstream=g)
    np.testing.assert_allclose(out, o, atol=1e-12)
    np.testing.assert_allclose(gx, gxo, atol=1e-12)
    np.testing.assert_allclose(gp, gpo, atol=1e-12)


@pytest.mark.parametrize("n,g", [(10, 2), (14, 3)])
def test_amplitude_sharding_device_resident_executor(n, g):
    """The executor ``run_nccl`` uses on GPUs (``gpu_apply_local_dev``: shards
    stay complex128 CUDA tensors, no host round trip), driven through the
    virtual-rank schedule, against the oracle."""
    import torch
    rng = np.random.default_rng(100 + n)
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
    ops = []
    for _ in range(80):
        k = kinds[rng.integers(len(kinds))]
        if k in ("CNOT", "CZ", "CR", "SWAP"):
            a, b = rng.choice(n, 2, replace=False)
            ops.append((k, (int(a), int(b)), float(rng.uniform(-6, 6)) if k == "CR" else None))
        else:
            ops.append((k, (int(rng.integers(n)),), float(rng.uniform(-6, 6)) if k[0] == "R" else None))
    sch = S.schedule(n, g, ops, [1, n - 2])
    dev_exec = S.gpu_apply_local_dev(n - g)
    calls = []

    def apply_local(shard, lops):
        out = dev_exec(torch.from_numpy(shard).to("cuda"), lops)
        assert out.is_cuda and out.dtype == torch.complex128
        calls.append(1)
        return out.cpu().numpy()
    shards, E = S.run_virtual(sch, apply_local)
    assert calls
    full = O.Circuit(n)
    for kind, t, a in ops:
        full.add(O.Op(kind, t, a))
    full.measure(1, n - 2)
    np.testing.assert_allclose(S.gather_state(shards, n - g, sch.final_layout), O.simulate(full), atol=1e-11)
    assert E == pytest.approx(O.expectation(full), abs=1e-11)
