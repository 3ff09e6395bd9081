"""GPU side of the multi-GPU layer on ONE device.

Amplitude sharding: every rank's local segments run as segment plans
(hq_plan_create_segment / hq_seg_forward / hq_seg_backward /
hq_shard_readout) on device shards; ranks are virtual (rows of one tensor,
exchanged by the in-place block swap that stands in for the NCCL all-to-all —
one GPU never runs ranks that wait on each other).  Checked against the CPU
oracle: E, the full adjoint gradient and the final state.  Batch sharding:
the evaluator the ranks use."""

import math

import numpy as np
import pytest

from conftest import normwise_error, parity_log
from oracle import hq_oracle as O
from paper_2301_03251_b200 import dist as D
from paper_2301_03251_b200 import shard as S
from paper_2301_03251_b200 import workloads as wl
from shard_numpy import hea_builder, oracle_reference, random_param_builder, same_up_to_phase, sharded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,g,seed", [(10, 1, 0), (12, 2, 1), (12, 3, 2), (14, 3, 3), (16, 2, 4)])
@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_amplitude_sharding_segment_plans_vs_oracle(n, g, seed, prec):
    import torch
    b, P = random_param_builder(n, 120, seed)
    theta = np.random.default_rng(seed).uniform(-3, 3, P)
    sc = sharded(b, P, theta, g, prec)
    ex = S.GpuExecutor(torch.device("cuda"))
    E, grad, _ = S.run_virtual(sc, theta, torch.device("cuda"), ex=ex)
    E0, g0, psi0 = oracle_reference(b, theta)
    tol = 1e-10 if prec == "c128" else 1e-5
    parity_log(f"shard.n{n}g{g}.E:{prec}", normwise=abs(E - E0) / max(abs(E0), 1.0))
    parity_log(f"shard.n{n}g{g}.grad:{prec}", normwise=normwise_error(grad, g0, floor=1.0))
    assert abs(E - E0) < tol * max(abs(E0), 1.0)
    assert normwise_error(grad, g0, floor=1.0) < tol
    _, _, sh = S.run_virtual(sc, theta, torch.device("cuda"), want_grad=False, ex=ex)
    got = S.gather_state(sh.cpu().numpy().astype(np.complex128), sc.L, sc.sched.final_layout)
    same_up_to_phase(got, psi0, 1e-11 if prec == "c128" else 2e-6)


@pytest.mark.parametrize("n", [14, 18])
def test_cfg5_shape_sharded_forward_and_adjoint(n):
    """cfg5's layer structure (depth 20, g = 3) on segment plans vs the oracle."""
    import torch
    b, P = hea_builder(n, 20 if n <= 14 else 6)
    theta = np.random.default_rng(n).uniform(0, 2 * math.pi, P)
    sc = sharded(b, P, theta, 3)
    E, grad, _ = S.run_virtual(sc, theta, torch.device("cuda"))
    E0, g0, _ = oracle_reference(b, theta)
    assert abs(E - E0) < 1e-10
    assert normwise_error(grad, g0) < 1e-10


def test_sharded_matches_unsharded_plan_at_full_depth():
    """n = 20, depth 20 (cfg5's shape at 20 qubits): the sharded forward + adjoint
    against the single-GPU plan of the same tape (E and all 800 derivatives)."""
    import torch
    from paper_2301_03251_b200 import engine, tracer as tr
    b, P = hea_builder(20, 20)
    theta = wl.params_for("cfg5")[:P]
    sc = sharded(b, P, theta, 3)
    E, grad, _ = S.run_virtual(sc, theta, torch.device("cuda"))
    tape = sc.tape
    plan = engine.Plan(tape, 0, P, "c128", tr.classify(tape, P, [True] * P, math.pi / 2, 0.5))
    out, jac = plan.forward(torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                            torch.tensor(theta, device="cuda"), True)
    assert abs(E - float(out[0])) < 1e-12
    assert normwise_error(grad, jac[0].cpu().numpy()) < 1e-10


def test_segment_plan_errors():
    import torch
    from paper_2301_03251_b200 import ConfigError, engine, qsim, tracer as tr
    b, P = hea_builder(10, 2)
    tape, _ = tr.trace(b, np.zeros((1, 0)), np.zeros(P))
    plan = engine.Plan(tape, 0, P, "c128")
    with pytest.raises(ConfigError):
        plan.seg_forward(torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                         torch.zeros(P, dtype=torch.float64, device="cuda"),
                         torch.zeros(1 << 10, dtype=torch.complex128, device="cuda"))


def test_batch_sharding_evaluator_on_gpu():
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


def test_library_communicator_single_rank():
    """hq_comm_* with one rank (the only size one GPU allows): all-reduce is
    the identity, the all-to-all copies the single chunk, and hq_backward_dp
    equals hq_forward + hq_vjp."""
    import torch
    from paper_2301_03251_b200 import engine, qsim, templates as T, tracer as tr
    comm = D.LibComm()
    assert comm.world == 1
    t = torch.arange(10, dtype=torch.float64, device="cuda")
    comm.allreduce_(t)
    torch.testing.assert_close(t, torch.arange(10, dtype=torch.float64, device="cuda"))
    src = torch.randn(1 << 12, dtype=torch.complex128, device="cuda")
    dst = torch.empty_like(src)
    comm.alltoall(src, dst)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    b = wl.make_builder("cfg2", qsim, T)
    x, th = wl.inputs_for("cfg2", 24), wl.params_for("cfg2")
    tape, _ = tr.trace(b, x, th)
    plan = engine.Plan(tape, 10, 60, "c128", tr.classify(tape, 70, [True] * 70, math.pi / 2, 0.5))
    xd, td = torch.tensor(x, device="cuda"), torch.tensor(th, device="cuda")
    up = torch.linspace(0.5, 1.5, 24, dtype=torch.float64, device="cuda")
    out, gx, gt = comm.backward_dp(plan, xd, td, up, want_x=True)
    o2, jac = plan.forward(xd, td, True)
    gx2, gt2 = plan.vjp(jac, up, True, True)
    torch.testing.assert_close(out, o2, rtol=0, atol=0)
    torch.testing.assert_close(gx, gx2, rtol=0, atol=0)
    torch.testing.assert_close(gt, gt2, rtol=0, atol=0)
    comm.close()
