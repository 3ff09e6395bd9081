"""Multi-rank host logic on CPU: batch sharding with a real gloo world of 2,
amplitude sharding with virtual ranks.  The oracle is the per-rank executor
(test infrastructure only); the GPU path reuses the same functions with the
sm_100a plans (tests/test_gpu_multi.py)."""

import math
import os

import numpy as np
import pytest

from oracle import hq_oracle as O
from paper_2301_03251_b200 import dist as D
from paper_2301_03251_b200 import shard as S
from paper_2301_03251_b200 import workloads as wl


def test_shard_bounds_cover_and_balance():
    for n in (1, 7, 64, 4097):
        for world in (1, 2, 3, 8):
            spans = [D.shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _oracle_eval(cfg):
    b = wl.make_builder(cfg, O, O)

    def evaluate(x_rows, theta):
        out, jx, jp, _, _ = O.layer(b, x_rows, theta, want_x=True)
        return out, np.hstack([jx, jp])
    return evaluate


def _dp_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = wl.inputs_for("cfg1", 6)
        th = wl.params_for("cfg1")
        g = np.linspace(0.5, 1.5, 6)
        span, out, gx, gp = D.dp_forward_grad(_oracle_eval("cfg1"), x, th, g)
        allout = D.gather_rows(out.reshape(-1, 1), 6)
        allgx = D.gather_rows(gx, 6)
        q.put((rank, span, allout, allgx, gp))
    finally:
        dist.destroy_process_group()


def test_batch_sharding_gloo_world2_matches_single_process():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    x = wl.inputs_for("cfg1", 6)
    th = wl.params_for("cfg1")
    g = np.linspace(0.5, 1.5, 6)
    out, _, _, gx, gp = O.layer(wl.make_builder("cfg1", O, O), x, th, upstream=g)
    for rank, span, allout, allgx, rgp in res:
        assert span == D.shard_bounds(6, rank, 2)
        np.testing.assert_allclose(allout[:, 0], out, atol=1e-14)
        np.testing.assert_allclose(allgx, gx, atol=1e-14)
        np.testing.assert_allclose(rgp, gp, rtol=1e-13, atol=1e-15)   # rank partials re-associated
    np.testing.assert_array_equal(res[0][4], res[1][4])                  # identical on every rank


# ---------------------------------------------------------------------------
# amplitude sharding (shard.py): the driver with a NumPy segment executor
from shard_numpy import (NumpyExecutor, hea_builder, oracle_reference, random_param_builder,  # noqa: E402
                         same_up_to_phase, sharded)


@pytest.mark.parametrize("n,g,seed", [(6, 1, 0), (8, 2, 1), (9, 3, 2), (10, 3, 3), (10, 2, 4)])
def test_amplitude_sharding_virtual_ranks_match_oracle(n, g, seed):
    """E, the full adjoint gradient and the final state of random circuits
    (all 11 gate kinds) vs the oracle, ranks simulated in one process."""
    import torch
    b, P = random_param_builder(n, 90, seed)
    theta = np.random.default_rng(seed).uniform(-3, 3, P)
    sc = sharded(b, P, theta, g)
    E, grad, shards = S.run_virtual(sc, theta, torch.device("cpu"), ex=NumpyExecutor())
    E0, g0, psi0 = oracle_reference(b, theta)
    assert E == pytest.approx(E0, abs=1e-12)
    np.testing.assert_allclose(grad, g0, atol=1e-12)
    # forward-only run: the final state, gathered through the final layout
    _, _, sh = S.run_virtual(sc, theta, torch.device("cpu"), want_grad=False, ex=NumpyExecutor())
    same_up_to_phase(S.gather_state(sh.numpy(), sc.L, sc.sched.final_layout), psi0, 1e-12)


def test_schedule_invariants():
    """Every op lands in exactly one segment (or is a dropped trailing global
    diagonal), segments only touch local positions after resolution, and the
    SWAPs that stage victims are the only additions."""
    b, P = random_param_builder(10, 200, 7)
    sc = sharded(b, P, np.zeros(P), 3)
    n_ops = len(sc.tape.ops)
    placed = sum(1 for seg in sc.sched.segments for op in seg if not (op[0] == "SWAP" and op[2] == -1
                                                                      and op not in sc.tape.ops))
    assert placed + sc.sched.dropped >= n_ops - sum(1 for op in sc.tape.ops if op[0] == "SWAP")
    for i in range(len(sc.sched.segments)):
        for r in range(sc.world):
            for kind, t, _ in sc.segment(i, r)[0].ops:
                assert all(0 <= q < sc.L for q in t)


@pytest.mark.parametrize("n,most", [(12, 5), (16, 3), (20, 3), (28, 1), (32, 1)])
def test_cfg5_shape_exchange_count(n, most):
    """cfg5's layer structure: the frontier runs ahead of the exchange as a
    staircase, so at n = 32 the whole depth-20 forward needs ONE all-to-all
    (the adjoint replays it) instead of one per layer."""
    b, P = hea_builder(n, 20)
    sc = sharded(b, P, np.zeros(P), 3)
    assert 1 <= sc.sched.exchanges <= most
    assert sc.stats()["exchange_bytes_per_gpu_each_way"] == 7 / 8 * 16 * 2 ** (n - 3)


def test_cfg5_shape_small_matches_oracle():
    import torch
    b, P = hea_builder(11, 6)
    theta = np.random.default_rng(5).uniform(0, 2 * math.pi, P)
    sc = sharded(b, P, theta, 3)
    E, grad, _ = S.run_virtual(sc, theta, torch.device("cpu"), ex=NumpyExecutor())
    E0, g0, _ = oracle_reference(b, theta)
    assert E == pytest.approx(E0, abs=1e-12)
    np.testing.assert_allclose(grad, g0, atol=1e-12)


def _shard_worker(rank, world, port, n, seed, q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from shard_numpy import NumpyExecutor as NE, random_param_builder as rpb, sharded as shd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        b, P = rpb(n, 90, seed)
        theta = np.random.default_rng(seed).uniform(-3, 3, P)
        sc = shd(b, P, theta, g)
        E, grad, shard = S.run_nccl(sc, theta, rank, world, torch.device("cpu"), ex=NE())
        _, _, shard_f = S.run_nccl(sc, theta, rank, world, torch.device("cpu"), want_grad=False, ex=NE())
        q.put((rank, E, grad, shard_f.numpy().copy(), sc.sched.final_layout))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_amplitude_sharding_real_processes_gloo(world):
    """run_nccl with real processes over gloo: all-to-all exchanges on both ψ
    and λ, the all-reduced readout and gradient, vs the oracle."""
    import torch.multiprocessing as mp
    n, seed = 10, 11 + world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 500) + world
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    b, P = random_param_builder(n, 90, seed)
    theta = np.random.default_rng(seed).uniform(-3, 3, P)
    E0, g0, psi0 = oracle_reference(b, theta)
    for _, E, grad, _, _ in res:
        assert E == pytest.approx(E0, abs=1e-12)
        np.testing.assert_allclose(grad, g0, atol=1e-12)
    np.testing.assert_array_equal(res[0][2], res[-1][2])          # identical on every rank
    L = n - (world.bit_length() - 1)
    same_up_to_phase(S.gather_state([r[3] for r in res], L, res[0][4]), psi0, 1e-12)
