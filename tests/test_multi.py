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
def _random_ops(n, depth, rng):
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
    ops = []
    for _ in range(depth):
        k = kinds[rng.integers(len(kinds))]
        if k in ("CNOT", "CZ", "CR", "SWAP"):
            a, b = rng.choice(n, 2, replace=False)
            ops.append((k, (int(a), int(b)), float(rng.uniform(-6, 6)) if k == "CR" else None))
        else:
            ops.append((k, (int(rng.integers(n)),), float(rng.uniform(-6, 6)) if k[0] == "R" else None))
    return ops


def _oracle_apply(L):
    def apply_local(shard, ops):
        c = O.Circuit(L)
        for kind, t, a in ops:
            c.add(O.Op(kind, t, a))
        return O.simulate(c, initial=shard)
    return apply_local


@pytest.mark.parametrize("n,g", [(5, 1), (7, 2), (8, 3), (10, 3)])
def test_amplitude_sharding_virtual_ranks_match_full_state(n, g):
    rng = np.random.default_rng(n * 10 + g)
    for trial in range(3):
        ops = _random_ops(n, 80, rng)
        measured = [int(q) for q in rng.choice(n, 3, replace=False)]
        sch = S.schedule(n, g, ops, measured)
        shards, E = S.run_virtual(sch, _oracle_apply(n - g))
        full = O.Circuit(n)
        for kind, t, a in ops:
            full.add(O.Op(kind, t, a))
        full.measure(*measured)
        want = O.simulate(full)
        got = S.gather_state(shards, n - g, sch.final_layout)
        np.testing.assert_allclose(got, want, atol=1e-12)
        assert E == pytest.approx(O.expectation(full), abs=1e-12)
        assert any(s[0] == "swap" for s in sch.steps) or g == 0


def test_cfg5_shape_schedule_swap_count_bounded():
    # the cfg5 layer structure at a small size: swaps stay O(layers)
    n, g, depth = 12, 3, 6
    th = np.random.default_rng(1).uniform(0, 2 * math.pi, depth * 2 * n)
    ops, k = [], 0
    for _ in range(depth):
        for q in range(n):
            ops.append(("RY", (q,), th[k])); ops.append(("RZ", (q,), th[k + 1])); k += 2
        for q in range(n - 1):
            ops.append(("CNOT", (q, q + 1), None))
    sch = S.schedule(n, g, ops, [0])
    n_swaps = sum(1 for s in sch.steps if s[0] == "swap")
    assert n_swaps <= 2 * (depth * g + g)   # lower bound: g per layer
    shards, E = S.run_virtual(sch, _oracle_apply(n - g))
    c = O.Circuit(n)
    for kind, t, a in ops:
        c.add(O.Op(kind, t, a))
    c.measure(0)
    assert E == pytest.approx(O.expectation(c), abs=1e-12)


def _shard_worker(rank, world, port, n, seed, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        rng = np.random.default_rng(seed)
        ops = _random_ops(n, 60, rng)
        measured = [int(x) for x in rng.choice(n, 2, replace=False)]
        sch = S.schedule(n, g, ops, measured)
        L = n - g
        oracle_apply = _oracle_apply(L)

        def apply_local_dev(shard, lops):   # CPU executor standing in for the GPU plan
            out = oracle_apply(shard.numpy(), lops)
            return torch.from_numpy(np.ascontiguousarray(out))
        shard, E = S.run_nccl(sch, apply_local_dev, rank, world, torch.device("cpu"))
        q.put((rank, shard.numpy(), E, sch.final_layout))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_amplitude_sharding_real_processes_gloo(world):
    # run_nccl's exchange path (pairwise isend/irecv of half shards, per-rank
    # phases, all-reduced readout) with real processes over gloo
    import torch.multiprocessing as mp
    n, seed = 7, 11 + world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 500) + world
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    rng = np.random.default_rng(seed)
    ops = _random_ops(n, 60, rng)
    measured = [int(x) for x in rng.choice(n, 2, replace=False)]
    full = O.Circuit(n)
    for kind, t, a in ops:
        full.add(O.Op(kind, t, a))
    full.measure(*measured)
    want = O.simulate(full)
    L = n - (world.bit_length() - 1)
    got = S.gather_state([r[1] for r in res], L, res[0][3])
    np.testing.assert_allclose(got, want, atol=1e-12)
    for r in res:
        assert r[2] == pytest.approx(O.expectation(full), abs=1e-12)
