"""cfg5 amplitude-sharded forward over NCCL: one rank per GPU,
2^g ranks hold the 2^n amplitudes (top g index bits = rank), global-qubit
swaps are pairwise NCCL send/recv of half a shard, local segments run through
the sm_100a plans on device-resident shards (shard.gpu_apply_local_dev).

  torchrun --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 tools/cfg5_sharded.py [--n 32]
  python tools/cfg5_sharded.py --n 20          # one rank (g = 0), functional check

Prints one JSON line on rank 0: device time of the second run (CUDA events, max
over ranks), E, the swap count and the schedule's local-step count.
"""
import argparse, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
from paper_2301_03251_b200 import shard as S, workloads as wl


def cfg5_ops(n, depth, theta):
    ops, k = [], 0
    for _ in range(depth):
        for q in range(n):
            ops.append(("RY", (q,), float(theta[k % theta.size])))
            ops.append(("RZ", (q,), float(theta[(k + 1) % theta.size])))
            k += 2
        for q in range(n - 1):
            ops.append(("CNOT", (q, q + 1), None))
    return ops


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--depth", type=int, default=20)
    ap.add_argument("--precision", default="c128")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    g = int(round(math.log2(world)))
    if 1 << g != world:
        raise SystemExit("world size must be a power of two")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
    ops = cfg5_ops(a.n, a.depth, wl.params_for("cfg5"))
    sch = S.schedule(a.n, g, ops, [0])
    ex = S.gpu_apply_local_dev(a.n - g, a.precision)
    S.run_nccl(sch, ex, rank, world, dev)   # warm-up: NCCL setup and the local segments' JIT plans
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    shard, E = S.run_nccl(sch, ex, rank, world, dev)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev if world > 1 else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"workload": f"cfg5-shape: n={a.n} depth={a.depth} {a.precision}, amplitude-sharded",
                          "ranks": world, "global_qubits": g, "ms": float(t.item()), "E": E,
                          "swaps": sum(1 for s in sch.steps if s[0] == "swap"),
                          "local_steps": sum(1 for s in sch.steps if s[0] == "local"),
                          "note": "second run of the schedule (the first builds the plans and NCCL channels)"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
