"""cfg5: one 32-qubit depth-20 circuit (complex128, 64 GiB state), amplitude-
sharded over 2^g ranks (shard.py).  Forward E and the full
1280-parameter adjoint gradient.

  python tools/cfg5_sharded.py --schedule            # schedule only (no GPU)
  python tools/cfg5_sharded.py                       # 8 virtual ranks on ONE GPU
  torchrun --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 tools/cfg5_sharded.py   # 8 GPUs, NCCL

Virtual mode runs every rank's segment plans on one device (rank shards are
rows of one [8, 2^29] tensor; the exchange is an in-place block swap standing
in for the all-to-all) and reports, per rank, the device time of its local
work (CUDA events around each rank's segment / readout launches; max over
ranks), the exchange volume per GPU, and a MODELED 8-GPU time = max-rank local
time + exchanges x bytes / NVLink bandwidth (900 GB/s per direction, nominal:
one GPU cannot measure NVLink).  Under torchrun the real NCCL all-to-all path
runs and the line carries device time, max over ranks.
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2301_03251_b200 import shard as S, tracer as tr, workloads as wl  # noqa: E402


def hea(n, depth):
    from paper_2301_03251_b200 import qsim

    def builder(inputs, params):
        c = qsim.Circuit(n)
        k = 0
        for _ in range(depth):
            for q in range(n):
                c.ry(q, params[k])
                c.rz(q, params[k + 1])
                k += 2
            for q in range(n - 1):
                c.cnot(q, q + 1)
        c.measure(0)
        return c
    return builder, 2 * n * depth


class TimedExecutor:
    """GpuExecutor with CUDA events around every rank's launches."""

    def __init__(self, inner):
        import torch
        self.inner = inner
        self.torch = torch
        self.recs = []

    def _t(self, rank, kind, fn, *a):
        ev0 = self.torch.cuda.Event(enable_timing=True)
        ev1 = self.torch.cuda.Event(enable_timing=True)
        ev0.record()
        r = fn(*a)
        ev1.record()
        self.recs.append((rank, kind, ev0, ev1))
        return r

    def seg_forward(self, sc, i, rank, buf, x, t):
        return self._t(rank, "fwd", self.inner.seg_forward, sc, i, rank, buf, x, t)

    def seg_backward(self, sc, i, rank, psi, lam, x, t):
        return self._t(rank, "bwd", self.inner.seg_backward, sc, i, rank, psi, lam, x, t)

    def readout(self, sc, rank, buf, lam):
        return self._t(rank, "readout", self.inner.readout, sc, rank, buf, lam)

    def zeros_jac(self, sc):
        return self.inner.zeros_jac(sc)

    def per_rank(self):
        self.torch.cuda.synchronize()
        out = {}
        for rank, kind, a, b in self.recs:
            out.setdefault(rank, {}).setdefault(kind, 0.0)
            out[rank][kind] += a.elapsed_time(b)
        self.recs = []
        return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--depth", type=int, default=20)
    ap.add_argument("--g", type=int, default=3)
    ap.add_argument("--precision", default="c128")
    ap.add_argument("--schedule", action="store_true", help="print the schedule statistics only")
    ap.add_argument("--nvlink-gbs", type=float, default=900.0)
    a = ap.parse_args()
    builder, P = hea(a.n, a.depth)
    theta = wl.params_for("cfg5")
    theta = np.resize(theta, P)
    tape, ok = tr.trace(builder, np.zeros((1, 0)), theta)
    assert ok
    world = int(os.environ.get("WORLD_SIZE", "1"))
    g = a.g if world == 1 else int(round(math.log2(world)))
    sc = S.ShardedCircuit(tape, 0, P, g, a.precision)
    st = sc.stats()
    if a.schedule:
        print(json.dumps({"workload": f"cfg5 n={a.n} depth={a.depth} {a.precision}", **st}))
        return
    import torch
    amp = 16 if a.precision == "c128" else 8
    xbytes = st["exchange_bytes_per_gpu_each_way"]
    if world == 1:
        dev = torch.device("cuda:0")
        ex = TimedExecutor(S.GpuExecutor(dev))
        ex.inner.prepare(sc, range(sc.world))            # JIT every segment plan outside the timings
        E, grad, st_ = S.run_virtual(sc, theta, dev, want_grad=False, ex=ex)   # warm-up
        del st_
        torch.cuda.empty_cache()
        ex.per_rank()
        res = {}
        for mode in ("forward", "forward+adjoint"):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            E, grad, st_ = S.run_virtual(sc, theta, dev, want_grad=mode != "forward", ex=ex)
            ev1.record()
            torch.cuda.synchronize()
            del st_
            torch.cuda.empty_cache()
            pr = ex.per_rank()
            local = max(sum(v.values()) for v in pr.values())
            n_x = sc.sched.exchanges * (1 if mode == "forward" else 3)   # adjoint replays on psi and lam
            model = local + n_x * xbytes / (a.nvlink_gbs * 1e9) * 1e3
            passes = sum(int(ex.inner._plan(sc, i, 0).stats(1)["n_passes"]) for i in range(len(sc.sched.segments)))
            shard = amp * (1 << sc.L)
            hbm = passes * shard * (2 if mode == "forward" else 6)    # fwd: ψ r+w; +bwd: ψ, λ r+w
            res[mode] = {"virtual_total_ms": ev0.elapsed_time(ev1), "max_rank_local_ms": local,
                         "per_rank_local_ms": {r: round(sum(v.values()), 3) for r, v in sorted(pr.items())},
                         "exchanges": n_x, "modeled_8gpu_ms": model, "local_passes_per_rank": passes,
                         "hbm_bytes_per_rank_local": hbm, "local_hbm_GBps": hbm / (local / 1e3) / 1e9, "E": E,
                         "grad_norm": None if grad is None else float(np.linalg.norm(grad))}
        print(json.dumps({"workload": f"cfg5: n={a.n} depth={a.depth} {a.precision}, {sc.world} virtual ranks on 1 GPU",
                          "schedule": st, "nvlink_bytes_per_gpu_per_exchange_each_way": xbytes,
                          "nvlink_model": f"{a.nvlink_gbs} GB/s per direction (nominal; not measurable on 1 GPU)",
                          **res}))
        return
    import torch.distributed as dist
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device(f"cuda:{local_rank}")
    dist.init_process_group("nccl", device_id=dev)
    ex = S.GpuExecutor(dev)
    ex.prepare(sc, [rank])
    S.run_nccl(sc, theta, rank, world, dev, want_grad=True, ex=ex)          # warm-up (NCCL channels)
    out = {}
    for mode in ("forward", "forward+adjoint"):
        torch.cuda.synchronize()
        dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        E, grad, _ = S.run_nccl(sc, theta, rank, world, dev, want_grad=mode != "forward", ex=ex)
        ev1.record()
        torch.cuda.synchronize()
        t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[mode] = {"ms": float(t.item()), "E": E,
                     "grad_norm": None if grad is None else float(np.linalg.norm(grad))}
    if rank == 0:
        print(json.dumps({"workload": f"cfg5: n={a.n} depth={a.depth} {a.precision}, {world} GPUs (NCCL all-to-all)",
                          "schedule": st, "nvlink_bytes_per_gpu_per_exchange_each_way": xbytes, **out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
