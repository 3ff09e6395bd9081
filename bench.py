#!/usr/bin/env python
"""Benchmark: circuit forward+grad evals/s on the cfg4 workload.

Workload ("step"): one forward + full parameter gradient of a batch of the
20-qubit hardware-efficient ansatz (depth 10, 610 gates, 400 parameters,
complex64) — BASELINE.json configs[3], the configuration the metric's
"% HBM roofline" and the 1/2/4/8-GPU scaling are quoted on.  Weak scaling:
every rank owns 4096 samples; the 400-dim gradient is all-reduced over NCCL.

  python bench.py [--gpus N --steps K --warmup W]          (our arm)
  python bench.py --impl reference [...]                     (reference CPU arm)

One JSON line on rank 0.  `value` is device-timed (CUDA events, inputs resident
in HBM, max over ranks); `e2e` goes through the public QuantumLayer API with
host tensors (H2D of inputs, D2H of outputs and gradients inside the timed
region); `roofline` uses the amplitude-update kernel's live CUDA-event time;
`cpu_baseline` times the NumPy oracle port of the reference on a bounded sample;
`complex128` repeats the device-timed step at the reference's own precision.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "circuit forward+grad evals/sec (n qubits, depth d, batch B); % HBM roofline"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--batch", type=int, default=None, help="samples per GPU")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c128", action="store_true", help="skip the complex128 companion measurement")
    ap.add_argument("--backend", default="nccl", help="process-group backend (gloo: dry runs of the "
                    "multi-rank path with several ranks on one device)")
    return ap.parse_args()


def fp_peak(prec):
    """Measured FMA throughput (tools/fma_peak.cu -> profiles/r01_fma_peak.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "r01_fma_peak.json")) as f:
            m = json.load(f)
        return (m["fp32_ffma2_tflops"] if prec == "c64" else m["fp64_dfma_tflops"]), "measured (tools/fma_peak.cu)"
    except Exception:
        return (75.0 if prec == "c64" else 37.0), "datasheet"


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [c.strip() for c in line.split(",")]
                if len(f) < 9:
                    continue
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                for name, val in zip(names, f[5:9]):
                    if val.lower() == "active":
                        reasons.add(name)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------
def cpu_baseline(cfg, x0, theta, budget_pairs=1):
    """Oracle port of the reference, one core, bounded sample."""
    from oracle import hq_oracle as O
    from paper_2301_03251_b200 import workloads as wl
    b = wl.make_builder(cfg, O, O)
    t0 = time.perf_counter()
    evals = O.sample_cost(b, x0, theta, budget_pairs)
    dt = time.perf_counter() - t0
    per_sample = 1 + 2 * theta.size          # cfg4: θ-only gradient (801 evaluations)
    return {"value": evals / dt / per_sample, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"1 sample: forward + {budget_pairs} shifted parameter pairs = {evals} of the "
                      f"{per_sample} circuit evaluations one forward+grad takes (reference "
                      f"parameter_shift_grad, qnn.py:35-52), {dt:.1f} s, extrapolated linearly"}


def _ref_worker(args):
    cfg, x_row, theta = args
    sys.path.insert(0, REPO)
    from oracle import hq_oracle as O
    from paper_2301_03251_b200 import workloads as wl
    return O.run(wl.make_builder(cfg, O, O), x_row, theta)


def run_reference(a):
    """--impl reference: the NumPy port of the reference on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor
    from paper_2301_03251_b200 import workloads as wl
    cfg = a.config
    n, d, P, B, prec = wl.CONFIGS[cfg]
    x = wl.inputs_for(cfg, 64 if cfg == "cfg4" else B)
    theta = wl.params_for(cfg)
    cores = os.cpu_count() or 1
    per_sample = 1 + 2 * P + (2 * d if cfg in ("cfg1", "cfg2") else 0)
    times = []
    with ProcessPoolExecutor(cores) as ex:
        for step in range(a.warmup + a.steps):
            # each step: one circuit evaluation per core (a shard of the
            # 1 + 2P evaluations of the per-sample shift rule)
            jobs = [(cfg, x[i % len(x)], theta) for i in range(cores)]
            t0 = time.perf_counter()
            list(ex.map(_ref_worker, jobs))
            dt = time.perf_counter() - t0
            if step >= a.warmup:
                times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = cores / (ms / 1e3) / per_sample
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, a.gpus, B, "c128"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"per step {cores} circuit evaluations in parallel "
                                       f"(1 per core) of the {per_sample} a sample's "
                                       f"forward+grad needs; samples/s extrapolated"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(cfg, world, B, prec):
    from paper_2301_03251_b200 import workloads as wl
    n = wl.CONFIGS[cfg][0]
    R, D, G = wl.gate_counts(cfg)
    return {"workload": f"{cfg}: {n}-qubit circuit ({G} gates), forward + {D}-angle gradient, "
                        f"{B} samples per GPU",
            "n_qubits": n, "gates": G, "batch_per_gpu": B, "global_batch": B * world,
            "precision": "complex64" if prec == "c64" else "complex128",
            "parallelism": f"dp{world} (sample-sharded, NCCL all-reduce of the parameter gradient)",
            "l2": "inputs larger than L2: the per-chunk state workspace is GiBs >> 126 MB L2"}


# ------------------------------------------------------------------------------
def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2301_03251_b200 import (QuantumLayer, Tensor, backward, qsim, tsum,
                                       workloads as wl)
    from paper_2301_03251_b200 import templates as T
    from paper_2301_03251_b200 import engine, tracer as tr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if a.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(a.backend)
    cfg = a.config
    n, d, P, B0, prec = wl.CONFIGS[cfg]
    prec = a.precision or prec
    B = a.batch or B0
    builder = wl.make_builder(cfg, qsim, T)
    xall = wl.inputs_for(cfg, B * world)
    x = np.ascontiguousarray(xall[rank * B:(rank + 1) * B])
    theta = wl.params_for(cfg)
    want_x = cfg in ("cfg1", "cfg2")
    tape, ok = tr.trace(builder, x, theta)
    assert ok
    grad = tr.classify(tape, d + P, [want_x] * d + [True] * P, math.pi / 2, 0.5)
    plan = engine.Plan(tape, d, P, prec, grad)
    dev = torch.device(f"cuda:{local}")
    xd = torch.from_numpy(x).to(dev)
    td = torch.from_numpy(theta).to(dev)
    up = torch.ones(B, dtype=torch.float64, device=dev)

    def step():
        out, jac = plan.forward(xd, td, True)
        gx, gt = plan.vjp(jac, up, want_x, True)
        if world > 1:
            dist.all_reduce(gt)
        return out, gt

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    plan.profile(True)
    with Clocks(local) as clk:
        ev0.record()
        for _ in range(a.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile(False)
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / a.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B / (ms / 1e3)
    st = plan.stats(B, True)
    launches_per_step = int(st["launches"]) + 1   # + hq_vjp (θ)
    if want_x:
        launches_per_step += 1

    # roofline: the dominant amplitude-update kernel class, live event time
    peak, peak_kind = peaks()
    b = 8 if prec == "c64" else 16
    S = int(st["n_passes"])
    fwd, bwd = prof["pass_fwd"], prof["pass_bwd"]
    if st["path"] == 1:
        # Dominant kernel class: the backward passes (hq_b*, incl. the fused
        # last-forward+first-backward kernel).  Algorithmic bytes per unit
        # (one sample's forward + full gradient) follow SURVEY.md §8(d), which
        # defines roofline.achieved: 2·2^n·b·(S_f + 2·S_b) with the model's
        # sweep count S = d·ceil(n/q_model) (q_model = 13 c64 / 12 c128); the
        # backward class carries the 2·S_b part (ψ and λ, read + write).  This
        # plan executes fewer sweeps (S below): "executed" reports the bytes of
        # the sweeps actually run, "traffic" the ncu-measured DRAM bytes.
        R, D, _ = wl.gate_counts(cfg)
        depth = 10 if cfg == "cfg4" else 20
        S_model = depth * -(-n // (13 if prec == "c64" else 12))
        name = "hq_b* (backward passes)" if bwd["ms"] >= fwd["ms"] else "hq_f* (forward passes)"
        dom = bwd if bwd["ms"] >= fwd["ms"] else fwd
        units = B * a.steps
        alg = (4 if dom is bwd else 2) * (1 << n) * b * S_model * units
        achieved = alg / (dom["ms"] / 1e3) / 1e9
        alg_exec = (4 if dom is bwd else 2) * (1 << n) * b * S * units
        t_all = (fwd["ms"] + bwd["ms"]) / 1e3
        traffic = None
        try:
            with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
                ref = json.load(f)["hq_b" if dom is bwd else "hq_f"]
            traffic = ref["dram_bytes_per_launch"] / ref["algorithmic_bytes_per_launch"] * (alg_exec / max(dom["launches"], 1))
        except Exception:
            pass
        bytes_unit = 2 * (1 << n) * b * (S_model + 2 * S_model)
        flops_unit = (1 << n) * (18 * R + 8 * D + 6)
        units_per_s = units / t_all
        fpeak, fkind = fp_peak(prec)
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_note": "ncu dram__bytes_read+write per launch (ratio to executed-sweep bytes from "
                                "profiles/ncu_traffic.json, scaled to this launch size)",
                "peak_source": peak_kind,
                "launches": dom["launches"], "avg_launch_ms": dom["ms"] / max(dom["launches"], 1),
                "algorithmic_bytes_per_launch": alg / max(dom["launches"], 1),
                "sweeps_model": S_model, "sweeps_executed": S,
                "executed": {"achieved": alg_exec / (dom["ms"] / 1e3) / 1e9,
                             "frac": alg_exec / (dom["ms"] / 1e3) / 1e9 / peak,
                             "bytes_per_launch": alg_exec / max(dom["launches"], 1)},
                "share_of_step": dom["ms"] / (ms * a.steps),
                "all_passes": {"bytes_per_unit": bytes_unit, "achieved": bytes_unit * units_per_s / 1e9,
                               "frac": bytes_unit * units_per_s / 1e9 / peak},
                "fp32": {"flops_per_unit": flops_unit, "achieved_TFLOPs": flops_unit * units_per_s / 1e12,
                         "peak_TFLOPs": fpeak, "peak_source": fkind,
                         "frac": flops_unit * units_per_s / 1e12 / fpeak if fpeak else None},
                "all_kernels_ms_per_step": {k: v["ms"] / a.steps for k, v in prof.items()}}
    else:
        dom = prof["onchip"]
        R, D, G = wl.gate_counts(cfg)
        flops = (1 << n) * (18 * R + 8 * D + 6) * B * a.steps
        achieved = flops / (dom["ms"] / 1e3) / 1e12
        roof = {"bound": "fp", "kernel": "k_onchip", "achieved": achieved, "unit": "TFLOP/s",
                "peak": None, "frac": None, "traffic": None,
                "note": "state resident in shared memory; launch/latency bound at this batch"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if prec == "c64" else "f64", "data": "synthetic",
            "config": workload_config(cfg, world, B, prec), "roofline": roof,
            "gpu_launches": launches_per_step * a.steps, "clocks": clk.summary(),
            "plan": plan.description}

    # e2e through the public API: host numpy in, host numpy out
    if not a.no_e2e:
        layer = QuantumLayer(builder, n_params=P, param_init=theta, precision=prec)

        def e2e_step():
            xt = Tensor(x, requires_grad=want_x, dtype=np.float64)
            out = layer(xt)
            backward(tsum(out))
            g = layer.params.grad
            if world > 1:
                gd = torch.from_numpy(g).to(dev)
                dist.all_reduce(gd)
                g = gd.cpu().numpy()
            layer.params.zero_grad()
            return g

        for _ in range(max(1, min(a.warmup, 2))):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k = max(2, a.steps // 2)
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0) * 1e3 / k
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        line["e2e"] = {"value": world * B / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
                       "steps": k, "h2d_bytes_per_step": int(x.nbytes + theta.nbytes + B * 8),
                       "d2h_bytes_per_step": int(B * 8 + theta.nbytes + (x.nbytes if want_x else 0)),
                       "api": "QuantumLayer.forward + hyqnet-style backward (host numpy tensors)"}

    # the same workload at the reference's own precision (complex128),
    # device-timed like `value` (companion number; `value` stays the plan's)
    if prec == "c64" and not a.no_c128:
        del plan
        torch.cuda.empty_cache()
        p128 = engine.Plan(tape, d, P, "c128", grad)

        def step128():
            out, jac = p128.forward(xd, td, True)
            gx, gt = p128.vjp(jac, up, want_x, True)
            if world > 1:
                dist.all_reduce(gt)
            return gt

        step128()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k = max(2, min(a.steps, 4))
        ev0.record()
        for _ in range(k):
            step128()
        ev1.record()
        torch.cuda.synchronize()
        t = torch.tensor([ev0.elapsed_time(ev1) / k], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v128 = world * B / (float(t.item()) / 1e3)
        R, D, _ = wl.gate_counts(cfg)
        f_unit = (1 << n) * (18 * R + 8 * D + 6)
        f64peak, f64kind = fp_peak("c128")
        line["complex128"] = {"value": v128, "unit": UNIT,
                              "ms_per_step": float(t.item()), "steps": k, "dtype": "f64",
                              "fp64": {"flops_per_unit": f_unit, "achieved_TFLOPs": f_unit * v128 / world / 1e12,
                                       "peak_TFLOPs": f64peak, "peak_source": f64kind,
                                       "frac": f_unit * v128 / world / 1e12 / f64peak},
                              "note": "same workload, complex128 amplitudes (the reference's precision)",
                              "plan": p128.description}
        del p128
        torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not a.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, x[0], theta)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
