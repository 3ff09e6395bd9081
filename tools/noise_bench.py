"""NOISY machine type throughput: NoiseQuantumLayer forward + shift-rule
gradient (inputs and params) on the cfg1 / cfg2 circuits, device-timed; the
oracle port's time for one sample's forward on one core for comparison."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_03251_b200 import engine, qsim, workloads as wl, templates as T
from paper_2301_03251_b200 import noise as N
from oracle import hq_oracle as O


def model(mod, ch):
    return mod.NoiseModel().add("CNOT", ch("depolarizing", 0.02)).add("RY", ch("amplitude_damping", 0.03)) \
        .add("RX", ch("bit_flip", 0.01)).add("RZ", ch("phase_flip", 0.01))


def run(cfg, B, shots, steps=3, grads=True, oracle_shots=None):
    n, d, P, _, _ = wl.CONFIGS[cfg]
    b = wl.make_builder(cfg, qsim, T)
    x = wl.inputs_for(cfg, B); th = wl.params_for(cfg)
    m = model(N, N.Channel)
    engine.run_batch_noisy(b, x, th, grads, grads, m, shots, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        e, jac = engine.run_batch_noisy(b, x, th, grads, grads, m, shots, 0)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    rows = (1 + 2 * (d + P)) if grads else 1
    traj = B * rows * shots
    # oracle: one forward evaluation of one sample on one core
    ob = wl.make_builder(cfg, O, O)
    om = model(O, O.Channel)
    osh = oracle_shots or shots
    t1 = time.perf_counter()
    O.noisy_expectation(ob([float(v) for v in x[0]], [float(v) for v in th]), om, osh, 0)
    one = (time.perf_counter() - t1) * shots / osh
    cpu_samples_per_s = 1.0 / (one * rows)
    return {"config": cfg, "n_qubits": n, "batch": B, "shots": shots, "gradients": grads,
            "ms_per_step": dt * 1e3,
            "samples_per_s": B / dt, "trajectories_per_s": traj / dt,
            "oracle_1core_samples_per_s": cpu_samples_per_s, "speedup_vs_1core_port": B / dt / cpu_samples_per_s}


if __name__ == "__main__":
    for cfg, B, shots in (("cfg1", 64, 100), ("cfg2", 64, 100)):
        print(json.dumps(run(cfg, B, shots)), flush=True)
    # global-memory trajectory kernel (n > 13): forward values only
    print(json.dumps(run("cfg3", 16, 20, grads=False)), flush=True)
    print(json.dumps(run("cfg4", 4, 10, steps=1, grads=False, oracle_shots=1)), flush=True)
