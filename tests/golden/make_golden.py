"""Generate golden vectors by running the REFERENCE implementation (hyqnet).

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``hyqnet`` from /root/reference/pkg/src, drives it through its own
public API (``QuantumLayer``, ``backward``, ``simulate``, ``QAELayer``) with the
same builders the product and oracle use (``workloads.make_builder``), and
writes ``tests/golden/*.npz``.  Nothing else in the repo reads /root/reference.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import hyqnet.qsim as rq  # noqa: E402
import hyqnet.templates as rt  # noqa: E402
from hyqnet.qnn import QAELayer, QuantumLayer  # noqa: E402
from hyqnet.tensor import Tensor, backward, tsum  # noqa: E402

from paper_2301_03251_b200 import workloads as wl  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({', '.join(arrays)})")


def layer_case(name, cfg, batch, want_x, seed_g=7):
    builder = wl.make_builder(cfg, rq, rt)
    x = wl.inputs_for(cfg, batch)
    theta = wl.params_for(cfg)
    layer = QuantumLayer(builder, n_params=theta.size, param_init=theta)
    xt = Tensor(x, requires_grad=want_x, dtype=np.float64)
    g = np.random.default_rng(seed_g).uniform(0.5, 1.5, (batch, 1))
    t0 = time.perf_counter()
    out = layer(xt)
    backward(tsum(out * Tensor(g, dtype=np.float64)))
    dt = time.perf_counter() - t0
    save(name, x=x, theta=theta, upstream=g[:, 0], out=out.numpy()[:, 0],
         grad_x=xt.grad if want_x else np.zeros_like(x), grad_p=layer.params.grad,
         seconds=np.array(dt))


def _cfg4_eval(args):
    # one reference circuit evaluation (QuantumLayer._run, qnn.py:120-121)
    xi, th = args
    builder = wl.make_builder("cfg4", rq, rt)
    layer = QuantumLayer(builder, n_params=th.size, param_init=th)
    return layer._run(xi, th)


def cfg4_case():
    """cfg4 (the bench config) pinned per SURVEY.md §8(c) and beyond: 4
    samples' forward, the FULL 400-entry shift-rule gradient row of sample 0,
    32 random rows entries of sample 1, and the layer's df_p for a random
    upstream over samples {0, 1} at those 32 indices (parameter_shift_grad,
    qnn.py:35-52, summed in sample order, qnn.py:147-152).  Evaluations run in
    a process pool; each is the reference's own QuantumLayer._run."""
    from concurrent.futures import ProcessPoolExecutor
    builder = wl.make_builder("cfg4", rq, rt)
    x = wl.inputs_for("cfg4", 4)
    theta = wl.params_for("cfg4")
    layer = QuantumLayer(builder, n_params=theta.size, param_init=theta)
    s, scale = layer.shift, layer.grad_scale
    rng = np.random.default_rng(404)
    idx1 = np.sort(rng.choice(theta.size, 32, replace=False))
    g = rng.uniform(0.5, 1.5, 2)
    jobs = [(x[i], theta) for i in range(4)]
    rows = [(0, j) for j in range(theta.size)] + [(1, int(j)) for j in idx1]
    for i, j in rows:
        tp = theta.copy(); tp[j] += s
        tm = theta.copy(); tm[j] -= s
        jobs += [(x[i], tp), (x[i], tm)]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(os.cpu_count()) as ex:
        vals = list(ex.map(_cfg4_eval, jobs, chunksize=4))
    dt = time.perf_counter() - t0
    out = np.array(vals[:4])
    ev = np.array(vals[4:]).reshape(-1, 2)
    jac0 = (ev[:theta.size, 0] - ev[:theta.size, 1]) * scale
    jac1 = (ev[theta.size:, 0] - ev[theta.size:, 1]) * scale
    # df_p at upstream g over samples 0, 1 (reference operation order)
    grad_p = np.zeros(idx1.size)
    grad_p += (ev[idx1, 0] - ev[idx1, 1]) * scale * float(g[0])
    grad_p += (ev[theta.size:, 0] - ev[theta.size:, 1]) * scale * float(g[1])
    save("cfg4", x=x, theta=theta, out=out, jac_idx=np.arange(theta.size), jac0=jac0,
         jac1_idx=idx1, jac1=jac1, upstream=g, grad_p_idx=idx1, grad_p=grad_p,
         evaluations=np.array(len(jobs)), seconds=np.array(dt))


def random_circuits_case():
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_circuit
    rng = np.random.default_rng(1234)
    kinds, q0, q1, ang, starts, nq, states, exps = [], [], [], [], [0], [], [], []
    for k in range(40):
        n = int(rng.integers(1, 6))
        c = random_circuit(rng, n, int(rng.integers(0, 24)))
        for op in c.ops:
            kinds.append(op.kind)
            q0.append(op.targets[0])
            q1.append(op.targets[1] if len(op.targets) > 1 else -1)
            ang.append(np.nan if op.angle is None else op.angle)
        starts.append(len(kinds))
        nq.append(n)
        st = rq.simulate(c).amplitudes
        states.append(np.pad(st, (0, 32 - st.size)))
        probs = rq.probabilities(rq.simulate(c), list(range(n)))
        exps.append(float(np.arange(probs.size) @ probs))
    save("random_circuits", kinds=np.array(kinds), q0=np.array(q0), q1=np.array(q1),
         angle=np.array(ang), starts=np.array(starts), n_qubits=np.array(nq),
         states=np.array(states), expectation=np.array(exps))


def reupload_case():
    # not shift-exact: input used twice, shared parameter, scaled parameter
    def builder(inputs, params):
        c = rq.Circuit(3)
        c.ry(0, inputs[0])
        c.rx(1, inputs[1])
        c.cnot(0, 1)
        c.ry(0, inputs[0])            # re-upload
        c.rz(1, params[0])
        c.rx(2, params[0])            # shared
        c.ry(2, 2.0 * params[1])      # scaled
        c.cr(1, 2, params[2] - 0.3)   # CR, affine
        c.h(2)
        c.cz(0, 2)
        c.swap(0, 2)
        c.ry(1, 0.5 * params[3] + inputs[1])
        c.measure(0, 2)
        return c
    rng = np.random.default_rng(3)
    x = rng.uniform(-np.pi, np.pi, (5, 2))
    theta = rng.uniform(0, 2 * np.pi, 4)
    layer = QuantumLayer(builder, n_params=4, param_init=theta)
    xt = Tensor(x, requires_grad=True, dtype=np.float64)
    g = rng.uniform(0.5, 1.5, (5, 1))
    out = layer(xt)
    backward(tsum(out * Tensor(g, dtype=np.float64)))
    save("reupload", x=x, theta=theta, upstream=g[:, 0], out=out.numpy()[:, 0], grad_x=xt.grad,
         grad_p=layer.params.grad)


def qae_cases():
    layer = QAELayer(1, 4, machine_type="exact_prob", param_init=np.linspace(0.1, 1.1, 18))
    x = np.array([[0.6, 0.8, 0.0, 0.0]])
    out = layer(Tensor(x, dtype=np.float64))
    backward(tsum(out))
    save("qae_1_4", x=x, theta=np.linspace(0.1, 1.1, 18), out=out.numpy()[:, 0],
         grad_p=layer.params.grad)
    rng = np.random.default_rng(1234)
    theta = rng.uniform(0, 2 * np.pi, 60)
    layer = QAELayer(2, 7, machine_type="exact_prob", param_init=theta)
    x = rng.standard_normal((3, 16))
    g = rng.uniform(0.5, 1.5, (3, 1))
    out = layer(Tensor(x, dtype=np.float64))
    backward(tsum(out * Tensor(g, dtype=np.float64)))
    save("qae_2_7", x=x, theta=theta, upstream=g[:, 0], out=out.numpy()[:, 0],
         grad_p=layer.params.grad)


def shots_case():
    # measure_shots counts (qsim.py:236-248) and SHOT_SAMPLING layer outputs
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_circuit
    rng = np.random.default_rng(99)
    kinds, q0, q1, ang, starts, nq, shots, seeds = [], [], [], [], [0], [], [], []
    extra = {}
    for k in range(6):
        n = int(rng.integers(1, 5))
        c = random_circuit(rng, n, int(rng.integers(1, 12)))
        for op in c.ops:
            kinds.append(op.kind)
            q0.append(op.targets[0])
            q1.append(op.targets[1] if len(op.targets) > 1 else -1)
            ang.append(np.nan if op.angle is None else op.angle)
        starts.append(len(kinds))
        nq.append(n)
        S, seed = int(rng.integers(50, 400)), int(rng.integers(0, 1000))
        shots.append(S)
        seeds.append(seed)
        counts = rq.measure_shots(rq.simulate(c), list(range(n)), S, seed)
        extra[f"keys{k}"] = np.array(list(counts.keys()))
        extra[f"vals{k}"] = np.array(list(counts.values()))

    def h_ry(inputs, params):
        c = rq.Circuit(1)
        c.h(0)
        c.ry(0, inputs[0])
        c.measure(0)
        return c
    th = np.linspace(-2, 2, 7)
    layer = QuantumLayer(h_ry, 0, machine_type="shot_sampling", shots=137, seed=5)
    x = Tensor(th.reshape(-1, 1), requires_grad=True, dtype=np.float64)
    out = layer(x)
    backward(tsum(out))
    save("shots", kinds=np.array(kinds), q0=np.array(q0), q1=np.array(q1), angle=np.array(ang),
         starts=np.array(starts), n_qubits=np.array(nq), shots=np.array(shots), seed=np.array(seeds),
         layer_theta=th, layer_out=out.numpy()[:, 0], layer_grad=x.grad[:, 0], **extra)


def embedding_case():
    rng = np.random.default_rng(5)
    vecs = [np.array([0.2, -0.4, 0.4, -0.8]), np.array([3, 1, -4, 1, -5, 9, -2, 6], float),
            np.array([0.6, 0.8]), rng.standard_normal(16), rng.standard_normal(5),
            np.array([0.0, 0.0, 1.0, 0.0])]
    out = []
    for v in vecs:
        n = max(1, int(np.ceil(np.log2(v.size))))
        c = rq.Circuit(n + 1)
        c.extend(rt.amplitude_embedding(v, qubits=list(range(1, n + 1))))
        out.append(np.pad(rq.simulate(c).amplitudes, (0, 32 - 2 ** (n + 1))))
    save("embedding", vecs=np.array([np.pad(v, (0, 16 - v.size)) for v in vecs]),
         sizes=np.array([v.size for v in vecs]), states=np.array(out))


def noise_cases():
    # simulate_noisy counts (noise.py:141-153) and NoiseQuantumLayer values /
    # shift-rule gradients (qnn.py:157-166) for mixed channel models
    import hyqnet.noise as rn
    from hyqnet.qnn import NoiseQuantumLayer
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_circuit
    rng = np.random.default_rng(2024)
    models = []

    def model(spec):
        m = rn.NoiseModel()
        for kind, name, p, q in spec:
            m.add(kind, rn.Channel(name, p), q)
        return m
    specs = [
        [("H", "bit_flip", 0.2, None), ("CNOT", "phase_flip", 0.3, None), ("RY", "depolarizing", 0.4, None)],
        [("RX", "amplitude_damping", 0.35, None), ("RY", "amplitude_damping", 0.5, None),
         ("CNOT", "depolarizing", 0.25, None), ("X", "bit_flip", 0.0, None)],
        [("RZ", "phase_flip", 0.15, None), ("H", "depolarizing", 1.0, None), ("CZ", "bit_flip", 0.4, 0),
         ("CZ", "amplitude_damping", 0.6, None), ("SWAP", "bit_flip", 0.1, None)],
        [("RY", "depolarizing", 0.3, 1), ("RY", "bit_flip", 0.05, None), ("CR", "amplitude_damping", 0.2, None),
         ("Y", "phase_flip", 0.5, None), ("Z", "depolarizing", 0.6, None), ("RX", "bit_flip", 0.3, None)],
    ]
    kinds, q0, q1, ang, starts, nq, shots, seeds, midx = [], [], [], [], [0], [], [], [], []
    extra = {}
    k = 0
    for trial in range(8):
        n = int(rng.integers(1, 6))
        c = random_circuit(rng, n, int(rng.integers(3, 20)))
        for op in c.ops:
            kinds.append(op.kind)
            q0.append(op.targets[0])
            q1.append(op.targets[1] if len(op.targets) > 1 else -1)
            ang.append(np.nan if op.angle is None else op.angle)
        starts.append(len(kinds))
        nq.append(n)
        S, seed = int(rng.integers(50, 300)), int(rng.integers(0, 1000))
        mi = trial % len(specs)
        shots.append(S); seeds.append(seed); midx.append(mi)
        counts = rn.simulate_noisy(c, model(specs[mi]), S, seed)
        extra[f"keys{trial}"] = np.array(list(counts.keys()))
        extra[f"vals{trial}"] = np.array(list(counts.values()))
    spec_arr = np.array([(i, kd, nm, p, -1 if q is None else q) for i, sp in enumerate(specs)
                         for kd, nm, p, q in sp], dtype=object)

    def builder(inputs, params):
        c = rq.Circuit(3)
        c.ry(0, inputs[0])
        c.rx(1, inputs[1])
        c.h(2)
        c.cnot(0, 1)
        c.ry(1, params[0])
        c.rz(2, params[1])
        c.cnot(1, 2)
        c.rx(0, params[2])
        c.measure(0, 2)
        return c
    x = rng.uniform(-2, 2, (3, 2))
    theta = rng.uniform(0, 6, 3)
    lay = NoiseQuantumLayer(builder, 3, model(specs[1]), shots=64, seed=11, param_init=theta)
    xt = Tensor(x, requires_grad=True, dtype=np.float64)
    g = rng.uniform(0.5, 1.5, (3, 1))
    out = lay(xt)
    backward(tsum(out * Tensor(g, dtype=np.float64)))
    save("noise", kinds=np.array(kinds), q0=np.array(q0), q1=np.array(q1), angle=np.array(ang),
         starts=np.array(starts), n_qubits=np.array(nq), shots=np.array(shots), seed=np.array(seeds),
         model=np.array(midx), specs=spec_arr.astype(str), layer_x=x, layer_theta=theta,
         layer_upstream=g[:, 0], layer_out=out.numpy()[:, 0], layer_grad_x=xt.grad,
         layer_grad_p=lay.params.grad, **extra)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "random", "reupload", "qae", "embed", "shots",
                             "noise"]
    if "cfg1" in which:
        layer_case("cfg1", "cfg1", 16, True)
    if "cfg2" in which:
        layer_case("cfg2", "cfg2", 16, True)
    if "cfg3" in which:
        layer_case("cfg3", "cfg3", 4, False)
    if "cfg4" in which:
        cfg4_case()
    if "random" in which:
        random_circuits_case()
    if "reupload" in which:
        reupload_case()
    if "qae" in which:
        qae_cases()
    if "embed" in which:
        embedding_case()
    if "shots" in which:
        shots_case()
    if "noise" in which:
        noise_cases()
