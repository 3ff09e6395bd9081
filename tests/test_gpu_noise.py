"""NOISY machine type on the GPU (hq_noisy) against the reference's golden
counts / NoiseQuantumLayer values and gradients, and the oracle on seeded cases.
Bit-exact: counts are integers drawn from the same per-shot Philox streams."""

import numpy as np
import pytest

from conftest import golden
from oracle import hq_oracle as O
from paper_2301_03251_b200 import (Circuit, NoiseModel, NoiseQuantumLayer, QuantumLayer, Tensor, backward,
                                   simulate_noisy, tsum)
from paper_2301_03251_b200 import noise as N
from paper_2301_03251_b200.qnn import NOISY

pytestmark = pytest.mark.gpu


def _models(g, mod):
    models = {}
    for i, kind, name, p, q in g["specs"]:
        m = models.setdefault(int(i), mod.NoiseModel())
        m.add(str(kind), mod.Channel(str(name), float(p)), None if int(q) < 0 else int(q))
    return models


def _circuits(g):
    out = []
    for k in range(len(g["n_qubits"])):
        c = Circuit(int(g["n_qubits"][k]))
        for i in range(g["starts"][k], g["starts"][k + 1]):
            kind = str(g["kinds"][i]).lower()
            tg = (int(g["q0"][i]),) if g["q1"][i] < 0 else (int(g["q0"][i]), int(g["q1"][i]))
            a = None if np.isnan(g["angle"][i]) else float(g["angle"][i])
            getattr(c, kind)(*tg) if a is None else getattr(c, kind)(*tg, a)
        out.append(c)
    return out


def test_noisy_counts_match_reference_golden():
    g = golden("noise")
    models = _models(g, N)
    for k, c in enumerate(_circuits(g)):
        counts = simulate_noisy(c, models[int(g["model"][k])], int(g["shots"][k]), int(g["seed"][k]))
        want = {str(key): int(v) for key, v in zip(g[f"keys{k}"], g[f"vals{k}"])}
        assert dict(counts) == want, k
        assert counts.shots == int(g["shots"][k])


def _layer_builder(inputs, params):
    c = Circuit(3)
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


def test_noise_layer_matches_reference_golden():
    g = golden("noise")
    m = _models(g, N)[1]
    layer = NoiseQuantumLayer(_layer_builder, 3, m, shots=64, seed=11, param_init=g["layer_theta"])
    x = Tensor(g["layer_x"], requires_grad=True, dtype=np.float64)
    out = layer(x)
    backward(tsum(out * Tensor(g["layer_upstream"].reshape(-1, 1), dtype=np.float64)))
    assert list(out.numpy()[:, 0]) == list(g["layer_out"])
    np.testing.assert_allclose(x.grad, g["layer_grad_x"], atol=1e-14)
    np.testing.assert_allclose(layer.params.grad, g["layer_grad_p"], atol=1e-13)


@pytest.mark.parametrize("n", [2, 5, 9, 13, 14, 16])
def test_noisy_random_models_vs_oracle(n):
    _random_models_vs_oracle(n)


@pytest.mark.parametrize("n", [14, 15])
def test_noisy_global_state_kernels_vs_oracle(n, monkeypatch):
    """n > 13 with few trajectories runs a CTA cluster per trajectory; the
    CTA-per-trajectory kernel (many trajectories) is forced here."""
    monkeypatch.setenv("HQ_NOISY_NO_CLUSTER", "1")
    _random_models_vs_oracle(n)


def _random_models_vs_oracle(n):
    rng = np.random.default_rng(n)
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
    chans = ["bit_flip", "phase_flip", "depolarizing", "amplitude_damping"]
    for trial in range(3):
        c, oc = Circuit(n), O.Circuit(n)
        for _ in range(25):
            k = kinds[rng.integers(len(kinds))]
            two = k in ("CNOT", "CZ", "CR", "SWAP")
            if two and n < 2:
                continue
            tg = tuple(int(q) for q in rng.choice(n, 2 if two else 1, replace=False))
            a = float(rng.uniform(-3, 3)) if k in ("RX", "RY", "RZ", "CR") else None
            getattr(c, k.lower())(*tg) if a is None else getattr(c, k.lower())(*tg, a)
            oc.add(O.Op(k, tg, a))
        # up to 6 measured qubits: both marginal paths (≤ 16 outcomes, > 16)
        meas = [int(q) for q in rng.choice(n, min(n, 2 + 2 * trial), replace=False)]
        c.measure(*meas)
        oc.measure(*meas)
        m, om = N.NoiseModel(), O.NoiseModel()
        for _ in range(5):
            k = kinds[rng.integers(len(kinds))]
            ch = chans[rng.integers(4)]
            p = float(rng.choice([0.0, rng.uniform(0, 1), 1.0]))
            q = None if rng.random() < 0.7 else int(rng.integers(n))
            m.add(k, N.Channel(ch, p), q)
            om.add(k, O.Channel(ch, p), q)
        shots, seed = int(rng.integers(20, 120)), int(rng.integers(0, 10**6))
        assert dict(simulate_noisy(c, m, shots, seed)) == O.simulate_noisy(oc, om, shots, seed)


def test_noisy_layer_batched_vs_oracle_and_trivial_model():
    rng = np.random.default_rng(8)
    x = rng.uniform(-2, 2, (5, 2))
    th = rng.uniform(0, 6, 3)
    m = N.NoiseModel().add("CNOT", N.depolarizing(0.3)).add("RY", N.amplitude_damping(0.4)) \
        .add("H", N.bit_flip(0.2), 2)
    om = O.NoiseModel().add("CNOT", O.Channel("depolarizing", 0.3)) \
        .add("RY", O.Channel("amplitude_damping", 0.4)).add("H", O.Channel("bit_flip", 0.2), 2)
    layer = QuantumLayer(_layer_builder, 3, machine_type=NOISY, noise_model=m, shots=80, seed=3, param_init=th)
    xt = Tensor(x, requires_grad=True, dtype=np.float64)
    out = layer(xt)
    backward(tsum(out))
    o, jx, jp = O.noisy_layer(_layer_builder_o, x, th, om, 80, 3)
    assert list(out.numpy()[:, 0]) == list(o)
    np.testing.assert_allclose(xt.grad, jx, atol=1e-14)
    np.testing.assert_allclose(layer.params.grad, jp.sum(0), atol=1e-13)
    # an all-zero model reproduces noiseless SHOT_SAMPLING counts (noise.py:1-6)
    zero = N.NoiseModel().add("CNOT", N.bit_flip(0.0))
    c = _layer_builder(list(x[0]), list(th))
    from paper_2301_03251_b200 import measure_shots, simulate
    want = measure_shots(simulate(c), list(c.measured_qubits), 200, 9)
    assert dict(simulate_noisy(c, zero, 200, 9)) == dict(want)


def _layer_builder_o(inputs, params):
    return _layer_builder.__wrapped__(inputs, params) if hasattr(_layer_builder, "__wrapped__") else \
        _to_oracle(_layer_builder(inputs, params))


def _to_oracle(c):
    oc = O.Circuit(c.n_qubits)
    for op in c.ops:
        oc.add(O.Op(op.kind, tuple(op.targets), op.angle))
    oc.measure(*c.measured_qubits)
    return oc


def test_host_level_trajectory_helpers_match_oracle():
    """apply_channel / run_trajectory (noise.py:93-138) with a caller's NumPy
    generator: the same draws as the oracle's restatement, the same final
    states (gates on the GPU, damping jumps on the host copy)."""
    g = golden("noise")
    circuits = _circuits(g)
    ours, theirs = _models(g, N), _models(g, O)
    for k, c in enumerate(circuits):
        mi = int(g["model"][k])
        oc = O.Circuit(c.n_qubits)
        for op in c.ops:
            oc.add(O.Op(op.kind, op.targets, op.angle))
        for seed in (0, 7):
            st = N.run_trajectory(c, ours[mi], np.random.default_rng(seed))
            want = O.run_trajectory(oc, theirs[mi], np.random.default_rng(seed))
            np.testing.assert_allclose(st.amplitudes, want, atol=1e-12)
    # a single channel application on a prepared state
    c = Circuit(2)
    c.h(0); c.cnot(0, 1)
    from paper_2301_03251_b200 import simulate
    st = simulate(c)
    N.apply_channel(st, 1, N.amplitude_damping(0.4), np.random.default_rng(3))
    psi = O.simulate(O.Circuit(2, ops=[O.Op("H", (0,)), O.Op("CNOT", (0, 1))]))
    O.apply_channel(psi, 2, 1, O.Channel("amplitude_damping", 0.4), np.random.default_rng(3))
    np.testing.assert_allclose(st.amplitudes, psi, atol=1e-12)
