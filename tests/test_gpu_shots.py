"""SHOT_SAMPLING on the device vs the reference's own shot streams (golden
vectors from hyqnet's measure_shots / QuantumLayer), bit-exact."""

import numpy as np
import pytest

from conftest import golden
from oracle import hq_oracle as O
from paper_2301_03251_b200 import (Circuit, QAELayer, QuantumLayer, StateVector, Tensor, backward,
                                   measure_shots, qsim, simulate, tsum)
from paper_2301_03251_b200 import engine

pytestmark = pytest.mark.gpu


def test_device_philox_stream_matches_numpy():
    for seed in (0, 5, 12345):
        u = engine.shot_uniforms(seed, 0, 300).cpu().numpy()
        want = [np.random.Generator(np.random.Philox(key=[seed, s])).random() for s in range(300)]
        np.testing.assert_array_equal(u, want)


def _circuits(g):
    out = []
    for k in range(len(g["n_qubits"])):
        c = Circuit(int(g["n_qubits"][k]))
        for i in range(g["starts"][k], g["starts"][k + 1]):
            tg = (int(g["q0"][i]),) if g["q1"][i] < 0 else (int(g["q0"][i]), int(g["q1"][i]))
            a = None if np.isnan(g["angle"][i]) else float(g["angle"][i])
            c.add(qsim.GateOp(str(g["kinds"][i]), tg, a))
        out.append(c)
    return out


def test_measure_shots_counts_match_reference():
    g = golden("shots")
    for k, c in enumerate(_circuits(g)):
        counts = measure_shots(simulate(c), list(range(c.n_qubits)), int(g["shots"][k]), int(g["seed"][k]))
        want = {str(key): int(v) for key, v in zip(g[f"keys{k}"], g[f"vals{k}"])}
        assert dict(counts) == want and counts.shots == int(g["shots"][k])


def h_ry(inputs, params):
    c = Circuit(1)
    c.h(0)
    c.ry(0, inputs[0])
    c.measure(0)
    return c


def test_shot_layer_values_and_gradients_match_reference():
    g = golden("shots")
    layer = QuantumLayer(h_ry, 0, machine_type="shot_sampling", shots=137, seed=5)
    x = Tensor(g["layer_theta"].reshape(-1, 1), requires_grad=True, dtype=np.float64)
    out = layer(x)
    backward(tsum(out))
    np.testing.assert_array_equal(out.numpy()[:, 0], g["layer_out"])
    np.testing.assert_array_equal(x.grad[:, 0], g["layer_grad"])


def test_shot_layer_deterministic_and_near_exact():
    a = QuantumLayer(h_ry, 0, machine_type="shot_sampling", shots=4000, seed=3)
    x = Tensor(np.array([[0.9]]), dtype=np.float64)
    v1, v2 = a(x).item(), a(x).item()
    assert v1 == v2
    assert abs(v1 - (1 + np.sin(0.9)) / 2) < 4 * np.sqrt(0.25 / 4000)


def test_qae_shot_mode_matches_oracle():
    layer = QAELayer(1, 4, machine_type="shot_sampling", shots=200, seed=2,
                     param_init=np.linspace(0.1, 1.1, 18))
    x = np.array([[0.6, 0.8, 0.0, 0.0], [0.0, 1.0, 0.0, 0.0]])
    out = layer(Tensor(x, dtype=np.float64)).numpy()[:, 0]
    b = O.qae_builder(1, 4)
    want = []
    for row in x:
        c = b(list(row), list(np.linspace(0.1, 1.1, 18)))
        counts = O.measure_shots(O.simulate(c), 4, [0], 200, 2)
        want.append(counts.get("0", 0) / 200)
    np.testing.assert_array_equal(out, want)
