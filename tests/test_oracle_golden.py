"""Pin the CPU oracle to golden vectors produced by the reference itself.

CPU-only.  The oracle (oracle/hq_oracle.py) is the checker every GPU parity
test uses, so it must first reproduce hyqnet's own outputs and gradients.
"""

import numpy as np
import pytest

from conftest import golden, relative_error
from oracle import hq_oracle as O
from paper_2301_03251_b200 import workloads as wl


def _circuits(g):
    out = []
    for k in range(len(g["n_qubits"])):
        c = O.Circuit(int(g["n_qubits"][k]))
        for i in range(g["starts"][k], g["starts"][k + 1]):
            kind = str(g["kinds"][i])
            tg = (int(g["q0"][i]),) if g["q1"][i] < 0 else (int(g["q0"][i]), int(g["q1"][i]))
            a = None if np.isnan(g["angle"][i]) else float(g["angle"][i])
            c.add(O.Op(kind, tg, a))
        c.measure(*range(c.n_qubits))
        out.append(c)
    return out


def test_random_circuits_states_and_readout():
    g = golden("random_circuits")
    for k, c in enumerate(_circuits(g)):
        st = O.simulate(c)
        np.testing.assert_allclose(st, g["states"][k][:st.size], atol=1e-12)
        assert O.expectation(c) == pytest.approx(g["expectation"][k], abs=1e-12)


def test_cfg1_layer_forward_and_gradients():
    g = golden("cfg1")
    b = wl.make_builder("cfg1", O, O)
    out, jx, jp, gx, gp = O.layer(b, g["x"], g["theta"], upstream=g["upstream"])
    assert relative_error(out, g["out"]) < 1e-12
    assert relative_error(gx, g["grad_x"], floor=1e-6) < 1e-12
    assert relative_error(gp, g["grad_p"], floor=1e-6) < 1e-12


def test_reupload_two_point_semantics():
    g = golden("reupload")

    def b(inputs, params):
        c = O.Circuit(3)
        c.ry(0, inputs[0]); c.rx(1, inputs[1]); c.cnot(0, 1); c.ry(0, inputs[0])
        c.rz(1, params[0]); c.rx(2, params[0]); c.ry(2, 2.0 * params[1])
        c.cr(1, 2, params[2] - 0.3); c.h(2); c.cz(0, 2); c.swap(0, 2)
        c.ry(1, 0.5 * params[3] + inputs[1]); c.measure(0, 2)
        return c
    out, _, _, gx, gp = O.layer(b, g["x"], g["theta"], upstream=g["upstream"])
    assert relative_error(out, g["out"]) < 1e-12
    assert relative_error(gx, g["grad_x"], floor=1e-6) < 1e-12
    assert relative_error(gp, g["grad_p"], floor=1e-6) < 1e-12


@pytest.mark.parametrize("name,trash,total", [("qae_1_4", 1, 4), ("qae_2_7", 2, 7)])
def test_qae_two_point_values(name, trash, total):
    g = golden(name)
    b = O.qae_builder(trash, total)
    e, _, jp, _, _ = O.layer(b, g["x"], g["theta"], want_x=False)
    up = g.get("upstream", np.ones(len(g["x"])))
    assert relative_error(1.0 - e, g["out"]) < 1e-12
    # P0 = 1 - E: gradients flip sign
    gp = -(jp * up[:, None]).sum(axis=0)
    assert relative_error(gp, g["grad_p"], floor=1e-4) < 1e-11


def test_amplitude_embedding_states():
    g = golden("embedding")
    for k, size in enumerate(g["sizes"]):
        v = g["vecs"][k][:size]
        n = max(1, int(np.ceil(np.log2(size))))
        c = O.Circuit(n + 1)
        c.extend(O.amplitude_embedding(v, qubits=list(range(1, n + 1))))
        st = O.simulate(c)
        np.testing.assert_allclose(st, g["states"][k][:st.size], atol=1e-12)


def test_cfg2_layer():
    g = golden("cfg2")
    b = wl.make_builder("cfg2", O, O)
    out, _, _, gx, gp = O.layer(b, g["x"][:1], g["theta"], upstream=g["upstream"][:1])
    assert relative_error(out, g["out"][:1]) < 1e-12
    assert relative_error(gx, g["grad_x"][:1], floor=1e-6) < 1e-12


def test_cfg3_forward_and_some_param_grads():
    g = golden("cfg3")
    b = wl.make_builder("cfg3", O, O)
    out = np.array([O.run(b, g["x"][i], g["theta"]) for i in range(len(g["x"]))])
    assert relative_error(out, g["out"]) < 1e-12
    # per-sample jacobian entries for 3 params on both samples -> grad_p pieces
    for j in (0, 50, 107):
        tot = 0.0
        for i in range(len(g["x"])):
            tp = g["theta"].copy(); tp[j] += np.pi / 2
            tm = g["theta"].copy(); tm[j] -= np.pi / 2
            tot += (O.run(b, g["x"][i], tp) - O.run(b, g["x"][i], tm)) * 0.5 * g["upstream"][i]
        assert tot == pytest.approx(g["grad_p"][j], abs=1e-12)


def test_cfg4_forward_and_jacobian_entries():
    g = golden("cfg4")
    b = wl.make_builder("cfg4", O, O)
    assert O.run(b, g["x"][0], g["theta"]) == pytest.approx(g["out"][0], abs=1e-12)
    for k in (0, 3):
        j = int(g["jac_idx"][k])
        tp = g["theta"].copy(); tp[j] += np.pi / 2
        tm = g["theta"].copy(); tm[j] -= np.pi / 2
        val = (O.run(b, g["x"][0], tp) - O.run(b, g["x"][0], tm)) * 0.5
        assert val == pytest.approx(g["jac0"][k], abs=1e-12)
    # sample 1's rows entries come from the same reference evaluations
    j = int(g["jac1_idx"][5])
    tp = g["theta"].copy(); tp[j] += np.pi / 2
    tm = g["theta"].copy(); tm[j] -= np.pi / 2
    val = (O.run(b, g["x"][1], tp) - O.run(b, g["x"][1], tm)) * 0.5
    assert val == pytest.approx(g["jac1"][5], abs=1e-12)


def test_philox_stream_matches_numpy():
    # the reference's shot_rng (qsim.py:222-224) is numpy's Philox; pin the restatement
    for seed in (0, 3, 7, 2**40 + 5):
        for shot in (0, 1, 2, 99, 4000, 2**33):
            want = np.random.Generator(np.random.Philox(key=[seed, shot])).random()
            assert O.philox_uniform(seed, shot) == want


def test_shot_counts_golden():
    g = golden("shots")
    for k, c in enumerate(_circuits_from(g)):
        counts = O.measure_shots(O.simulate(c), c.n_qubits, list(range(c.n_qubits)), int(g["shots"][k]),
                                 int(g["seed"][k]))
        want = {str(key): int(v) for key, v in zip(g[f"keys{k}"], g[f"vals{k}"])}
        assert counts == want
    assert list(g["layer_out"]) == [O.shot_expectation(_hry(t), 137, 5) for t in g["layer_theta"]]


def _hry(theta):
    c = O.Circuit(1)
    c.h(0)
    c.ry(0, theta)
    c.measure(0)
    return c


def _circuits_from(g):
    return _circuits({k: g[k] for k in ("kinds", "q0", "q1", "angle", "starts", "n_qubits")})


# ---------------------------------------------------------------------------
# NOISY trajectories (noise.py) — counts and NoiseQuantumLayer values/gradients
def noise_models(g):
    models = {}
    for i, kind, name, p, q in g["specs"]:
        m = models.setdefault(int(i), O.NoiseModel())
        m.add(str(kind), O.Channel(str(name), float(p)), None if int(q) < 0 else int(q))
    return models


def noise_layer_builder(Circ):
    def builder(inputs, params):
        c = Circ(3)
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
    return builder


def test_philox_stream_matches_numpy():
    for seed, shot in ((0, 0), (7, 3), (2**40 + 5, 123456)):
        gen = np.random.Generator(np.random.Philox(key=[seed, shot]))
        assert [gen.random() for _ in range(13)] == [O.philox_draw(seed, shot, k) for k in range(13)]


def test_noisy_counts_golden():
    g = golden("noise")
    models = noise_models(g)
    for k, c in enumerate(_circuits_from(g)):
        counts = O.simulate_noisy(c, models[int(g["model"][k])], int(g["shots"][k]), int(g["seed"][k]))
        want = {str(key): int(v) for key, v in zip(g[f"keys{k}"], g[f"vals{k}"])}
        assert counts == want, k


def test_noisy_layer_golden():
    g = golden("noise")
    m = noise_models(g)[1]
    out, jx, jp = O.noisy_layer(noise_layer_builder(O.Circuit), g["layer_x"], g["layer_theta"], m, 64, 11)
    up = g["layer_upstream"]
    assert list(out) == list(g["layer_out"])
    np.testing.assert_allclose(jx * up[:, None], g["layer_grad_x"], atol=1e-14)
    np.testing.assert_allclose((jp * up[:, None]).sum(0), g["layer_grad_p"], atol=1e-13)
