"""The reference's own hot-path assertions, run against the drop-in through a
``hyqnet`` module alias (``import hyqnet.qsim`` etc. resolve to this package).

Restated from the reference test suite (the reference tree is not on the GPU
box, so the assertions are re-expressed here with an independent dense-matrix
oracle built by basis-state bit logic): ``pkg/tests/test_qsim.py:85-196``
(gate kernels vs dense matrices, endianness, conventions, simulate,
probabilities), ``test_qnn.py:29-266`` (shift-rule known answers, layer closed
forms, batch independence, dtype, errors, shots, QAE), ``test_templates.py:
68-161`` (amplitude embedding, composite gates) and ``test_acceptance.py:
108-128`` (200 random circuits gate by gate with the norm checked after every
gate; the H-RY closed forms at 50 angles).  Test infrastructure only.
"""

import sys
import types

import numpy as np
import pytest

import importlib

import paper_2301_03251_b200 as _pkg

_mods = {name: importlib.import_module(f"paper_2301_03251_b200.{name}")
         for name in ("qsim", "qnn", "templates", "tensor", "errors", "noise")}

pytestmark = pytest.mark.gpu


def _install_alias():
    if "hyqnet" in sys.modules and getattr(sys.modules["hyqnet"], "__drop_in__", False):
        return
    root = types.ModuleType("hyqnet")
    root.__dict__.update({k: getattr(_pkg, k) for k in dir(_pkg) if not k.startswith("_")})
    root.__drop_in__ = True
    root.__path__ = []
    sys.modules["hyqnet"] = root
    for name, mod in _mods.items():
        sys.modules[f"hyqnet.{name}"] = mod
        setattr(root, name, mod)


_install_alias()
from hyqnet.errors import CircuitError, ConfigError, EncodingError  # noqa: E402
from hyqnet.noise import NoiseModel, bit_flip  # noqa: E402
from hyqnet.qnn import (EXACT_PROB, SHOT_SAMPLING, NoiseQuantumLayer, QAELayer, QuantumLayer,  # noqa: E402
                        parameter_shift_grad)
from hyqnet.qsim import Circuit, GateOp, StateVector, apply_gate, gate_matrix, probabilities, simulate  # noqa: E402
from hyqnet.templates import amplitude_embedding, ccz, cry, crz, cswap, toffoli  # noqa: E402
from hyqnet.tensor import Tensor, backward, tsum  # noqa: E402


# --- independent dense oracle (basis-state bit logic) ------------------------
def _single(kind, a):
    h = 0.5 * (a if a is not None else 0.0)
    return {"H": np.array([[1, 1], [1, -1]]) / np.sqrt(2), "X": np.array([[0, 1], [1, 0]]),
            "Y": np.array([[0, -1j], [1j, 0]]), "Z": np.diag([1, -1]),
            "RX": np.array([[np.cos(h), -1j * np.sin(h)], [-1j * np.sin(h), np.cos(h)]]),
            "RY": np.array([[np.cos(h), -np.sin(h)], [np.sin(h), np.cos(h)]]),
            "RZ": np.diag([np.exp(-1j * h), np.exp(1j * h)])}[kind].astype(complex)


def dense(n, op):
    dim = 1 << n
    u = np.zeros((dim, dim), dtype=complex)
    if len(op.targets) == 1:
        q, m = op.targets[0], _single(op.kind, op.angle)
        for j in range(dim):
            b = (j >> q) & 1
            u[j & ~(1 << q), j] += m[0, b]
            u[j | (1 << q), j] += m[1, b]
        return u
    a, b = op.targets
    for j in range(dim):
        ba, bb = (j >> a) & 1, (j >> b) & 1
        if op.kind == "CNOT":
            u[j ^ (1 << b) if ba else j, j] = 1
        elif op.kind == "CZ":
            u[j, j] = -1 if ba and bb else 1
        elif op.kind == "CR":
            u[j, j] = np.exp(1j * op.angle) if ba and bb else 1
        else:
            u[(j & ~(1 << a) & ~(1 << b)) | (bb << a) | (ba << b), j] = 1
    return u


def dense_circuit(c):
    u = np.eye(1 << c.n_qubits, dtype=complex)
    for op in c.ops:
        u = dense(c.n_qubits, op) @ u
    return u


def random_circuit(rng, n, gates):
    c = Circuit(n)
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ"] + (["CNOT", "CZ", "CR", "SWAP"] if n >= 2 else [])
    for _ in range(gates):
        k = kinds[rng.integers(len(kinds))]
        ang = float(rng.uniform(-2 * np.pi, 2 * np.pi))
        if k in ("CNOT", "CZ", "CR", "SWAP"):
            a, b = rng.choice(n, 2, replace=False)
            c.add(GateOp(k, (int(a), int(b)), ang if k == "CR" else None))
        else:
            c.add(GateOp(k, (int(rng.integers(n)),), ang if k.startswith("R") else None))
    return c


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


# --- test_qsim.py:85-196 ------------------------------------------------------
GATES = [GateOp("H", (0,)), GateOp("X", (0,)), GateOp("Y", (0,)), GateOp("Z", (0,)),
         GateOp("RX", (0,), 0.7), GateOp("RY", (0,), -1.2), GateOp("RZ", (0,), 2.5), GateOp("CNOT", (0, 1)),
         GateOp("CZ", (1, 0)), GateOp("CR", (0, 1), 0.9), GateOp("SWAP", (0, 2))]


@pytest.mark.parametrize("op", GATES, ids=lambda op: op.kind)
def test_gate_matches_dense(op, rng):
    psi = rng.standard_normal(8) + 1j * rng.standard_normal(8)
    psi /= np.linalg.norm(psi)
    sv = StateVector(3)
    sv.amplitudes[:] = psi
    apply_gate(sv, op)
    np.testing.assert_allclose(sv.amplitudes, dense(3, op) @ psi, atol=1e-12)


def test_gate_on_high_qubit_and_endianness(rng):
    psi = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    psi /= np.linalg.norm(psi)
    sv = StateVector(4)
    sv.amplitudes[:] = psi
    op = GateOp("RY", (3,), 0.4)
    apply_gate(sv, op)
    np.testing.assert_allclose(sv.amplitudes, dense(4, op) @ psi, atol=1e-12)
    sv = StateVector(2)
    apply_gate(sv, GateOp("X", (0,)))
    np.testing.assert_array_equal(sv.amplitudes, [0, 1, 0, 0])     # X(0): index 1
    apply_gate(sv, GateOp("CNOT", (0, 1)))
    np.testing.assert_array_equal(sv.amplitudes, [0, 0, 0, 1])     # control 0 set: index 3


def test_conventions():
    th = 0.618
    c, s = np.cos(th / 2), np.sin(th / 2)
    np.testing.assert_allclose(gate_matrix("RY", th), [[c, -s], [s, c]], atol=1e-15)
    circ = Circuit(2)
    circ.x(0); circ.x(1); circ.cr(0, 1, 0.77)
    np.testing.assert_allclose(simulate(circ).amplitudes, [0, 0, 0, np.exp(0.77j)], atol=1e-15)


def test_simulate_random_circuits_and_norm(rng):
    for _ in range(25):
        c = random_circuit(rng, int(rng.integers(1, 5)), int(rng.integers(0, 21)))
        np.testing.assert_allclose(simulate(c).amplitudes, dense_circuit(c)[:, 0], atol=1e-10)
    c = Circuit(1)
    c.x(0)
    init = StateVector(1)
    simulate(c, init)
    np.testing.assert_array_equal(init.amplitudes, [1, 0])           # initial state not mutated
    assert abs(simulate(random_circuit(rng, 4, 30)).norm() - 1.0) < 1e-12


def test_probabilities_order_and_marginals(rng):
    c = Circuit(2)
    c.h(0); c.cnot(0, 1)
    np.testing.assert_allclose(probabilities(simulate(c), [0, 1]), [0.5, 0, 0, 0.5], atol=1e-15)
    c = Circuit(2)
    c.x(1)
    st = simulate(c)
    np.testing.assert_allclose(probabilities(st, [0]), [1, 0], atol=1e-15)
    np.testing.assert_allclose(probabilities(st, [1]), [0, 1], atol=1e-15)
    np.testing.assert_allclose(probabilities(st, [0, 1]), [0, 0, 1, 0], atol=1e-15)
    np.testing.assert_allclose(probabilities(st, [1, 0]), [0, 1, 0, 0], atol=1e-15)
    st = simulate(random_circuit(rng, 3, 12))
    np.testing.assert_allclose(probabilities(st, [0, 1, 2]), np.abs(st.amplitudes) ** 2, atol=1e-12)


# --- test_qnn.py:29-266 ---------------------------------------------------------
def h_ry(inputs, params):
    c = Circuit(1)
    c.h(0)
    c.ry(0, inputs[0])
    c.measure(0)
    return c


def ry_param(inputs, params):
    c = Circuit(1)
    c.ry(0, params[0])
    c.measure(0)
    return c


def test_parameter_shift_known_answers():
    def execute(v):
        c = Circuit(1)
        c.ry(0, v[0])
        return float(np.abs(simulate(c).amplitudes[1]) ** 2)
    for th in np.linspace(-np.pi, np.pi, 9):
        (g,) = parameter_shift_grad(execute, [th], shift=np.pi / 2, grad_scale=0.5, upstream=1.0)
        assert g == pytest.approx(np.sin(th) / 2, abs=1e-12)
    (g,) = parameter_shift_grad(lambda v: v[0] * 2.0, [0.3], shift=0.1, grad_scale=0.5, upstream=3.0)
    assert g == pytest.approx(2.0 * 0.1 * 2 * 0.5 * 3.0)
    g = parameter_shift_grad(lambda v: v[0] * v[1], [2.0, 5.0], shift=np.pi / 2, grad_scale=0.5, upstream=1.0)
    assert g[0] == pytest.approx(np.pi / 2 * 5.0) and g[1] == pytest.approx(np.pi / 2 * 2.0)


def test_layer_closed_forms():
    layer = QuantumLayer(h_ry, n_params=0, machine_type=EXACT_PROB)
    th = np.linspace(-2 * np.pi, 2 * np.pi, 17)
    np.testing.assert_allclose(layer(Tensor(th.reshape(-1, 1), dtype=np.float64)).numpy()[:, 0],
                               (1 + np.sin(th)) / 2, atol=1e-12)
    x = Tensor(np.array([[0.4]]), requires_grad=True)
    backward(tsum(layer(x)))
    assert x.grad[0, 0] == pytest.approx(np.cos(0.4) / 2, abs=1e-10)
    lay = QuantumLayer(ry_param, n_params=1, machine_type=EXACT_PROB, param_init=[0.8])
    backward(tsum(lay(Tensor(np.zeros((1, 1))))))
    assert lay.params.grad[0] == pytest.approx(np.sin(0.8) / 2, abs=1e-10)


def test_layer_batch_dtype_and_sum():
    layer = QuantumLayer(h_ry, n_params=0)
    x = np.array([[0.1], [0.7], [-1.3]])
    together = layer(Tensor(x, dtype=np.float64)).numpy()
    single = [layer(Tensor(r.reshape(1, -1), dtype=np.float64)).numpy() for r in x]
    np.testing.assert_allclose(together, np.vstack(single), atol=1e-14)
    assert layer(Tensor(np.zeros((1, 1), dtype=np.float32))).dtype == np.float32
    assert layer(Tensor(np.zeros((1, 1), dtype=np.float64))).dtype == np.float64
    lay = QuantumLayer(ry_param, n_params=1, param_init=[0.5])
    backward(tsum(lay(Tensor(np.zeros((3, 1))))))
    assert lay.params.grad[0] == pytest.approx(3 * np.sin(0.5) / 2, abs=1e-10)


def test_layer_errors():
    def broken(inputs, params):
        raise ValueError("boom")
    with pytest.raises(CircuitError):
        QuantumLayer(broken, n_params=0)(Tensor(np.zeros((1, 1))))
    with pytest.raises(CircuitError):
        QuantumLayer(lambda i, p: None, n_params=0)(Tensor(np.zeros((1, 1))))
    for kw in ({"machine_type": "analog"}, {"n_params": -1}, {"shots": 0}, {"shift": 0.0},
               {"n_params": 2, "param_init": [1.0]}, {"machine_type": "noisy"}):
        args = {"n_params": 0, **kw}
        with pytest.raises(ConfigError):
            QuantumLayer(h_ry, **args)


def test_shots_deterministic_near_exact_and_zero_noise():
    a = QuantumLayer(h_ry, 0, machine_type=SHOT_SAMPLING, shots=100, seed=7)
    b = QuantumLayer(h_ry, 0, machine_type=SHOT_SAMPLING, shots=100, seed=7)
    x = Tensor(np.array([[0.3]]))
    np.testing.assert_array_equal(a(x).numpy(), b(x).numpy())
    lay = QuantumLayer(h_ry, 0, machine_type=SHOT_SAMPLING, shots=4000, seed=3)
    got = lay(Tensor(np.array([[0.9]]), dtype=np.float64)).item()
    assert abs(got - (1 + np.sin(0.9)) / 2) < 4 * np.sqrt(0.25 / 4000)
    model = NoiseModel()
    model.add("H", bit_flip(0.0))
    noisy = NoiseQuantumLayer(h_ry, 0, noise_model=model, shots=250, seed=5)
    clean = QuantumLayer(h_ry, 0, machine_type=SHOT_SAMPLING, shots=250, seed=5)
    x = Tensor(np.array([[0.6], [1.1]]), dtype=np.float64)
    np.testing.assert_array_equal(noisy(x).numpy(), clean(x).numpy())


def test_grad_scale_one_uses_raw_difference():
    for scale in (0.5, 1.0):
        layer = QuantumLayer(h_ry, 0, grad_scale=scale)
        x = Tensor(np.array([[0.4]]), requires_grad=True)
        backward(tsum(layer(x)))
        assert x.grad[0, 0] == pytest.approx(2 * scale * np.cos(0.4) / 2, abs=1e-10)


def test_qae_layout_range_and_known_values(rng):
    layer = QAELayer(trash_qubits=2, total_qubits=7)
    assert layer.training_size == 4 and layer.n_params == 60 and layer.params.data.shape == (60,)
    assert layer.reference_qubits == [1, 2] and layer.training_register == [3, 4, 5, 6]
    assert layer.trash_register == [5, 6]
    out = QAELayer(2, 7, machine_type=EXACT_PROB, seed=1)(Tensor(rng.standard_normal((3, 16)),
                                                                 dtype=np.float64)).numpy()
    assert np.all(out >= 0.5 - 1e-9) and np.all(out <= 1.0 + 1e-9)
    x = np.zeros((1, 16))
    x[0, :4] = 0.5
    assert QAELayer(2, 7, machine_type=EXACT_PROB, param_init=np.zeros(60))(
        Tensor(x, dtype=np.float64)).item() == pytest.approx(1.0)
    x = np.zeros((1, 4))
    x[0, 2] = 1.0
    assert QAELayer(1, 4, machine_type=EXACT_PROB, param_init=np.zeros(18))(
        Tensor(x, dtype=np.float64)).item() == pytest.approx(0.5)
    a = QAELayer(2, 7, machine_type=SHOT_SAMPLING, shots=100, seed=2, param_init=np.linspace(0, 1, 60))
    b = QAELayer(2, 7, machine_type=SHOT_SAMPLING, shots=100, seed=2, param_init=np.linspace(0, 1, 60))
    xe = Tensor(np.eye(1, 16), dtype=np.float64)
    np.testing.assert_array_equal(a(xe).numpy(), b(xe).numpy())


def test_qae_gradient_is_the_two_point_value_for_all_params():
    layer = QAELayer(1, 4, machine_type=EXACT_PROB, param_init=np.linspace(0.1, 1.1, 18))
    x = Tensor(np.array([[0.6, 0.8, 0.0, 0.0]]), dtype=np.float64)
    backward(tsum(layer(x)))
    analytic = layer.params.grad.copy()
    for i in range(18):
        layer.params.data[i] += layer.shift
        up = layer(x).item()
        layer.params.data[i] -= 2 * layer.shift
        down = layer(x).item()
        layer.params.data[i] += layer.shift
        assert analytic[i] == pytest.approx((up - down) * layer.grad_scale, abs=1e-10)
    # the per-qubit rotation triples are shift-exact: finite differences agree
    eps, single = 1e-6, list(range(0, 6)) + list(range(12, 18))
    fd = []
    for i in single:
        layer.params.data[i] += eps
        up = layer(x).item()
        layer.params.data[i] -= 2 * eps
        down = layer(x).item()
        layer.params.data[i] += eps
        fd.append((up - down) / (2 * eps))
    np.testing.assert_allclose(analytic[single], fd, atol=1e-7, rtol=1e-4)


def test_qae_input_not_differentiated_and_errors():
    layer = QAELayer(1, 4, machine_type=EXACT_PROB)
    x = Tensor(np.array([[1.0, 0.0, 0.0, 0.0]]), requires_grad=True)
    backward(tsum(layer(x)))
    assert x.grad is None and layer.params.grad is not None
    with pytest.raises(CircuitError):
        QAELayer(2, 7)(Tensor(np.ones((1, 17))))
    for args, kw in (((0, 4), {}), ((2, 3), {}), ((2, 7), {"machine_type": "noisy"}),
                     ((2, 7), {"param_init": np.zeros(10)})):
        with pytest.raises(ConfigError):
            QAELayer(*args, **kw)


# --- test_templates.py:68-161 ---------------------------------------------------
@pytest.mark.parametrize("vec", [[1, 0, 0, 0], [0, 1, 0, 0], [0.5, 0.5, 0.5, 0.5], [0.2, -0.4, 0.4, -0.8],
                                 [-1, 0, 0, 0], [0, 0, 0, -1], [3, 1, -4, 1, -5, 9, -2, 6]], ids=repr)
def test_amplitude_embedding_exact(vec):
    vec = np.asarray(vec, dtype=float)
    c = Circuit(int(np.log2(len(vec))), ops=amplitude_embedding(vec))
    np.testing.assert_allclose(simulate(c).amplitudes, vec / np.linalg.norm(vec), atol=1e-12)


def test_amplitude_embedding_random_padded_subset(rng):
    for n in (1, 2, 3, 4):
        v = rng.standard_normal(2 ** n)
        c = Circuit(n, ops=amplitude_embedding(v))
        np.testing.assert_allclose(simulate(c).amplitudes, v / np.linalg.norm(v), atol=1e-12)
    c = Circuit(2, ops=amplitude_embedding([0.6, 0.8], qubits=[0, 1]))
    np.testing.assert_allclose(simulate(c).amplitudes, [0.6, 0.8, 0, 0], atol=1e-12)
    v = rng.standard_normal(4)
    got = simulate(Circuit(3, ops=amplitude_embedding(v, qubits=[1, 2]))).amplitudes.reshape(2, 2, 2)
    np.testing.assert_allclose(got[:, :, 0], (v / np.linalg.norm(v)).reshape(2, 2), atol=1e-12)
    np.testing.assert_allclose(got[:, :, 1], 0, atol=1e-12)
    for bad, kw in (([0, 0, 0, 0], {}), ([1.0, np.nan], {}), ([1, 2, 3], {"qubits": [0]})):
        with pytest.raises(EncodingError):
            amplitude_embedding(bad, **kw)


def _unitary(n, ops):
    return np.column_stack([
        simulate(Circuit(n, ops=list(ops)), StateVector.from_amplitudes(np.eye(1 << n)[k])).amplitudes
        for k in range(1 << n)])


def _controlled(m, n, c, t):
    u = np.zeros((1 << n, 1 << n), dtype=complex)
    for j in range(1 << n):
        if (j >> c) & 1:
            b = (j >> t) & 1
            u[j & ~(1 << t), j] += m[0, b]
            u[j | (1 << t), j] += m[1, b]
        else:
            u[j, j] = 1
    return u


def test_composite_gates():
    th = 0.83
    m = np.array([[np.cos(th / 2), -np.sin(th / 2)], [np.sin(th / 2), np.cos(th / 2)]])
    np.testing.assert_allclose(_unitary(2, cry(0, 1, th)), _controlled(m, 2, 0, 1), atol=1e-12)
    th = -1.37
    m = np.diag([np.exp(-1j * th / 2), np.exp(1j * th / 2)])
    np.testing.assert_allclose(_unitary(2, crz(1, 0, th)), _controlled(m, 2, 1, 0), atol=1e-12)
    want = np.eye(8, dtype=complex)
    want[7, 7] = -1
    np.testing.assert_allclose(_unitary(3, ccz(0, 1, 2)), want, atol=1e-12)
    np.testing.assert_allclose(_unitary(3, toffoli(0, 1, 2)), np.eye(8)[:, [0, 1, 2, 7, 4, 5, 6, 3]], atol=1e-12)
    perm = list(range(8))
    perm[0b011], perm[0b101] = perm[0b101], perm[0b011]
    np.testing.assert_allclose(_unitary(3, cswap(0, 1, 2)), np.eye(8)[:, perm], atol=1e-12)
    got = _unitary(4, toffoli(3, 1, 0))
    for idx in range(16):
        out = int(np.argmax(np.abs(got[:, idx])))
        want_i = idx ^ 1 if ((idx >> 3) & 1) and ((idx >> 1) & 1) else idx
        assert out == want_i and abs(got[out, idx] - 1) < 1e-12


# --- test_acceptance.py:108-128 ------------------------------------------------
def test_acceptance_random_circuits_gate_by_gate():
    rng = np.random.default_rng(424242)
    for _ in range(200):
        n = int(rng.integers(1, 5))
        c = random_circuit(rng, n, int(rng.integers(1, 21)))
        sv = StateVector(n)
        for op in c.ops:
            apply_gate(sv, op)
            assert abs(np.linalg.norm(sv.amplitudes) - 1.0) <= 1e-10
        assert np.max(np.abs(sv.amplitudes - dense_circuit(c)[:, 0])) <= 1e-10


def test_acceptance_rotation_closed_forms():
    layer = QuantumLayer(h_ry, n_params=0, machine_type=EXACT_PROB)
    for th in np.linspace(-2 * np.pi, 2 * np.pi, 50):
        x = Tensor(np.array([[th]]), dtype=np.float64, requires_grad=True)
        out = layer(x)
        assert abs(out.data[0, 0] - (1 + np.sin(th)) / 2) <= 1e-10
        backward(tsum(out))
        assert abs(x.grad[0, 0] - np.cos(th) / 2) <= 1e-8
