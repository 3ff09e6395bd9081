"""Host-side logic (CPU): circuit API + validation, tracer, gradient classifier,
templates vs the oracle's restatement, autograd boundary."""

import math

import numpy as np
import pytest

from oracle import hq_oracle as O
from paper_2301_03251_b200 import (Circuit, CircuitError, ConfigError, EncodingError, FormatError,
                                   GateOp, StatePrepOp, Tensor, backward, tsum, workloads as wl)
from paper_2301_03251_b200 import templates as T
from paper_2301_03251_b200 import qsim
from paper_2301_03251_b200 import tracer as tr
from paper_2301_03251_b200.qnn import QuantumLayer


class TestCircuitApi:
    def test_gateop_validation(self):
        for args in [("T", (0,)), ("RX", (0,)), ("H", (0,), 0.5), ("CNOT", (0,)), ("X", (0, 1)),
                     ("CNOT", (1, 1)), ("X", (-1,)), ("RY", (0,), float("nan"))]:
            with pytest.raises(CircuitError):
                GateOp(*args)

    def test_circuit_range_and_measure(self):
        c = Circuit(2)
        with pytest.raises(CircuitError):
            c.x(2)
        c.measure(0, 1)
        with pytest.raises(CircuitError):
            c.measure(0)
        with pytest.raises(CircuitError):
            Circuit(0)
        with pytest.raises(CircuitError):
            Circuit(qsim.MAX_QUBITS + 1)

    def test_text_round_trip(self):
        c = Circuit(3)
        c.h(0); c.cnot(0, 2); c.ry(1, 0.25); c.cr(1, 2, -0.5); c.measure(0, 2)
        p = qsim.parse_circuit_text(qsim.format_circuit_text(c))
        assert p.ops == c.ops and p.measured_qubits == c.measured_qubits
        for bad in ("FOO 0\n", "H zero\n", "RX 0\n"):
            with pytest.raises(FormatError):
                qsim.parse_circuit_text(bad)

    def test_probabilities_order(self):
        sv = qsim.StateVector(3)
        sv.amplitudes[:] = 0
        sv.amplitudes[0b110] = 1.0  # q1 = 1, q2 = 1
        p = qsim.probabilities(sv, [2, 0])
        assert p[0b01] == 1.0  # bit 0 of outcome = qubit 2


class TestTemplates:
    def test_gate_lists_match_oracle(self, rng):
        pairs = [
            (T.cry(0, 1, 0.83), O.cry(0, 1, 0.83)),
            (T.crz(1, 0, -1.37), O.crz(1, 0, -1.37)),
            (T.ccz(0, 1, 2), O.ccz(0, 1, 2)),
            (T.toffoli(3, 1, 0), O.toffoli(3, 1, 0)),
            (T.cswap(0, 1, 2), O.cswap(0, 1, 2)),
            (T.angle_embedding([0.1, 0.2], "X"), O.angle_embedding([0.1, 0.2], "X")),
        ]
        for v in (rng.standard_normal(16), [0.6, 0.8], [0.0, 0.0, 1.0, 0.0], [3, 1, -4, 1, -5]):
            pairs.append((T.amplitude_embedding(v), O.amplitude_embedding(v)))
        for mine, ref in pairs:
            assert [(o.kind, o.targets) for o in mine] == [(o.kind, o.targets) for o in ref]
            for a, b in zip(mine, ref):
                assert (a.angle is None) == (b.angle is None)
                if a.angle is not None:
                    assert a.angle == pytest.approx(b.angle, abs=1e-15)

    def test_embedding_errors(self):
        for bad in ([0, 0, 0, 0], [1.0, np.nan]):
            with pytest.raises(EncodingError):
                T.amplitude_embedding(bad)
        with pytest.raises(EncodingError):
            T.amplitude_embedding([1, 2, 3], qubits=[0])
        with pytest.raises(EncodingError):
            T.angle_embedding([0.1], axis="W")
        with pytest.raises(EncodingError):
            T.basis_embedding([2])


class TestTracer:
    def test_cfg1_is_affine_and_adjoint(self):
        b = wl.make_builder("cfg1", qsim, T)
        x = wl.inputs_for("cfg1", 4)
        th = wl.params_for("cfg1")
        tape, ok = tr.trace(b, x, th)
        assert ok and len(tape.ops) == 36 and len(tape.slot_const) == 28
        mode, slot, factor = tr.classify(tape, 28, [True] * 28, math.pi / 2, 0.5)
        assert (mode == tr.MODE_ADJOINT).all()
        np.testing.assert_allclose(factor, 1.0)   # 2 * 0.5 * sin(pi/2)

    def test_affine_forms(self):
        def b(inputs, params):
            c = Circuit(2)
            c.ry(0, 2.0 * inputs[0] - params[1] / 4 + 0.5)
            c.rz(1, -(params[0] + 1.0))
            c.cr(0, 1, math.pi * params[1])
            return c
        tape, ok = tr.trace(b, np.array([[0.3]]), np.array([0.1, 0.2]))
        assert ok
        assert tape.slot_terms[0] == {0: 2.0, 2: -0.25} and tape.slot_const[0] == 0.5
        assert tape.slot_terms[1] == {1: -1.0} and tape.slot_const[1] == -1.0
        assert tape.slot_terms[2] == {2: math.pi}
        mode, slot, factor = tr.classify(tape, 3, [True] * 3, math.pi / 2, 0.5)
        # x0 and theta0 once each; theta1 twice -> two-point
        assert list(mode) == [tr.MODE_ADJOINT, tr.MODE_ADJOINT, tr.MODE_TWOPOINT]
        assert factor[0] == pytest.approx(math.sin(2.0 * math.pi / 2))
        assert factor[1] == pytest.approx(math.sin(-math.pi / 2))

    def test_hidden_nonlinearity_detected(self):
        def b(inputs, params):
            c = Circuit(1)
            c.ry(0, float(np.sin(inputs[0])))
            return c
        _, ok = tr.trace(b, np.array([[0.3], [0.9]]), np.zeros(0))
        assert not ok

    def test_product_of_traced_values_is_non_affine(self):
        def b(inputs, params):
            c = Circuit(1)
            c.ry(0, inputs[0] * params[0])
            return c
        _, ok = tr.trace(b, np.array([[0.3]]), np.array([0.2]))
        assert not ok

    def test_data_dependent_structure_detected(self):
        def b(inputs, params):
            c = Circuit(2)
            if inputs[0] > 0:
                c.x(1)
            c.ry(0, inputs[0])
            return c
        _, ok = tr.trace(b, np.array([[0.3], [-0.2]]), np.zeros(0))
        assert not ok

    def test_branch_on_middle_row_detected(self):
        # the branch flips only on row 1: first/last/random probes all agree
        def b(inputs, params):
            c = Circuit(2)
            if inputs[0] > 2.0:
                c.x(1)
            c.ry(0, inputs[0])
            return c
        _, ok = tr.trace(b, np.array([[0.3], [2.5], [0.5]]), np.zeros(0))
        assert not ok

    @pytest.mark.parametrize("fn", [lambda v: max(v, 1.5), lambda v: min(v, -3.0),
                                    lambda v: float(round(v)), lambda v: float(math.floor(v)),
                                    lambda v: float(int(v)), lambda v: 0.3 if v else 0.1])
    def test_value_inspection_detected(self, fn):
        def b(inputs, params):
            c = Circuit(1)
            c.ry(0, fn(inputs[0]))
            return c
        _, ok = tr.trace(b, np.array([[0.3], [2.5], [0.5]]), np.zeros(0))
        assert not ok

    def test_constant_comparisons_stay_traced(self):
        # comparisons between constants (or a traced constant) are not data-dependent
        def b(inputs, params):
            c = Circuit(1)
            k = 0.0 * inputs[0] + 1.0
            if k > 0.5 and len(params) == 1:
                c.ry(0, params[0])
            return c
        _, ok = tr.trace(b, np.array([[0.3], [2.5]]), np.array([0.2]))
        assert ok

    def test_middle_row_branch_matches_oracle_per_sample(self):
        # the layer falls back to per-sample evaluation: row 1 sees its X gate
        from paper_2301_03251_b200 import engine
        called = []

        def fake_per_sample(builder, xd, pd, *a, **k):
            called.append(True)
            return np.zeros(xd.shape[0]), None, {"plan": None, "path": "per_sample"}

        def b(inputs, params):
            c = Circuit(2)
            if inputs[0] > 2.0:
                c.x(1)
            c.ry(0, inputs[0])
            return c
        orig = engine.run_per_sample
        engine.run_per_sample = fake_per_sample
        try:
            engine.run_batch(b, np.array([[0.3], [2.5], [0.5]]), np.zeros(0), False, False)
        finally:
            engine.run_per_sample = orig
        assert called

    def test_amplitude_embedding_lowers_to_state_load(self):
        b = wl.make_builder("cfg3", qsim, T)
        x = wl.inputs_for("cfg3", 3)
        tape, ok = tr.trace(b, x, wl.params_for("cfg3"))
        assert ok
        assert tape.ops[0][0] == "STATEPREP" and len(tape.preps) == 1
        assert tape.preps[0][2] == 512
        mode, _, _ = tr.classify(tape, 512 + 108, [True] * 620, math.pi / 2, 0.5)
        assert (mode[:512] == tr.MODE_TWOPOINT).all()
        assert (mode[512:] == tr.MODE_ADJOINT).all()

    def test_builder_error_wrapped(self):
        def b(inputs, params):
            raise ValueError("boom")
        with pytest.raises(CircuitError):
            tr.trace(b, np.zeros((1, 1)), np.zeros(0))

    def test_unused_variable_is_zero(self):
        def b(inputs, params):
            c = Circuit(1)
            c.ry(0, params[0])
            return c
        tape, ok = tr.trace(b, np.zeros((1, 2)), np.array([0.1]))
        mode, _, _ = tr.classify(tape, 3, [True] * 3, math.pi / 2, 0.5)
        assert list(mode) == [tr.MODE_ZERO, tr.MODE_ZERO, tr.MODE_ADJOINT]


class TestLayerConfig:
    def test_config_validation(self):
        b = wl.make_builder("cfg1", qsim, T)
        for kw in (dict(machine_type="analog"), dict(n_params=-1), dict(shots=0),
                   dict(shift=0.0), dict(n_params=2, param_init=[1.0]),
                   dict(machine_type="noisy"), dict(precision="c32")):
            args = dict(n_params=0)
            args.update(kw)
            with pytest.raises(ConfigError):
                QuantumLayer(b, **args)

    def test_default_init_draws_from_package_generator(self):
        from paper_2301_03251_b200 import manual_seed
        manual_seed(0)
        a = QuantumLayer(lambda i, p: None, n_params=5).params.data.copy()
        manual_seed(0)
        want = np.random.default_rng(0).uniform(0, 2 * np.pi, 5)
        np.testing.assert_array_equal(a, want)


class TestAutogradBoundary:
    def test_sum_backward(self):
        x = Tensor(np.array([[1.0, 2.0]]), requires_grad=True)
        y = tsum(x * 3.0 - 1.0)
        backward(y)
        np.testing.assert_array_equal(x.grad, [[3.0, 3.0]])


# ---------------------------------------------------------------------------
def _tape_expectation(tape, x_row, theta):
    """Oracle EXACT_PROB of a traced tape at concrete values."""
    from oracle import hq_oracle as Ora
    vals = list(x_row) + list(theta)
    c = Ora.Circuit(tape.n_qubits)
    for kind, tg, slot in tape.ops:
        ang = None
        if slot >= 0:
            ang = tape.slot_const[slot] + sum(coef * vals[v] for v, coef in tape.slot_terms[slot].items())
        c.add(Ora.Op(kind, tg, ang))
    if tape.measured:
        c.measure(*tape.measured)
    return Ora.expectation(c)


@pytest.mark.parametrize("seed", range(6))
def test_light_cone_keeps_expectation(seed):
    from paper_2301_03251_b200 import tracer as tr
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 9))
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
    plan = []
    for _ in range(40):
        k = kinds[rng.integers(len(kinds))]
        two = k in ("CNOT", "CZ", "CR", "SWAP")
        tg = tuple(int(q) for q in rng.choice(n, 2 if two else 1, replace=False))
        plan.append((k, tg, int(rng.integers(0, 5))))
    meas = [int(q) for q in rng.choice(n, int(rng.integers(1, 3)), replace=False)]

    def builder(inputs, params):
        c = Circuit(n)
        for k, tg, v in plan:
            ang = (inputs[v] if v < 2 else params[v - 2]) if k in ("RX", "RY", "RZ", "CR") else None
            getattr(c, k.lower())(*tg) if ang is None else getattr(c, k.lower())(*tg, ang)
        c.measure(*meas)
        return c
    x = rng.uniform(-3, 3, (2, 2))
    th = rng.uniform(0, 6, 3)
    tape, ok = tr.trace(builder, x, th)
    assert ok
    lc = tr.light_cone(tape) or tape
    for trial in range(3):
        xr = rng.uniform(-3, 3, 2)
        tr_ = rng.uniform(0, 6, 3)
        assert _tape_expectation(lc, xr, tr_) == pytest.approx(_tape_expectation(tape, xr, tr_), abs=1e-12)


def test_light_cone_cfg4_shrinks():
    from paper_2301_03251_b200 import tracer as tr, workloads as wl, qsim, templates as T
    b = wl.make_builder("cfg4", qsim, T)
    tape, ok = tr.trace(b, wl.inputs_for("cfg4", 2), wl.params_for("cfg4"))
    lc = tr.light_cone(tape)
    assert lc.n_qubits == 10 and len(lc.ops) == 164 and lc.measured == [0]


def test_non_finite_middle_row_raises_reference_error():
    # qsim.py:60-63: the sample's GateOp construction fails; the traced path
    # only builds probe rows, so engine checks every row's angles
    from paper_2301_03251_b200 import engine
    b = wl.make_builder("cfg1", qsim, T)
    x = wl.inputs_for("cfg1", 5)
    tape, ok = tr.trace(b, x, wl.params_for("cfg1"))
    assert ok
    engine._check_finite(tape, x, wl.params_for("cfg1"))      # finite: no error
    x[2, 1] = np.nan
    with pytest.raises(CircuitError, match="RY requires one finite angle"):
        engine._check_finite(tape, x, wl.params_for("cfg1"))
    th = wl.params_for("cfg1")
    th[4] = np.inf
    with pytest.raises(CircuitError, match="requires one finite angle"):
        engine._check_finite(tape, wl.inputs_for("cfg1", 5), th)
