"""Builder tracing: turn ``circuit_builder(inputs, params)`` into one tape.

The reference calls the user builder once per circuit evaluation —
``QuantumLayer._build`` (``qnn.py:95-105``) runs for every sample and for every
shifted evaluation of the shift rule (``qnn.py:35-52,136-153``).  Here the
builder is run a handful of times per forward with :class:`TracedFloat`
arguments: floats whose arithmetic also records an affine form
``const + Σ coef·var`` over the variables (inputs 0..d-1, params d..d+P-1).
The result is a *tape*: gate structure + one affine slot per angle, valid for
the whole batch, which the GPU evaluates per sample.

Soundness checks (anything failing them takes the per-sample host path in
``engine.py``, which reproduces the reference exactly, just slower):

* every angle is affine in the variables (no product of two traced values,
  no value-losing call such as ``np.sin(x)`` — caught because the recorded
  constant changes between traces);
* the gate structure is identical at the first and last batch rows and at a
  random point (data-dependent structure, e.g. ``templates.py:50``);
* the builder never inspects the value of a variable-dependent scalar:
  comparisons, truth tests, ``int``/``round``/``floor``/``ceil``/``divmod``
  (and so ``max``/``min``/``if x > c``) on a traced value mark the trace
  data-dependent, because a branch that flips only on a middle row would be
  invisible to the probes.

:func:`classify` decides per variable whether the adjoint pass reproduces the
reference's two-point value: a variable entering exactly one
frequency-1 gate (RX/RY/RZ/CR) with coefficient c has
``E(v+s) - E(v-s) = (2 sin(c s)/c)·dE/dv`` exactly, so
``grad = grad_scale·2·sin(c·s)·dE/dα``.  Everything else (several occurrences,
inputs feeding a state load) is evaluated by the batched two-point rule.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field

import numpy as np

from .errors import CircuitError

_NUM = (int, float, np.integer, np.floating)

# Set while a builder runs on traced scalars whenever it inspects the VALUE of a
# variable-dependent scalar (comparison, truth test, int/round/floor/...): the
# circuit may then depend on the data in a way two or three probe rows cannot
# rule out, so the trace is rejected and the per-sample path runs.
_probe = threading.local()


def _mark_data_dependent():
    _probe.data_dependent = True


def _fv(v) -> float:
    """Plain value of a number without marking the trace (internal use)."""
    return float.__float__(v) if isinstance(v, float) else float(v)


plain_float = _fv


class TracedFloat(float):
    """Float that carries ``_c + Σ _t[var]·var``; ``_t is None`` = non-affine."""

    __slots__ = ("_c", "_t")

    def __new__(cls, value, const, terms):
        obj = float.__new__(cls, value)
        obj._c = const
        obj._t = terms
        return obj

    # -- helpers -----------------------------------------------------------------
    @staticmethod
    def _lift(v):
        if isinstance(v, TracedFloat):
            return v._c, v._t
        if isinstance(v, _NUM) and not isinstance(v, bool):
            return _fv(v), {}
        return None

    def _affine(self, other, sa, sb, value):
        b = TracedFloat._lift(other)
        if b is None:
            return NotImplemented
        if self._t is None or b[1] is None:
            return TracedFloat(value, 0.0, None)
        terms = {k: sa * c for k, c in self._t.items()}
        for k, c in b[1].items():
            terms[k] = terms.get(k, 0.0) + sb * c
        return TracedFloat(value, sa * self._c + sb * b[0], terms)

    def _scaled(self, k, value):
        if self._t is None:
            return TracedFloat(value, 0.0, None)
        return TracedFloat(value, self._c * k, {v: c * k for v, c in self._t.items()})

    def _opaque(self, value):
        if self._t is not None and not self._t:   # traced constant stays a constant
            return TracedFloat(value, value, {})
        return TracedFloat(value, 0.0, None)

    # -- arithmetic --------------------------------------------------------------
    def __add__(self, o):
        r = self._affine(o, 1.0, 1.0, 0.0)
        return r if r is NotImplemented else TracedFloat(_fv(self) + _fv(o), r._c, r._t)

    __radd__ = __add__

    def __sub__(self, o):
        r = self._affine(o, 1.0, -1.0, 0.0)
        return r if r is NotImplemented else TracedFloat(_fv(self) - _fv(o), r._c, r._t)

    def __rsub__(self, o):
        r = self._affine(o, -1.0, 1.0, 0.0)
        return r if r is NotImplemented else TracedFloat(_fv(o) - _fv(self), r._c, r._t)

    def __mul__(self, o):
        b = TracedFloat._lift(o)
        if b is None:
            return NotImplemented
        value = _fv(self) * _fv(o)
        if b[1] is not None and not b[1]:
            return self._scaled(b[0], value)
        if self._t is not None and not self._t and b[1] is not None:
            return o._scaled(self._c, value)
        return TracedFloat(value, 0.0, None)

    __rmul__ = __mul__

    def __truediv__(self, o):
        b = TracedFloat._lift(o)
        if b is None:
            return NotImplemented
        value = _fv(self) / _fv(o)
        if b[1] is not None and not b[1]:
            return self._scaled(1.0 / b[0], value)
        return TracedFloat(value, 0.0, None)

    def __rtruediv__(self, o):
        if TracedFloat._lift(o) is None:
            return NotImplemented
        return self._opaque(_fv(o) / _fv(self))

    def __neg__(self):
        return self._scaled(-1.0, -_fv(self))

    def __pos__(self):
        return self

    def __abs__(self):
        return self._opaque(abs(_fv(self)))

    def __pow__(self, o, mod=None):
        if TracedFloat._lift(o) is None:
            return NotImplemented
        return self._opaque(_fv(self) ** _fv(o))

    def __rpow__(self, o):
        if TracedFloat._lift(o) is None:
            return NotImplemented
        return self._opaque(_fv(o) ** _fv(self))

    def __mod__(self, o):
        if TracedFloat._lift(o) is None:
            return NotImplemented
        return self._opaque(_fv(self) % _fv(o))

    def __floordiv__(self, o):
        if TracedFloat._lift(o) is None:
            return NotImplemented
        return self._opaque(_fv(self) // _fv(o))

    def __reduce__(self):
        return (float, (_fv(self),))

    # -- value inspection: a branch on a variable marks the trace data-dependent
    def _variable(self):
        return self._t is None or any(c != 0.0 for c in self._t.values())

    def _inspect(self, other=None):
        if self._variable() or (isinstance(other, TracedFloat) and other._variable()):
            _mark_data_dependent()

    def __lt__(self, o):
        self._inspect(o)
        return float.__lt__(self, o)

    def __le__(self, o):
        self._inspect(o)
        return float.__le__(self, o)

    def __gt__(self, o):
        self._inspect(o)
        return float.__gt__(self, o)

    def __ge__(self, o):
        self._inspect(o)
        return float.__ge__(self, o)

    def __eq__(self, o):
        self._inspect(o)
        return float.__eq__(self, o)

    def __ne__(self, o):
        self._inspect(o)
        return float.__ne__(self, o)

    __hash__ = float.__hash__

    def __bool__(self):
        self._inspect()
        return float.__bool__(self)

    def __int__(self):
        self._inspect()
        return float.__int__(self)

    def __trunc__(self):
        self._inspect()
        return float.__trunc__(self)

    def __floor__(self):
        self._inspect()
        return float.__floor__(self)

    def __ceil__(self):
        self._inspect()
        return float.__ceil__(self)

    def __round__(self, ndigits=None):
        self._inspect()
        return float.__round__(self, ndigits) if ndigits is not None else float.__round__(self)

    def __divmod__(self, o):
        self._inspect(o)
        return float.__divmod__(self, o)


# ------------------------------------------------------------------------------
@dataclass
class Tape:
    """Batch-invariant circuit: gate structure plus affine slot expressions."""

    n_qubits: int
    measured: list
    ops: list                  # (kind, targets tuple, slot or -1)
    preps: list                # (qubits tuple, first slot, n_values)
    slot_const: list = field(default_factory=list)
    slot_terms: list = field(default_factory=list)   # list of dict var -> coef
    affine: bool = True

    def structure_key(self):
        return (self.n_qubits, tuple(self.measured),
                tuple((k, t) for k, t, _ in self.ops),
                tuple((q, n) for q, _, n in self.preps))

    def same_as(self, other: "Tape") -> bool:
        if not (self.affine and other.affine):
            return False
        if self.structure_key() != other.structure_key():
            return False
        for c1, t1, c2, t2 in zip(self.slot_const, self.slot_terms,
                                  other.slot_const, other.slot_terms):
            if t1.keys() != t2.keys():
                return False
            if abs(c1 - c2) > 1e-9 * max(1.0, abs(c1)):
                return False
            for k in t1:
                if abs(t1[k] - t2[k]) > 1e-12 * max(1.0, abs(t1[k])):
                    return False
        return True


def _slot(tape: Tape, value) -> int:
    if isinstance(value, TracedFloat):
        if value._t is None:
            tape.affine = False
            terms = {}
        else:
            terms = {k: c for k, c in value._t.items() if c != 0.0}
        const = value._c
    elif isinstance(value, _NUM):
        const, terms = _fv(value), {}
    else:
        raise CircuitError(f"gate angle {value!r} is not a number")
    tape.slot_const.append(_fv(const))
    tape.slot_terms.append(terms)
    return len(tape.slot_const) - 1


def check_circuit(circuit):
    """Duck-typed circuit check (our Circuit or a reference hyqnet Circuit)."""
    if not all(hasattr(circuit, a) for a in ("n_qubits", "ops", "measured_qubits")):
        raise CircuitError("circuit builder must return a Circuit")
    return circuit


def tape_from_circuit(circuit) -> Tape:
    check_circuit(circuit)
    measured = [int(q) for q in circuit.measured_qubits] or list(range(circuit.n_qubits))
    tape = Tape(int(circuit.n_qubits), measured, [], [])
    for op in circuit.ops:
        if op.kind == "STATEPREP":
            first = len(tape.slot_const)
            for v in op.values:
                _slot(tape, v)
            tape.preps.append((tuple(op.targets), first, len(op.values)))
            tape.ops.append(("STATEPREP", tuple(op.targets), len(tape.preps) - 1))
        elif op.angle is None:
            tape.ops.append((op.kind, tuple(op.targets), -1))
        else:
            tape.ops.append((op.kind, tuple(op.targets), _slot(tape, op.angle)))
    return tape


def traced_call(builder, inputs, params):
    """Run the builder on traced scalars; error wrapping as ``qnn.py:96-104``."""
    d = len(inputs)
    xs = [TracedFloat(float(v), 0.0, {i: 1.0}) for i, v in enumerate(inputs)]
    ps = [TracedFloat(float(v), 0.0, {d + j: 1.0}) for j, v in enumerate(params)]
    _probe.data_dependent = False
    try:
        circuit = builder(xs, ps)
    except CircuitError:
        raise
    except Exception as exc:
        raise CircuitError(f"circuit builder failed: {exc}") from exc
    finally:
        dep = getattr(_probe, "data_dependent", False)
        _probe.data_dependent = False
    if circuit is None or not hasattr(circuit, "ops"):
        raise CircuitError("circuit builder must return a Circuit")
    tape = tape_from_circuit(circuit)
    if dep:
        tape.affine = False       # value-dependent control flow: per-sample path
    return tape


def trace(builder, x: np.ndarray, theta: np.ndarray, seed: int = 12345):
    """Trace at the first and last rows and at a random point.

    Returns ``(tape, ok)``; ``ok`` is False when the builder is not provably
    batch-invariant and affine (the caller then uses the per-sample path).
    """
    tape = traced_call(builder, x[0], theta)
    if not tape.affine:
        return tape, False
    rng = np.random.default_rng(seed)
    probes = []
    if x.shape[0] > 1:
        probes.append((x[-1], theta, True))
    probes.append((rng.uniform(-math.pi, math.pi, x.shape[1]),
                   rng.uniform(0.0, 2 * math.pi, theta.shape[0]), False))
    for xi, ti, real in probes:
        try:
            other = traced_call(builder, xi, ti)
        except CircuitError:
            # a real row failing is the reference's error too; a failing random
            # probe only means the builder cannot be proven batch-invariant
            if real:
                raise
            return tape, False
        if not tape.same_as(other):
            return tape, False
    return tape, True


# ------------------------------------------------------------------------------
MODE_ZERO, MODE_ADJOINT, MODE_TWOPOINT = 0, 1, 2
_FREQ1 = ("RX", "RY", "RZ", "CR")


def classify(tape: Tape, n_vars: int, wanted, shift: float, grad_scale: float):
    """Per-variable gradient mode, adjoint slot and factor (see module doc)."""
    occ = [[] for _ in range(n_vars)]
    in_prep = [False] * n_vars
    for kind, _, slot in tape.ops:
        if kind == "STATEPREP":
            _, first, count = tape.preps[slot]
            for s in range(first, first + count):
                for v in tape.slot_terms[s]:
                    in_prep[v] = True
        elif slot >= 0:
            for v, c in tape.slot_terms[slot].items():
                occ[v].append((slot, c, kind))
    mode = np.zeros(n_vars, np.int32)
    vslot = np.full(n_vars, -1, np.int32)
    factor = np.zeros(n_vars, np.float64)
    for v in range(n_vars):
        if not wanted[v]:
            continue
        if in_prep[v]:
            mode[v] = MODE_TWOPOINT
        elif not occ[v]:
            mode[v] = MODE_ZERO          # E does not depend on v: E(v+s)-E(v-s) = 0
        elif len(occ[v]) == 1 and occ[v][0][2] in _FREQ1:
            slot, c, _ = occ[v][0]
            mode[v] = MODE_ADJOINT
            vslot[v] = slot
            factor[v] = 2.0 * grad_scale * math.sin(c * shift)
        else:
            mode[v] = MODE_TWOPOINT
    return mode, vslot, factor


_DIAGONAL = ("Z", "RZ", "CZ", "CR")


def light_cone(tape: Tape):
    """Backward light cone of the EXACT_PROB readout (opt-in, ``HQ_LIGHTCONE=1``).

    E = Σ_i w(i)|ψ_i|² with w depending only on the measured qubits M.  Walking
    the tape backwards with K = qubits of the gates kept so far, a gate is
    dropped when it cannot change E:
      * it touches none of M ∪ K (a unitary on qubits the readout never sees);
      * it is diagonal (Z/RZ/CZ/CR) on qubits outside K (commutes with the
        diagonal readout and nothing later acts on them);
      * CNOT(c, t) with t outside M ∪ K and c outside K (it only permutes a
        traced-out bit, conditioned on a bit the readout reads diagonally).
    The kept gates act on M ∪ K only; the other qubits stay in |0> and are
    removed (qubits renumbered, measured order kept).  Variables left only in
    dropped gates get a zero derivative, which is also what the reference's
    two-point rule returns for them (E does not depend on them).
    Returns the reduced tape, or None when nothing can be removed or the tape
    has state loads."""
    if tape.preps or not tape.affine:
        return None
    M = set(tape.measured) if tape.measured else set(range(tape.n_qubits))
    K = set()
    kept = []
    for kind, tg, slot in reversed(tape.ops):
        qs = set(tg)
        if not (qs & (M | K)):
            continue
        if kind in _DIAGONAL and not (qs & K):
            continue
        if kind == "CNOT" and tg[1] not in (M | K) and tg[0] not in K:
            continue
        kept.append((kind, tg, slot))
        K |= qs
    kept.reverse()
    active = sorted(M | K)
    if len(kept) == len(tape.ops) and len(active) == tape.n_qubits:
        return None
    new = {q: i for i, q in enumerate(active)}
    out = Tape(len(active), [new[q] for q in tape.measured], [(k, tuple(new[q] for q in tg), s) for k, tg, s in kept],
               [], list(tape.slot_const), list(tape.slot_terms), True)
    return out
