"""Circuit data model of the drop-in boundary, executed on the B200.

The builder-facing API restates ``pkg/src/hyqnet/qsim.py``:

* gate kinds and ``gate_matrix`` conventions      — ``qsim.py:19-45``
  (half-angle rotations, RZ = diag(e^{-iθ/2}, e^{iθ/2}), CR = e^{iθ} on |11⟩)
* ``GateOp`` validation                           — ``qsim.py:48-71``
* ``Circuit`` + helper methods + ``measure``      — ``qsim.py:94-140``
* little-endian qubits: qubit k is bit k of the amplitude index (``qsim.py:143-147``)
* ``probabilities`` outcome order                  — ``qsim.py:194-211``

``simulate`` / ``probabilities`` do not run NumPy loops: they lower the
circuit to a plan and run the sm_100a kernels (``engine.py``).  The qubit cap
is raised from the reference's 24 (``qsim.py:17``) to what one B200's HBM holds.

One extension: :class:`StatePrepOp`, emitted by ``templates.amplitude_embedding``
only while a builder is being traced; it is the native state load that replaces
the O(2^T) multiplexed-RY cascade (``templates.py:46-106``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import CircuitError, ContractError, FormatError

MAX_QUBITS = 34

SINGLE_GATES = ("H", "X", "Y", "Z")
ROTATION_GATES = ("RX", "RY", "RZ")
CONTROLLED_GATES = ("CNOT", "CZ", "CR", "SWAP")
GATE_KINDS = SINGLE_GATES + ROTATION_GATES + CONTROLLED_GATES

_R2 = 1.0 / np.sqrt(2.0)


def gate_matrix(kind: str, angle: float | None = None) -> np.ndarray:
    """2x2 complex128 matrix of a single-qubit kind (``qsim.py:33-45``)."""
    if kind == "H":
        return np.array([[_R2, _R2], [_R2, -_R2]], dtype=np.complex128)
    if kind == "X":
        return np.array([[0, 1], [1, 0]], dtype=np.complex128)
    if kind == "Y":
        return np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
    if kind == "Z":
        return np.array([[1, 0], [0, -1]], dtype=np.complex128)
    if kind in ROTATION_GATES:
        c, s = np.cos(angle / 2.0), np.sin(angle / 2.0)
        if kind == "RX":
            return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
        if kind == "RY":
            return np.array([[c, -s], [s, c]], dtype=np.complex128)
        return np.array([[np.exp(-0.5j * angle), 0], [0, np.exp(0.5j * angle)]],
                        dtype=np.complex128)
    raise CircuitError(f"{kind} has no single-qubit matrix")


@dataclass(frozen=True)
class GateOp:
    """One gate: ``kind``, ``targets`` (control first for 2-qubit kinds), ``angle``."""

    kind: str
    targets: tuple
    angle: float | None = None

    def __post_init__(self):
        object.__setattr__(self, "targets", tuple(int(q) for q in self.targets))
        if self.kind not in GATE_KINDS:
            raise CircuitError(f"unknown gate kind {self.kind!r}")
        if self.kind in ROTATION_GATES or self.kind == "CR":
            if self.angle is None or not np.isfinite(self.angle):
                raise CircuitError(f"{self.kind} requires one finite angle")
        elif self.angle is not None:
            raise CircuitError(f"{self.kind} takes no angle")
        arity = 2 if self.kind in CONTROLLED_GATES else 1
        if len(self.targets) != arity:
            raise CircuitError(f"{self.kind} acts on {arity} qubit(s), got {self.targets}")
        if len(set(self.targets)) != arity:
            raise CircuitError(f"duplicate targets in {self.kind} {self.targets}")
        if min(self.targets) < 0:
            raise CircuitError(f"negative qubit index in {self.targets}")


@dataclass(frozen=True)
class StatePrepOp:
    """Native amplitude load: ``values`` (traced input scalars, zero-padded to
    2^len(targets)) normalised onto ``targets`` (value bit i -> targets[i])."""

    targets: tuple
    values: tuple
    kind: str = "STATEPREP"
    angle: None = None


class StateVector:
    """Host copy of 2^n complex128 amplitudes, initialised to |0...0>."""

    def __init__(self, n_qubits: int):
        if not 1 <= n_qubits <= MAX_QUBITS:
            raise CircuitError(f"n_qubits must be in 1..{MAX_QUBITS}, got {n_qubits}")
        self.n_qubits = int(n_qubits)
        self.amplitudes = np.zeros(2 ** self.n_qubits, dtype=np.complex128)
        self.amplitudes[0] = 1.0

    @classmethod
    def from_amplitudes(cls, amps) -> "StateVector":
        amps = np.asarray(amps, dtype=np.complex128).reshape(-1)
        n = int(round(np.log2(amps.size)))
        if amps.size != 1 << n or n < 1:
            raise CircuitError(f"{amps.size} amplitudes is not a power of two >= 2")
        out = cls.__new__(cls)
        out.n_qubits, out.amplitudes = n, amps.copy()
        return out

    def copy(self) -> "StateVector":
        return StateVector.from_amplitudes(self.amplitudes)

    def norm(self) -> float:
        return float(np.sqrt(np.sum(np.abs(self.amplitudes) ** 2)))


@dataclass
class Circuit:
    """Ordered tape plus measured qubits (``qsim.py:94-140``)."""

    n_qubits: int
    ops: list = field(default_factory=list)
    measured_qubits: list = field(default_factory=list)

    def __post_init__(self):
        if not 1 <= self.n_qubits <= MAX_QUBITS:
            raise CircuitError(f"n_qubits must be in 1..{MAX_QUBITS}, got {self.n_qubits}")
        ops, measured = self.ops, self.measured_qubits
        self.ops, self.measured_qubits = [], []
        self.extend(ops)
        self.measure(*measured)

    def add(self, op) -> None:
        if max(op.targets) >= self.n_qubits:
            raise CircuitError(f"{op.kind} targets {op.targets} exceed {self.n_qubits} qubits")
        self.ops.append(op)

    def extend(self, ops) -> None:
        for op in ops:
            self.add(op)

    def h(self, q): self.add(GateOp("H", (q,)))
    def x(self, q): self.add(GateOp("X", (q,)))
    def y(self, q): self.add(GateOp("Y", (q,)))
    def z(self, q): self.add(GateOp("Z", (q,)))
    def rx(self, q, angle): self.add(GateOp("RX", (q,), angle))
    def ry(self, q, angle): self.add(GateOp("RY", (q,), angle))
    def rz(self, q, angle): self.add(GateOp("RZ", (q,), angle))
    def cnot(self, control, target): self.add(GateOp("CNOT", (control, target)))
    def cz(self, control, target): self.add(GateOp("CZ", (control, target)))
    def cr(self, control, target, angle): self.add(GateOp("CR", (control, target), angle))
    def swap(self, a, b): self.add(GateOp("SWAP", (a, b)))

    def measure(self, *qubits) -> None:
        for q in qubits:
            if not 0 <= q < self.n_qubits:
                raise CircuitError(f"measured qubit {q} out of range")
            if q in self.measured_qubits:
                raise CircuitError(f"qubit {q} measured twice")
            self.measured_qubits.append(q)


def simulate(circuit, initial: StateVector | None = None, precision: str = "c128") -> StateVector:
    """Final state of ``circuit`` computed on the GPU (``qsim.py:179-191``).

    The caller's ``initial`` state is not mutated.
    """
    from . import engine
    if initial is not None and initial.n_qubits != circuit.n_qubits:
        raise CircuitError(f"initial state has {initial.n_qubits} qubits, "
                           f"circuit has {circuit.n_qubits}")
    init = None if initial is None else initial.amplitudes
    amps = engine.simulate_circuit(circuit, init, precision=precision)
    return StateVector.from_amplitudes(amps)


def apply_gate(state: StateVector, op) -> None:
    """Apply one gate to ``state`` in place (``qsim.py:150-176``), on the GPU."""
    from . import engine
    if max(op.targets) >= state.n_qubits:
        raise CircuitError(f"{op.kind} targets {op.targets} exceed {state.n_qubits} qubits")
    c = Circuit(state.n_qubits)
    c.add(op)
    state.amplitudes[:] = engine.simulate_circuit(c, state.amplitudes)


def measure_shots(state: StateVector, qubits, shots: int, seed: int):
    """``qsim.py:236-248`` (device sampling; see ``qnn.measure_shots``)."""
    from .qnn import measure_shots as _ms
    return _ms(state, qubits, shots, seed)


def shot_rng(seed: int, shot: int):
    """``qsim.py:222-224``."""
    from .qnn import shot_rng as _sr
    return _sr(seed, shot)


def probabilities(state, qubits):
    """Marginal Born distribution over ``qubits``; outcome bit i = qubits[i]
    (``qsim.py:194-211``).  A host ``StateVector`` (the reference's type) is
    reduced on the host copy; a device state — a CUDA tensor of amplitudes
    ([2^n] complex, or [rows, 2^n] / [rows, 2^n, 2] batches) — is reduced on
    the GPU by ``hq_marginal`` and the result stays on the device."""
    if hasattr(state, "is_cuda") and state.is_cuda:
        return _device_probabilities(state, qubits)
    qubits = [int(q) for q in qubits]
    if len(set(qubits)) != len(qubits):
        raise CircuitError(f"duplicate qubits in {qubits}")
    for q in qubits:
        if not 0 <= q < state.n_qubits:
            raise CircuitError(f"qubit {q} out of range for {state.n_qubits} qubits")
    p = np.abs(state.amplitudes) ** 2
    idx = np.arange(p.size)
    outcome = np.zeros(p.size, dtype=np.int64)
    for i, q in enumerate(qubits):
        outcome |= ((idx >> q) & 1) << i
    return np.bincount(outcome, weights=p, minlength=1 << len(qubits))


def _device_probabilities(state, qubits):
    import torch
    from . import engine
    if state.is_complex():                      # [2^n] or [rows, 2^n]
        single = state.dim() == 1
        t = torch.view_as_real(state.to(torch.complex128).contiguous())
    else:                                       # [2^n, 2] or [rows, 2^n, 2]
        single = state.dim() == 2
        t = state.to(torch.float64)
    t = t.reshape(1 if single else t.shape[0], -1, 2)
    n = int(t.shape[1]).bit_length() - 1
    if 1 << n != t.shape[1]:
        raise CircuitError(f"{t.shape[1]} amplitudes is not a power of two")
    qubits = [int(q) for q in qubits]
    if len(set(qubits)) != len(qubits):
        raise CircuitError(f"duplicate qubits in {qubits}")
    for q in qubits:
        if not 0 <= q < n:
            raise CircuitError(f"qubit {q} out of range for {n} qubits")
    p = engine.marginal_probabilities(t.contiguous(), n, qubits)
    return p[0] if single else p


def readout_weights(n_qubits: int, measured) -> list:
    """Measured qubit list the EXACT_PROB readout uses (``qnn.py:108``)."""
    measured = list(measured) or list(range(n_qubits))
    return [int(q) for q in measured]


class Counts(dict):
    """Bitstring -> count map carrying the shot total (``qsim.py:214-219``)."""

    def __init__(self, mapping=(), shots: int = 0):
        super().__init__(mapping)
        self.shots = int(shots)


def bitstring(index: int, width: int) -> str:
    return format(index, f"0{width}b")


def _check_shots(shots):
    if shots < 1:
        raise ContractError(f"shots must be >= 1, got {shots}")


def format_circuit_text(circuit) -> str:
    """One op per line (``qsim.py:281-291``)."""
    lines = []
    for op in circuit.ops:
        t = ",".join(str(q) for q in op.targets)
        lines.append(f"{op.kind} {t} {op.angle!r}" if op.angle is not None else f"{op.kind} {t}")
    if circuit.measured_qubits:
        lines.append("MEASURE " + " ".join(str(q) for q in circuit.measured_qubits))
    return "\n".join(lines) + "\n"


def parse_circuit_text(text: str) -> Circuit:
    """Inverse of :func:`format_circuit_text` (``qsim.py:251-278``)."""
    ops, measured, top = [], [], 0
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        kind = tok[0].upper()
        try:
            if kind == "MEASURE":
                measured.extend(int(t) for t in tok[1:])
                used = measured
            else:
                targets = tuple(int(t) for t in tok[1].split(","))
                ops.append(GateOp(kind, targets, float(tok[2]) if len(tok) > 2 else None))
                used = targets
        except (IndexError, ValueError) as exc:   # CircuitError is a ValueError too
            raise FormatError(f"bad circuit line {raw!r}: {exc}") from None
        if used:
            top = max(top, max(used))
    c = Circuit(top + 1)
    c.extend(ops)
    c.measure(*measured)
    return c
