"""CPU ORACLE — test infrastructure only, never the product.

A plain NumPy restatement of the reference's hot path (VQNet 2.0 / hyqnet,
``/root/reference/pkg/src/hyqnet``), used by ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs as the checker
and as the CPU timing baseline ("port").  Nothing in the package imports it.

Parity is PINNED: ``tests/test_oracle_golden.py`` checks this module against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``
imports hyqnet from /root/reference and records outputs/gradients).

Restated pieces (file:line in the reference):

* gate matrices                         qsim.py:25-45
* ``apply_gate`` on the little-endian state (qubit k = index bit k)
                                        qsim.py:143-176
* ``simulate`` from |0...0> or a copy   qsim.py:179-191
* ``probabilities`` marginal ordering   qsim.py:194-211
* EXACT_PROB readout  E = Σ_j j·P(j)    qnn.py:107-116
* two-point ``parameter_shift_grad``    qnn.py:35-52
* ``QuantumLayer.forward`` + df_x/df_p  qnn.py:123-154
* templates (embeddings, cry/crz, ccz/toffoli/cswap)   templates.py:16-143
* ``Circuit`` builder API + validation  qsim.py:48-140
* SHOT_SAMPLING draws (Philox4x64-10 per shot)          qsim.py:222-248
* NOISY trajectories: channels, NoiseModel, apply_channel, run_trajectory,
  simulate_noisy, NoiseQuantumLayer values + shift-rule gradients
                                        noise.py:23-153, qnn.py:107-111,157-166

The reference has no compiled code (it is pure Python + NumPy),
so there is no ``oracle/_ref`` build; ``oracle/Makefile`` is a no-op.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_R2 = 1.0 / math.sqrt(2.0)
_KINDS1 = ("H", "X", "Y", "Z", "RX", "RY", "RZ")
_KINDS2 = ("CNOT", "CZ", "CR", "SWAP")


class OracleError(ValueError):
    pass


# ---------------------------------------------------------------------------
# circuit data model (qsim.py:48-140)
@dataclass(frozen=True)
class Op:
    kind: str
    targets: tuple
    angle: float | None = None

    def __post_init__(self):
        object.__setattr__(self, "targets", tuple(int(q) for q in self.targets))
        if self.kind not in _KINDS1 + _KINDS2:
            raise OracleError(f"unknown gate {self.kind}")
        if (self.kind.startswith("R") or self.kind == "CR") and self.angle is None:
            raise OracleError(f"{self.kind} needs an angle")
        arity = 2 if self.kind in _KINDS2 else 1
        if len(self.targets) != arity or len(set(self.targets)) != arity:
            raise OracleError(f"bad targets {self.targets}")


@dataclass
class Circuit:
    n_qubits: int
    ops: list = field(default_factory=list)
    measured_qubits: list = field(default_factory=list)

    def add(self, op):
        if max(op.targets) >= self.n_qubits:
            raise OracleError("qubit out of range")
        self.ops.append(op)

    def extend(self, ops):
        for op in ops:
            self.add(op if isinstance(op, Op) else Op(op.kind, op.targets, op.angle))

    def h(self, q): self.add(Op("H", (q,)))
    def x(self, q): self.add(Op("X", (q,)))
    def y(self, q): self.add(Op("Y", (q,)))
    def z(self, q): self.add(Op("Z", (q,)))
    def rx(self, q, a): self.add(Op("RX", (q,), float(a)))
    def ry(self, q, a): self.add(Op("RY", (q,), float(a)))
    def rz(self, q, a): self.add(Op("RZ", (q,), float(a)))
    def cnot(self, c, t): self.add(Op("CNOT", (c, t)))
    def cz(self, c, t): self.add(Op("CZ", (c, t)))
    def cr(self, c, t, a): self.add(Op("CR", (c, t), float(a)))
    def swap(self, a, b): self.add(Op("SWAP", (a, b)))

    def measure(self, *qs):
        for q in qs:
            if q in self.measured_qubits:
                raise OracleError("measured twice")
            self.measured_qubits.append(int(q))


# ---------------------------------------------------------------------------
# state-vector simulator (qsim.py:25-45, 143-211)
def gate_matrix(kind, angle=None):
    if kind == "H":
        return np.array([[_R2, _R2], [_R2, -_R2]], dtype=np.complex128)
    if kind == "X":
        return np.array([[0, 1], [1, 0]], dtype=np.complex128)
    if kind == "Y":
        return np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
    if kind == "Z":
        return np.array([[1, 0], [0, -1]], dtype=np.complex128)
    c, s = math.cos(angle / 2.0), math.sin(angle / 2.0)
    if kind == "RX":
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
    if kind == "RY":
        return np.array([[c, -s], [s, c]], dtype=np.complex128)
    if kind == "RZ":
        return np.array([[np.exp(-0.5j * angle), 0], [0, np.exp(0.5j * angle)]], dtype=np.complex128)
    raise OracleError(kind)


def _pair_view(psi, n, t):
    # [high, bit t, low] view: element (h, b, l) is index h*2^(t+1) + b*2^t + l
    return psi.reshape(1 << (n - 1 - t), 2, 1 << t)


def _quad_view(psi, n, a, b):
    lo, hi = min(a, b), max(a, b)
    v = psi.reshape(1 << (n - 1 - hi), 2, 1 << (hi - lo - 1), 2, 1 << lo)
    return v, (1 if a == hi else 3), (1 if b == hi else 3)


def _sel(v, ax_a, va, ax_b, vb):
    idx = [slice(None)] * 5
    idx[ax_a] = va
    idx[ax_b] = vb
    return tuple(idx)


def apply_gate(psi, n, op):
    """In-place update of the complex128 state (qsim.py:150-176)."""
    if op.kind in _KINDS1:
        m = gate_matrix(op.kind, op.angle)
        v = _pair_view(psi, n, op.targets[0])
        n0 = m[0, 0] * v[:, 0, :] + m[0, 1] * v[:, 1, :]
        n1 = m[1, 0] * v[:, 0, :] + m[1, 1] * v[:, 1, :]
        v[:, 0, :] = n0
        v[:, 1, :] = n1
        return psi
    a, b = op.targets
    v, axa, axb = _quad_view(psi, n, a, b)
    if op.kind == "CNOT":
        s10, s11 = _sel(v, axa, 1, axb, 0), _sel(v, axa, 1, axb, 1)
        tmp = v[s10].copy()
        v[s10] = v[s11]
        v[s11] = tmp
    elif op.kind == "CZ":
        s11 = _sel(v, axa, 1, axb, 1)
        v[s11] = -v[s11]
    elif op.kind == "CR":
        s11 = _sel(v, axa, 1, axb, 1)
        v[s11] = np.exp(1j * op.angle) * v[s11]
    elif op.kind == "SWAP":
        s01, s10 = _sel(v, axa, 0, axb, 1), _sel(v, axa, 1, axb, 0)
        tmp = v[s01].copy()
        v[s01] = v[s10]
        v[s10] = tmp
    return psi


def simulate(circuit, initial=None):
    """Final amplitudes (qsim.py:179-191); ``initial`` is not mutated."""
    n = int(circuit.n_qubits)
    if initial is None:
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[0] = 1.0
    else:
        psi = np.array(initial, dtype=np.complex128).reshape(-1).copy()
    for op in circuit.ops:
        apply_gate(psi, n, op)
    return psi


def probabilities(psi, n, qubits):
    """Marginal over ``qubits``; outcome bit i = qubits[i] (qsim.py:194-211)."""
    p = np.abs(psi) ** 2
    idx = np.arange(p.size)
    out_idx = np.zeros(p.size, dtype=np.int64)
    for i, q in enumerate(qubits):
        out_idx |= ((idx >> q) & 1) << i
    return np.bincount(out_idx, weights=p, minlength=1 << len(qubits))


def expectation(circuit):
    """EXACT_PROB readout (qnn.py:107-116)."""
    qubits = list(circuit.measured_qubits) or list(range(circuit.n_qubits))
    probs = probabilities(simulate(circuit), circuit.n_qubits, qubits)
    return float(np.arange(probs.size) @ probs)


# ---------------------------------------------------------------------------
# templates (templates.py:16-143)
def angle_embedding(features, axis="Y", qubits=None):
    qubits = list(range(len(features))) if qubits is None else list(qubits)
    return [Op("R" + axis, (q,), float(f)) for f, q in zip(features, qubits)]


def basis_embedding(bits, qubits=None):
    qubits = list(range(len(bits))) if qubits is None else list(qubits)
    return [Op("X", (q,)) for b, q in zip(bits, qubits) if b]


def _ucry(controls, target, angles, ops):
    if not np.any(angles):
        return
    if not controls:
        ops.append(Op("RY", (target,), float(angles[0])))
        return
    h = len(angles) // 2
    lo, hi = angles[:h], angles[h:]
    _ucry(controls[1:], target, (lo + hi) / 2.0, ops)
    ops.append(Op("CNOT", (controls[0], target)))
    _ucry(controls[1:], target, (lo - hi) / 2.0, ops)
    ops.append(Op("CNOT", (controls[0], target)))


def amplitude_embedding(vector, qubits=None):
    v = np.asarray(vector, dtype=np.float64).reshape(-1)
    norm = np.linalg.norm(v)
    if v.size == 0 or not np.all(np.isfinite(v)) or norm == 0.0:
        raise OracleError("bad embedding vector")
    n = max(1, int(np.ceil(np.log2(v.size))))
    qubits = list(range(n)) if qubits is None else [int(q) for q in qubits]
    n = len(qubits)
    amps = np.zeros(1 << n)
    amps[:v.size] = v / norm
    norms = [None] * (n + 1)
    norms[n] = np.abs(amps)
    for d in range(n - 1, -1, -1):
        norms[d] = np.hypot(norms[d + 1][0::2], norms[d + 1][1::2])
    ops = []
    for depth in range(n):
        target = qubits[n - 1 - depth]
        controls = [qubits[n - 1 - k] for k in range(depth)]
        if depth == n - 1:
            pr = amps.reshape(-1, 2)
            angles = 2.0 * np.arctan2(pr[:, 1], pr[:, 0])
        else:
            ch = norms[depth + 1]
            angles = 2.0 * np.arctan2(ch[1::2], ch[0::2])
        _ucry(controls, target, angles, ops)
    return ops


def cry(c, t, a):
    return [Op("RY", (t,), a / 2.0), Op("CNOT", (c, t)), Op("RY", (t,), -a / 2.0), Op("CNOT", (c, t))]


def crz(c, t, a):
    return [Op("RZ", (t,), a / 2.0), Op("CNOT", (c, t)), Op("RZ", (t,), -a / 2.0), Op("CNOT", (c, t))]


def ccz(a, b, t):
    return [Op("CR", (b, t), math.pi / 2.0), Op("CNOT", (a, b)), Op("CR", (b, t), -math.pi / 2.0),
            Op("CNOT", (a, b)), Op("CR", (a, t), math.pi / 2.0)]


def toffoli(a, b, t):
    return [Op("H", (t,))] + ccz(a, b, t) + [Op("H", (t,))]


def cswap(c, a, b):
    return [Op("CNOT", (b, a))] + toffoli(c, a, b) + [Op("CNOT", (b, a))]


# ---------------------------------------------------------------------------
# layer semantics (qnn.py:35-52, 95-154)
def parameter_shift_grad(execute, values, shift, grad_scale, upstream):
    values = np.asarray(values, dtype=np.float64)
    g = np.zeros(values.size)
    for i in range(values.size):
        s = values.copy()
        s[i] = values[i] + shift
        ep = execute(s)
        s[i] = values[i] - shift
        em = execute(s)
        g[i] = (ep - em) * grad_scale * upstream
    return g


def run(builder, inputs, params):
    return expectation(builder([float(v) for v in inputs], [float(v) for v in params]))


def layer(builder, x, theta, want_x=True, want_p=True, shift=math.pi / 2, grad_scale=0.5,
          upstream=None):
    """QuantumLayer.forward + df_x/df_p (qnn.py:123-154).

    Returns (out [N], jac_x [N, d] at upstream 1, jac_p [N, P] at upstream 1,
    grad_x [N, d] with upstream, grad_p [P] = Σ_i in sample order).
    """
    x = np.asarray(x, dtype=np.float64)
    theta = np.asarray(theta, dtype=np.float64)
    n, d = x.shape
    g = np.ones(n) if upstream is None else np.asarray(upstream, dtype=np.float64).reshape(n)
    out = np.array([run(builder, x[i], theta) for i in range(n)])
    jx = np.zeros((n, d))
    jp = np.zeros((n, theta.size))
    gx = np.zeros((n, d))
    gp = np.zeros(theta.size)
    for i in range(n):
        if want_x:
            jx[i] = parameter_shift_grad(lambda v: run(builder, v, theta), x[i], shift, grad_scale, 1.0)
            gx[i] = parameter_shift_grad(lambda v: run(builder, v, theta), x[i], shift, grad_scale, g[i])
        if want_p and theta.size:
            jp[i] = parameter_shift_grad(lambda v: run(builder, x[i], v), theta, shift, grad_scale, 1.0)
            gp += jp[i] * g[i]
    return out, jx, jp, gx, gp


def sample_cost(builder, x_row, theta, n_param_pairs, shift=math.pi / 2):
    """One forward + ``n_param_pairs`` shifted parameter pairs of one sample —
    the bounded CPU-baseline unit.  Returns evaluations done."""
    run(builder, x_row, theta)
    k = min(int(n_param_pairs), theta.size)
    for j in range(k):
        t = theta.copy()
        t[j] = theta[j] + shift
        run(builder, x_row, t)
        t[j] = theta[j] - shift
        run(builder, x_row, t)
    return 1 + 2 * k


def qae_builder(trash_qubits, total_qubits):
    """QAELayer circuit (qnn.py:196-250) as a builder; the layer output is
    P(aux = 0) = 1 - E with E the measure(0) readout (qnn.py:252-258)."""
    t = total_qubits - 1 - trash_qubits
    refs = list(range(1, 1 + trash_qubits))
    train = list(range(1 + trash_qubits, total_qubits))
    trash = train[-trash_qubits:]

    def build(inputs, params):
        it = iter(params)
        c = Circuit(total_qubits)
        c.extend(amplitude_embedding(inputs, qubits=train))

        def triple(q):
            c.rz(q, next(it)); c.ry(q, next(it)); c.rz(q, next(it))

        for q in train:
            triple(q)
        for a in train:
            for b in train:
                if a != b:
                    c.extend(crz(a, b, next(it)))
                    c.extend(cry(a, b, next(it)))
                    c.extend(crz(a, b, next(it)))
        for q in train:
            triple(q)
        c.h(0)
        for tq, rq_ in zip(trash, refs):
            c.extend(cswap(0, tq, rq_))
        c.h(0)
        c.measure(0)
        return c
    build.n_params = 6 * t + 3 * t * (t - 1)
    return build


# ---------------------------------------------------------------------------
# SHOT_SAMPLING (qsim.py:222-248, qnn.py:27-32, 117-118)
_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_MASK = (1 << 64) - 1


def philox_uniform(seed, shot):
    """First draw of np.random.Generator(np.random.Philox(key=[seed, shot])).random():
    Philox4x64-10, counter (1,0,0,0) (bumped before the first block), key
    (seed, shot), output word 0 >> 11 times 2^-53."""
    c = [1, 0, 0, 0]
    k = [seed & _MASK, shot & _MASK]
    for r in range(10):
        if r:
            k = [(k[0] + _W0) & _MASK, (k[1] + _W1) & _MASK]
        p0, p1 = _M0 * c[0], _M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & _MASK, (p0 >> 64) ^ c[3] ^ k[1], p0 & _MASK]
    return (c[0] >> 11) * (1.0 / 9007199254740992.0)


def measure_shots(psi, n, qubits, shots, seed):
    """Counts dict {bitstring: count} (qsim.py:236-248)."""
    cum = np.cumsum(probabilities(psi, n, qubits))
    tally = {}
    for s in range(shots):
        u = philox_uniform(seed, s)
        idx = min(int(np.searchsorted(cum, u, side="right")), len(cum) - 1)
        key = format(idx, f"0{len(qubits)}b")
        tally[key] = tally.get(key, 0) + 1
    return tally


def shot_expectation(circuit, shots, seed):
    qubits = list(circuit.measured_qubits) or list(range(circuit.n_qubits))
    counts = measure_shots(simulate(circuit), circuit.n_qubits, qubits, shots, seed)
    return sum(int(k, 2) * c for k, c in counts.items()) / shots


# ---------------------------------------------------------------------------
# NOISY machine type: per-shot Kraus trajectories (noise.py:1-153)
def philox_draw(seed, shot, k):
    """k-th ``random()`` of np.random.Generator(np.random.Philox(key=[seed, shot])):
    block b = k // 4 uses counter b + 1 (the counter is bumped before every
    block), output word k % 4, (w >> 11)·2^-53 (numpy philox4x64 buffering)."""
    b, wsel = divmod(int(k), 4)
    c = [(b + 1) & _MASK, 0, 0, 0]
    key = [seed & _MASK, shot & _MASK]
    for r in range(10):
        if r:
            key = [(key[0] + _W0) & _MASK, (key[1] + _W1) & _MASK]
        p0, p1 = _M0 * c[0], _M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ key[0], p1 & _MASK, (p0 >> 64) ^ c[3] ^ key[1], p0 & _MASK]
    return (c[wsel] >> 11) * (1.0 / 9007199254740992.0)


CHANNEL_NAMES = ("bit_flip", "phase_flip", "depolarizing", "amplitude_damping")


@dataclass(frozen=True)
class Channel:
    """noise.py:23-34."""
    name: str
    param: float

    def __post_init__(self):
        if self.name not in CHANNEL_NAMES:
            raise OracleError(f"unknown channel {self.name!r}")
        if not 0.0 <= self.param <= 1.0:
            raise OracleError(f"{self.name} parameter {self.param} outside [0, 1]")


class NoiseModel:
    """Gate kind (optionally per qubit) -> channel list (noise.py:54-78)."""

    def __init__(self):
        self.by_kind, self.by_kind_qubit = {}, {}

    def add(self, kind, channel, qubit=None):
        if qubit is None:
            self.by_kind.setdefault(kind, []).append(channel)
        else:
            self.by_kind_qubit.setdefault((kind, int(qubit)), []).append(channel)
        return self

    def channels_for(self, kind, qubit):
        ov = self.by_kind_qubit.get((kind, qubit))
        return ov if ov is not None else self.by_kind.get(kind, [])


class _ShotStream:
    """Sequential draws of one shot's Philox substream (qsim.py:222-224)."""

    def __init__(self, seed, shot):
        self.seed, self.shot, self.k = seed, shot, 0

    def random(self):
        u = philox_draw(self.seed, self.shot, self.k)
        self.k += 1
        return u


def apply_channel(psi, n, qubit, ch, rng):
    """One Kraus jump in place; zero-parameter channels draw nothing (noise.py:93-127)."""
    p = ch.param
    if p == 0.0:
        return
    if ch.name == "bit_flip":
        if rng.random() < p:
            apply_gate(psi, n, Op("X", (qubit,)))
    elif ch.name == "phase_flip":
        if rng.random() < p:
            apply_gate(psi, n, Op("Z", (qubit,)))
    elif ch.name == "depolarizing":
        u = rng.random()
        if u < 0.75 * p:
            apply_gate(psi, n, Op("XYZ"[int(u // (0.25 * p))], (qubit,)))
    else:  # amplitude_damping
        v = _pair_view(psi, n, qubit)
        p_jump = p * float((np.abs(v[:, 1, :]) ** 2).sum())
        if rng.random() < p_jump:
            v[:, 0, :] = np.sqrt(p) * v[:, 1, :]
            v[:, 1, :] = 0.0
            norm = np.sqrt(p_jump)
        else:
            v[:, 1, :] = np.sqrt(1.0 - p) * v[:, 1, :]
            norm = np.sqrt(1.0 - p_jump)
        if norm > 0:
            psi /= norm


def run_trajectory(circuit, noise, rng):
    """noise.py:130-138: channels act after each gate on every qubit it touched."""
    n = int(circuit.n_qubits)
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1.0
    for op in circuit.ops:
        apply_gate(psi, n, op)
        for q in op.targets:
            for ch in noise.channels_for(op.kind, q):
                apply_channel(psi, n, q, ch, rng)
    return psi


def simulate_noisy(circuit, noise, shots, seed):
    """Counts dict of per-shot trajectories, one final draw each (noise.py:141-153)."""
    qubits = list(circuit.measured_qubits) or list(range(circuit.n_qubits))
    tally = {}
    for s in range(shots):
        rng = _ShotStream(seed, s)
        psi = run_trajectory(circuit, noise, rng)
        cum = np.cumsum(probabilities(psi, circuit.n_qubits, qubits))
        idx = min(int(np.searchsorted(cum, rng.random(), side="right")), len(cum) - 1)
        key = format(idx, f"0{len(qubits)}b")
        tally[key] = tally.get(key, 0) + 1
    return tally


def noisy_expectation(circuit, noise, shots, seed):
    """qnn.py:107-111 + expectation_from_counts (qnn.py:27-32)."""
    counts = simulate_noisy(circuit, noise, shots, seed)
    return sum(int(k, 2) * c for k, c in counts.items()) / shots


def noisy_layer(builder, x, theta, noise, shots, seed, want_x=True, want_p=True,
                shift=math.pi / 2, grad_scale=0.5):
    """NoiseQuantumLayer forward + shift-rule jacobians (qnn.py:123-166)."""
    x = np.asarray(x, dtype=np.float64)
    theta = np.asarray(theta, dtype=np.float64)
    ex = lambda i, p: noisy_expectation(builder([float(v) for v in i], [float(v) for v in p]),
                                        noise, shots, seed)
    out = np.array([ex(x[i], theta) for i in range(len(x))])
    jx = np.array([parameter_shift_grad(lambda v: ex(v, theta), x[i], shift, grad_scale, 1.0)
                   if want_x else np.zeros(x.shape[1]) for i in range(len(x))])
    jp = np.array([parameter_shift_grad(lambda v: ex(x[i], v), theta, shift, grad_scale, 1.0)
                   if want_p and theta.size else np.zeros(theta.size) for i in range(len(x))])
    return out, jx, jp
