"""Amplitude sharding of ONE circuit across R = 2^g ranks.

The reference holds one dense vector and stops at 24 qubits (``qsim.py:17,81``);
cfg5 (32 qubits, complex128: 64 GiB) is split by amplitude.  Global index
i = (rank << L) | local, L = n − g: the top g index bits are the rank.

Exchange.  ONE all-to-all swaps all g rank bits with the top g local bits
(the "staging" positions L−g..L−1): rank r sends its contiguous chunk j
(staging bits = j) to rank j and stores the chunk it receives from rank j at
chunk j — exactly ``ncclAllToAll`` / ``dist.all_to_all_single`` on contiguous
equal chunks, so nothing is packed or unpacked, and the exchange is an
involution (the adjoint replays it unchanged).  7/8 of the shard moves per
exchange at g = 3.

Schedule (:func:`schedule`).  A layout maps logical qubits to physical bit
positions.  The tape is scheduled as a frontier: every op whose exchange
qubits (targets of non-diagonal kinds) are local and whose earlier same-qubit
ops are done is emitted, in tape order, into the current local segment —
across layer boundaries, so on a CNOT-chain ansatz the frontier runs ahead as
a staircase.  When nothing more can run, g victims (the local qubits whose next
exchange use is furthest away) are moved to the staging positions by SWAP
gates at the end of the segment (register renamings inside the last pass's
tile), and the exchange follows.  cfg5 (n = 32, depth 20, g = 3) needs ONE
exchange for the whole forward (see ``tools/cfg5_sharded.py --schedule``).

Rank-constant qubits.  Inside a segment a global qubit may only be a control
or sit on a diagonal gate:
* CNOT(global c, local t) -> X(t) on ranks whose bit c is 1;
* CZ / CR with one global qubit -> Z / "phase on |1>" (the kernels' RZ form,
  diag(1, e^{iα}) — exactly CR's action) on the local qubit, same ranks;
* RZ / Z on a global qubit, and CZ / CR with both qubits global, are deferred
  until one of their qubits is local again (they commute with every
  intervening op on that qubit, which can only be a control or diagonal use),
  and skipped if the circuit ends first (they commute with the diagonal
  readout: E and every other derivative are unchanged, their own derivative
  is 0); only a request for the final state applies them, as the per-rank
  scalar ``tail_phase``.
So no rank ever carries a scalar phase of its own; the kernels' dropped phases
(RZ e^{-iθ/2}, rotation signs) are the same on every rank — a global phase,
invisible to E and to the adjoint dots.

Adjoint.  λ = w·ψ at the end (w from the measured qubits; measured qubits at
rank positions contribute a per-rank constant), then the steps in reverse:
segment backward passes (ψ un-applied, G† on λ, derivative dots into jacobian
rows), and each exchange replayed on ψ and on λ.  The per-rank rows are summed
by one all-reduce of the [d + P] vector (replaces df_p, ``qnn.py:145-153``).

Execution is generic over an executor (per-segment forward / backward /
readout on one rank's shard) and an exchange: :class:`GpuExecutor` runs
segment plans (``hq_plan_create_segment`` / ``hq_seg_*`` / ``hq_shard_readout``
in ``include/hq.h``) on device shards; :func:`run_nccl` drives one rank per
process over NCCL all-to-all; :func:`run_virtual` drives all ranks on one
device (parity tests, and the one-GPU measurement of the per-rank work).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import tracer as tr
from .errors import ConfigError

_EXCH = {"H": 1, "X": 1, "Y": 1, "RX": 1, "RY": 1}   # exchange on targets[0]
_DIAG = ("Z", "RZ", "CZ", "CR")


def exchange_qubits(kind, targets):
    """Qubits whose amplitudes the gate mixes (must be local)."""
    if kind in _EXCH:
        return [targets[0]]
    if kind == "CNOT":
        return [targets[1]]
    if kind == "SWAP":
        return list(targets)
    return []


@dataclass
class Schedule:
    n: int
    g: int
    steps: list = field(default_factory=list)          # ("local", [(kind, phys targets, slot)]) | ("exchange",)
    final_layout: list = field(default_factory=list)   # logical -> physical
    measured: list = field(default_factory=list)
    tail: list = field(default_factory=list)           # trailing global diagonal ops (commute with the readout)

    @property
    def dropped(self):
        return len(self.tail)

    @property
    def L(self):
        return self.n - self.g

    @property
    def exchanges(self):
        return sum(1 for s in self.steps if s[0] == "exchange")

    @property
    def segments(self):
        return [s[1] for s in self.steps if s[0] == "local"]


def schedule(n: int, g: int, ops, measured) -> Schedule:
    """Frontier schedule of ``ops`` = [(kind, logical targets, slot)] over 2^g ranks."""
    L = n - g
    if g < 0 or L < 2 * g or L < 2:
        raise ConfigError(f"amplitude sharding needs n - g >= max(2g, 2) local qubits (n={n}, g={g})")
    pos = list(range(n))            # logical -> physical
    at = list(range(n))             # physical -> logical
    sch = Schedule(n, g, measured=list(measured) or list(range(n)))
    stage = list(range(L - g, L))
    pending = list(range(len(ops)))
    deferred = []                   # op indices: diagonal ops whose qubits are all global
    cur = []

    def glob(q):
        return pos[q] >= L

    def emit(k):
        kind, tg, slot = ops[k]
        if kind in _DIAG and all(glob(q) for q in tg):
            deferred.append(k)      # rank-constant diagonal: wait until a qubit is local
            return
        cur.append((kind, tuple(pos[q] for q in tg), slot))

    while True:
        blocked = set()
        rest = []
        for k in pending:
            kind, tg, _ = ops[k]
            qs = set(tg)
            if qs & blocked or any(glob(q) for q in exchange_qubits(kind, tg)):
                rest.append(k)
                blocked |= qs
                continue
            emit(k)
        pending = rest
        if not pending or g == 0:
            break
        # victims: local qubits whose next exchange use is furthest (never: +inf);
        # ties prefer qubits already in the staging positions (no SWAP needed)
        nxt = {}
        for idx, k in enumerate(pending):
            for q in exchange_qubits(ops[k][0], ops[k][1]):
                nxt.setdefault(q, idx)
        local = [at[p] for p in range(L)]
        local.sort(key=lambda q: (-nxt.get(q, len(pending) + 1), 0 if pos[q] >= L - g else 1, -pos[q]))
        victims = set(local[:g])
        free = [p for p in stage if at[p] not in victims]
        for q in sorted(victims, key=lambda v: pos[v]):
            if pos[q] >= L - g:
                continue
            p = free.pop(0)
            a, b = pos[q], p
            cur.append(("SWAP", (a, b), -1))
            qa, qb = at[a], at[b]
            at[a], at[b] = qb, qa
            pos[qa], pos[qb] = b, a
        sch.steps.append(("local", cur))
        sch.steps.append(("exchange",))
        cur = []
        for i in range(g):
            s, G = L - g + i, L + i
            qs, qg = at[s], at[G]
            at[s], at[G] = qg, qs
            pos[qs], pos[qg] = G, s
        still = []
        for k in deferred:
            if any(not glob(q) for q in ops[k][1]):
                cur.append((ops[k][0], tuple(pos[q] for q in ops[k][1]), ops[k][2]))
            else:
                still.append(k)
        deferred = still
    if cur:
        sch.steps.append(("local", cur))
    sch.tail = [(ops[k][0], tuple(pos[q] for q in ops[k][1]), ops[k][2]) for k in deferred]
    sch.final_layout = pos
    return sch


def resolve(ops, L: int, rank: int):
    """One rank's local gate list (positions < L): rank-constant controls and
    diagonal qubits resolved (module doc).  No scalar phases arise."""
    out = []

    def bit(p):
        return (rank >> (p - L)) & 1

    for kind, t, slot in ops:
        glob = [p >= L for p in t]
        if not any(glob):
            out.append((kind, t, slot))
        elif kind == "CNOT" and glob[0] and not glob[1]:
            if bit(t[0]):
                out.append(("X", (t[1],), -1))
        elif kind in ("CZ", "CR") and glob.count(True) == 1:
            gp, lp = (t[0], t[1]) if glob[0] else (t[1], t[0])
            if bit(gp):
                out.append(("Z", (lp,), -1) if kind == "CZ" else ("RZ", (lp,), slot))
        else:
            raise ValueError(f"{kind}{t} on a global qubit must have been scheduled local or deferred")
    return out


def tail_phase(sc, rank: int, x_row, theta) -> complex:
    """Scalar phase of this rank from the trailing rank-constant diagonal ops
    (in the kernels' forms: RZ = diag(1, e^{iθ})).  Only the final STATE needs
    it — E and every derivative are independent of these ops."""
    L = sc.L
    x = np.asarray(x_row, np.float64).reshape(-1)
    th = np.asarray(theta, np.float64).reshape(-1)
    ph = 1.0 + 0.0j
    for kind, t, slot in sc.sched.tail:
        if not all((rank >> (p - L)) & 1 for p in t):
            continue
        if kind in ("Z", "CZ"):
            ph *= -1.0
        else:
            a = sc.tape.slot_const[slot]
            for v, c in sc.tape.slot_terms[slot].items():
                a += c * (x[v] if v < sc.n_inputs else th[v - sc.n_inputs])
            ph *= np.exp(1j * a)
    return ph


def readout_weights(sch: Schedule, rank: int):
    """(pos, wk, w0): w(local j) = w0 + Σ wk[i]·bit(j, pos[i]) for this rank
    (outcome bit i = measured[i], qnn.py:108,116)."""
    L = sch.L
    pos, wk, w0 = [], [], 0.0
    for i, q in enumerate(sch.measured):
        P = sch.final_layout[q]
        if P < L:
            pos.append(P)
            wk.append(float(1 << i))
        elif (rank >> (P - L)) & 1:
            w0 += float(1 << i)
    return pos, wk, w0


# ------------------------------------------------------------------------------
class ShardedCircuit:
    """A traced tape (one circuit) scheduled over 2^g ranks, with the adjoint
    gradient spec of the reference's df_p semantics (``tracer.classify``)."""

    def __init__(self, tape: tr.Tape, n_inputs: int, n_params: int, g: int, precision: str = "c128",
                 shift: float = math.pi / 2, grad_scale: float = 0.5, want_x: bool = False, want_p: bool = True):
        if tape.preps:
            raise ConfigError("amplitude-sharded circuits take no state loads")
        self.tape = tape
        self.n, self.g = tape.n_qubits, int(g)
        self.n_inputs, self.n_params = int(n_inputs), int(n_params)
        self.n_vars = self.n_inputs + self.n_params
        self.precision = precision
        self.shift, self.grad_scale = float(shift), float(grad_scale)
        wanted = [want_x] * self.n_inputs + [want_p] * self.n_params
        self.mode, self.vslot, self.factor = tr.classify(tape, self.n_vars, wanted, shift, grad_scale)
        if (self.mode == tr.MODE_TWOPOINT).any():
            raise ConfigError("amplitude-sharded gradients need every differentiated variable in exactly one "
                              "RX/RY/RZ/CR angle (the adjoint reproduces the two-point value there)")
        self.sched = schedule(self.n, self.g, list(tape.ops), tape.measured)
        self._var_of_slot = {int(s): v for v, s in enumerate(self.vslot) if s >= 0}
        self._seg_cache = {}

    @property
    def L(self):
        return self.sched.L

    @property
    def world(self):
        return 1 << self.g

    def segment(self, i: int, rank: int):
        """(tape, grad spec) of segment i for ``rank`` (over the L local qubits)."""
        key = (i, rank)
        if key not in self._seg_cache:
            ops = resolve(self.sched.segments[i], self.L, rank)
            t = tr.Tape(self.L, [0], [(k, tuple(q), int(s) if s is not None else -1) for k, q, s in ops], [],
                        list(self.tape.slot_const), list(self.tape.slot_terms), True)
            mode = np.zeros(self.n_vars, np.int32)
            vslot = np.full(self.n_vars, -1, np.int32)
            factor = np.zeros(self.n_vars)
            for _, _, s in t.ops:
                v = self._var_of_slot.get(s)
                if v is not None and self.mode[v] == tr.MODE_ADJOINT:
                    mode[v], vslot[v], factor[v] = tr.MODE_ADJOINT, s, self.factor[v]
            self._seg_cache[key] = (t, (mode, vslot, factor))
        return self._seg_cache[key]

    def stats(self):
        seg_ops = [len(s) for s in self.sched.segments]
        amp = 16 if self.precision == "c128" else 8
        moved = (self.world - 1) / self.world * (amp << self.L) if self.g else 0.0
        return {"n": self.n, "g": self.g, "ranks": self.world, "local_qubits": self.L,
                "exchanges_forward": self.sched.exchanges, "segments": len(seg_ops), "segment_ops": seg_ops,
                "dropped_trailing_diagonals": self.sched.dropped,
                "exchange_bytes_per_gpu_each_way": moved}


# ------------------------------------------------------------------------------
def execute(sc: ShardedCircuit, ex, x_row, theta, ranks, psi, exchange, allreduce, want_grad: bool, lam=None):
    """Run the schedule for the ranks this process holds.

    ``psi`` / ``lam``: lists of shard buffers (one per entry of ``ranks``);
    ``exchange(bufs) -> bufs`` performs the all-to-all; ``allreduce(v)`` sums
    over all ranks (process group or identity).  ``ex`` provides
    ``seg_forward(sc, i, rank, buf, x, θ)``, ``seg_backward(...) -> jac row``,
    ``readout(sc, rank, buf, lam_out) -> partial E`` and ``zeros_like_jac``.
    Returns (E, grad [d + P] | None, psi)."""
    segs = 0
    for step in sc.sched.steps:
        if step[0] == "local":
            for r, buf in zip(ranks, psi):
                ex.seg_forward(sc, segs, r, buf, x_row, theta)
            segs += 1
        else:
            psi = exchange(psi)
    e = None
    for k, (r, buf) in enumerate(zip(ranks, psi)):
        part = ex.readout(sc, r, buf, lam[k] if want_grad else None)
        e = part if e is None else e + part
    E = allreduce(e)
    if not want_grad:
        return E, None, psi
    jac = ex.zeros_jac(sc)
    for step in reversed(sc.sched.steps):
        if step[0] == "local":
            segs -= 1
            for k, r in enumerate(ranks):
                jac = jac + ex.seg_backward(sc, segs, r, psi[k], lam[k], x_row, theta)
        else:
            psi = exchange(psi)
            lam = exchange(lam)
    return E, allreduce(jac), psi


class GpuExecutor:
    """Segment plans (one per distinct resolved segment) on one CUDA device."""

    def __init__(self, device):
        self.device = device
        self.plans = {}

    def _plan(self, sc, i, rank):
        from . import engine
        tape, grad = sc.segment(i, rank)
        # everything a plan depends on (not the ShardedCircuit's identity)
        key = (engine.tape_key(tape), sc.n_inputs, sc.n_params, sc.precision, tuple(grad[0]), tuple(grad[1]),
               tuple(grad[2]), sc.shift, sc.grad_scale)
        if key not in self.plans:
            import torch
            with torch.cuda.device(self.device):
                self.plans[key] = engine.Plan(tape, sc.n_inputs, sc.n_params, sc.precision, grad, sc.shift,
                                              sc.grad_scale, segment=True)
        return self.plans[key]

    def prepare(self, sc, ranks):
        """Build (JIT) every segment plan up front (outside timed regions)."""
        for i in range(len(sc.sched.segments)):
            for r in ranks:
                self._plan(sc, i, r)

    def seg_forward(self, sc, i, rank, buf, x, theta):
        if sc.segment(i, rank)[0].ops:
            self._plan(sc, i, rank).seg_forward(x, theta, buf)

    def seg_backward(self, sc, i, rank, psi, lam, x, theta):
        if not sc.segment(i, rank)[0].ops:
            return self.zeros_jac(sc)
        return self._plan(sc, i, rank).seg_backward(x, theta, psi, lam)[0]

    def readout(self, sc, rank, buf, lam_out):
        from . import engine
        pos, wk, w0 = readout_weights(sc.sched, rank)
        return engine.shard_readout(buf, sc.L, sc.precision, pos, wk, w0, lam_out)

    def zeros_jac(self, sc):
        import torch
        return torch.zeros(sc.n_vars, dtype=torch.float64, device=self.device)


def _dtype(precision):
    import torch
    return torch.complex128 if precision in ("c128", "complex128") else torch.complex64


def _inputs(sc, x_row, theta, device):
    import torch
    x = torch.as_tensor(np.asarray(x_row, np.float64).reshape(1, -1), device=device)
    if x.shape[1] == 0:
        x = torch.zeros((1, 1), dtype=torch.float64, device=device)
    t = torch.as_tensor(np.asarray(theta, np.float64).reshape(-1), device=device)
    if t.numel() == 0:
        t = torch.zeros(1, dtype=torch.float64, device=device)
    return x.contiguous(), t.contiguous()


def run_nccl(sc: ShardedCircuit, theta, rank: int, world: int, device, x_row=(), want_grad=True, group=None,
             ex: GpuExecutor | None = None):
    """One rank per process (NCCL over NVLink on GPUs, gloo on CPU tests).
    Returns (E, grad [d + P] numpy | None, this rank's final shard)."""
    import torch
    import torch.distributed as dist
    if world != sc.world:
        raise ConfigError(f"schedule is for {sc.world} ranks, world is {world}")
    ex = ex or GpuExecutor(device)
    x, t = _inputs(sc, x_row, theta, device)
    psi = torch.zeros(1 << sc.L, dtype=_dtype(sc.precision), device=device)
    if rank == 0:
        psi[0] = 1.0
    lam = [torch.empty_like(psi)] if want_grad else None
    spare = [torch.empty_like(psi) if sc.sched.exchanges else None]   # all-to-all needs a second buffer

    def exchange(bufs):
        # all g rank bits <-> the top g local bits: contiguous equal chunks
        out = spare[0]
        dist.all_to_all_single(torch.view_as_real(out).reshape(-1), torch.view_as_real(bufs[0]).reshape(-1),
                               group=group)
        spare[0] = bufs[0]
        return [out]

    def allreduce(v):
        if world > 1:
            dist.all_reduce(v, group=group)
        return v

    E, grad, psi_l = execute(sc, ex, x, t, [rank], [psi], exchange, allreduce, want_grad, lam)
    out = psi_l[0]
    if not want_grad and sc.sched.tail:
        out.mul_(complex(tail_phase(sc, rank, x_row, theta)))   # state output only (E is independent)
    return float(E.item()), (grad.cpu().numpy() if grad is not None else None), out


def virtual_exchange(bufs):
    """All ranks in one process: rank r's chunk j <-> rank j's chunk r (in
    place, pairwise block swaps)."""
    import torch
    R = len(bufs)
    views = [b.view(R, -1) for b in bufs]
    tmp = torch.empty_like(views[0][0])
    for r in range(R):
        for j in range(r + 1, R):
            tmp.copy_(views[r][j])
            views[r][j].copy_(views[j][r])
            views[j][r].copy_(tmp)
    return bufs


def run_virtual(sc: ShardedCircuit, theta, device, x_row=(), want_grad=True, ex: GpuExecutor | None = None):
    """All 2^g ranks in this process on one device (rank shards are rows of
    one [R, 2^L] tensor).  Returns (E, grad | None, shards [R, 2^L])."""
    import torch
    ex = ex or GpuExecutor(device)
    R = sc.world
    x, t = _inputs(sc, x_row, theta, device)
    psi = torch.zeros((R, 1 << sc.L), dtype=_dtype(sc.precision), device=device)
    psi[0, 0] = 1.0
    lam = torch.empty_like(psi) if want_grad else None
    E, grad, _ = execute(sc, ex, x, t, list(range(R)), [psi[r] for r in range(R)], virtual_exchange,
                         lambda v: v, want_grad, [lam[r] for r in range(R)] if want_grad else None)
    if not want_grad and sc.sched.tail:
        for r in range(R):
            psi[r].mul_(complex(tail_phase(sc, r, x_row, theta)))
    return float(E.item()), (grad.cpu().numpy() if grad is not None else None), psi


def gather_state(shards, L: int, layout) -> np.ndarray:
    """Logical full state from the rank shards (tests / small n)."""
    full = np.concatenate([np.asarray(s).reshape(-1) for s in shards])
    phys = np.arange(full.size)
    logical = np.zeros_like(phys)
    for q in range(len(layout)):
        logical |= ((phys >> layout[q]) & 1) << q
    out = np.empty_like(full)
    out[logical] = full
    return out
