"""Amplitude sharding of ONE circuit across R = 2^g ranks.

Global index i = (rank << L) | local with L = n - g: the top g index bits
("global qubits") select the rank.  A layout maps logical qubits to physical
bit positions; the schedule is a list of steps:

* ``("local", ops)``   gates whose exchange qubits (targets of non-diagonal
  kinds) sit at local positions.  Controls / diagonal qubits at global
  positions are rank constants, resolved per rank (a CNOT with a global
  control becomes an X or nothing, a CZ/CR/RZ/Z on a global qubit becomes a
  local phase gate or a per-rank scalar phase).
* ``("swap", G, l)``   exchange global position G with local position l: every
  rank trades the half of its shard whose bit l differs from its rank bit with
  partner ``rank ^ (1 << (G - L))`` — NCCL send/recv pairs on GPUs (half the
  shard per swap), a local permutation for virtual ranks.

Per-rank scalar phases accumulate on the host and are applied to the shard
before it is exchanged (they matter once shards interfere) and before the
amplitudes are reported.  The readout adds each rank's partial Σ w|ψ|², where
measured qubits at global positions contribute their rank bit.

``schedule`` is pure host logic; ``run_virtual`` executes it with pluggable
local executors (NumPy oracle on CPU tests, the sm_100a plans on one GPU);
``run_nccl`` runs one rank per process.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_EXCH = {"H": 1, "X": 1, "Y": 1, "RX": 1, "RY": 1}   # exchange on targets[0]


def exchange_qubits(kind, targets):
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
    steps: list = field(default_factory=list)   # ("local", [(kind, targets_phys, angle)]) | ("swap", G, l)
    final_layout: list = field(default_factory=list)   # logical -> physical
    measured: list = field(default_factory=list)

    @property
    def L(self):
        return self.n - self.g


def schedule(n: int, g: int, ops, measured) -> Schedule:
    """ops: [(kind, logical targets, angle)] with concrete angles."""
    L = n - g
    if g < 0 or L < 2:
        raise ValueError("need at least 2 local qubits")
    pos = list(range(n))            # logical -> physical
    at = list(range(n))             # physical -> logical
    sch = Schedule(n, g, measured=list(measured) or list(range(n)))
    cur = []

    def next_use(logical, start):
        # next time the qubit must be local (exchange use); controls and
        # diagonal uses work from a global position
        for k in range(start, len(ops)):
            if logical in exchange_qubits(ops[k][0], ops[k][1]):
                return k
        return len(ops) + 1

    for k, (kind, targets, angle) in enumerate(ops):
        need = [q for q in exchange_qubits(kind, targets) if pos[q] >= L]
        for q in need:
            # bring q local: evict the local position whose logical qubit is
            # needed latest and is not used by this op
            cands = [p for p in range(L) if at[p] not in targets]
            victim = max(cands, key=lambda p: next_use(at[p], k))
            if cur:
                sch.steps.append(("local", cur))
                cur = []
            G = pos[q]
            sch.steps.append(("swap", G, victim))
            lq = at[victim]
            at[victim], at[G] = q, lq
            pos[q], pos[lq] = victim, G
        cur.append((kind, tuple(pos[t] for t in targets), angle))
    if cur:
        sch.steps.append(("local", cur))
    sch.final_layout = pos
    return sch


def resolve_local(ops, L, rank):
    """Per-rank local gate list (positions < L) + scalar phase for this rank.

    Gates on global positions (>= L) are diagonal or controls here (the
    scheduler moved every exchange qubit local)."""
    out, phase = [], 1.0 + 0.0j

    def bit(p):
        return (rank >> (p - L)) & 1

    for kind, t, angle in ops:
        glob = [p >= L for p in t]
        if not any(glob):
            out.append((kind, t, angle))
            continue
        if kind in ("Z", "RZ"):
            b = bit(t[0])
            if kind == "Z":
                phase *= -1.0 if b else 1.0
            else:
                phase *= np.exp((0.5j if b else -0.5j) * angle)
        elif kind == "CNOT":            # global control, local target
            if bit(t[0]):
                out.append(("X", (t[1],), None))
        elif kind in ("CZ", "CR"):
            ph = -1.0 if kind == "CZ" else np.exp(1j * angle)
            if all(glob):
                if bit(t[0]) and bit(t[1]):
                    phase *= ph
            else:
                gp, lp = (t[0], t[1]) if glob[0] else (t[1], t[0])
                if bit(gp):
                    if kind == "CZ":
                        out.append(("Z", (lp,), None))
                    else:
                        # phase e^{iα} on |1> of lp == RZ(α) up to e^{iα/2}
                        out.append(("RZ", (lp,), angle))
                        phase *= np.exp(0.5j * angle)
        else:
            raise ValueError(f"{kind} on a global qubit must have been swapped local")
    return out, phase


def swap_exchange(shards, L, G, l):
    """Virtual-rank global<->local swap: returns new shards (list of arrays)."""
    k = G - L
    R = len(shards)
    new = [s.copy() for s in shards]
    idx = np.arange(1 << L)
    lbit = (idx >> l) & 1
    for r in range(R):
        rb = (r >> k) & 1
        partner = r ^ (1 << k)
        # positions of r whose local bit differs from r's rank bit go to the partner;
        # they come back from the partner's positions whose bit equals r's bit
        sel = lbit != rb
        src = shards[partner]
        # element (r, l with bit l = 1-rb) <- partner element (partner, l with bit l flipped)
        new[r][sel] = src[idx[sel] ^ (1 << l)]
    return new


def readout_partial(shard, L, rank, layout, measured):
    """Σ_l w(rank, l)|ψ(l)|² with outcome bit i = measured[i] (qnn.py:108,116)."""
    p = np.abs(shard) ** 2
    idx = np.arange(p.size)
    w = np.zeros(p.size)
    for i, q in enumerate(measured):
        P = layout[q]
        if P < L:
            w += ((idx >> P) & 1) * float(1 << i)
        elif (rank >> (P - L)) & 1:
            w += float(1 << i)
    return float(w @ p)


def gather_state(shards, L, layout):
    """Logical full state from virtual-rank shards (tests / small n)."""
    n = len(layout)
    full = np.concatenate(shards)
    phys = np.arange(full.size)
    logical = np.zeros_like(phys)
    for q in range(n):
        logical |= ((phys >> layout[q]) & 1) << q
    out = np.empty_like(full)
    out[logical] = full
    return out


def run_virtual(sch: Schedule, apply_local, initial=None):
    """Execute a schedule over 2^g virtual ranks in one process.

    ``apply_local(shard, ops) -> shard`` runs a local gate list on one shard
    (positions < L).  Returns (shards, E)."""
    L, R = sch.L, 1 << sch.g
    if initial is None:
        shards = [np.zeros(1 << L, dtype=np.complex128) for _ in range(R)]
        shards[0][0] = 1.0
    else:
        full = np.asarray(initial, dtype=np.complex128)
        shards = [full[r << L:(r + 1) << L].copy() for r in range(R)]
    phases = [1.0 + 0.0j] * R
    for step in sch.steps:
        if step[0] == "local":
            for r in range(R):
                ops, ph = resolve_local(step[1], L, r)
                if ops:
                    shards[r] = apply_local(shards[r], ops)
                phases[r] *= ph
        else:
            shards = [s * ph for s, ph in zip(shards, phases)]
            phases = [1.0 + 0.0j] * R
            shards = swap_exchange(shards, L, step[1], step[2])
    shards = [s * ph for s, ph in zip(shards, phases)]
    E = sum(readout_partial(shards[r], L, r, sch.final_layout, sch.measured) for r in range(R))
    return shards, E


# ---------------------------------------------------------------------------
# GPU execution
def gpu_apply_local(L, precision="c128"):
    """Local executor on the current CUDA device: the shard's gate list runs as
    a plan with its angles as per-call inputs, starting from the shard."""
    from . import engine

    def apply_local(shard, ops):
        from .qsim import Circuit, GateOp
        c = Circuit(L)
        for kind, t, a in ops:
            c.add(GateOp(kind, t, a))
        return engine.final_states([c], precision, init=shard)[0]
    return apply_local


def gpu_apply_local_dev(L, precision="c128"):
    """Device-resident local executor for ``run_nccl``: the rank's complex128
    CUDA shard goes through the plan as its initial state and the result stays
    on the device (plans are cached per local-segment structure)."""
    from . import engine

    def apply_local_dev(shard, ops):
        from .qsim import Circuit, GateOp
        c = Circuit(L)
        for kind, t, a in ops:
            c.add(GateOp(kind, t, a))
        return engine.final_state_device(c, shard, precision)
    return apply_local_dev


def _pack_half(shard, l, bit):
    """Elements of a device shard whose local bit l == bit, in index order."""
    import torch
    n = shard.shape[0]
    v = shard.view(n >> (l + 1), 2, 1 << l)
    return v[:, bit, :].reshape(-1)


def run_nccl(sch: Schedule, apply_local_dev, rank: int, world: int, device, group=None):
    """One rank per process.  ``apply_local_dev(shard_tensor, ops) -> tensor``
    runs a local gate list on this rank's complex128 device shard; swaps are
    pairwise NCCL send/recv of half a shard.  Returns (shard, E)."""
    import torch
    import torch.distributed as dist
    L = sch.L
    if (1 << sch.g) != world:
        raise ValueError(f"schedule is for {1 << sch.g} ranks, world is {world}")
    shard = torch.zeros(1 << L, dtype=torch.complex128, device=device)
    if rank == 0:
        shard[0] = 1.0
    phase = 1.0 + 0.0j
    for step in sch.steps:
        if step[0] == "local":
            ops, ph = resolve_local(step[1], L, rank)
            if ops:
                shard = apply_local_dev(shard, ops)
            phase *= ph
        else:
            G, l = step[1], step[2]
            k = G - L
            rb = (rank >> k) & 1
            partner = rank ^ (1 << k)
            shard = shard * phase
            phase = 1.0 + 0.0j
            send = _pack_half(shard, l, 1 - rb).contiguous()
            recv = torch.empty_like(send)
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, send, partner, group),
                                           dist.P2POp(dist.irecv, recv, partner, group)])
            for r in reqs:
                r.wait()
            # our elements with bit l = 1-rb are replaced by the partner's with bit l = rb
            v = shard.view((1 << L) >> (l + 1), 2, 1 << l)
            v[:, 1 - rb, :] = recv.view((1 << L) >> (l + 1), 1 << l)
    shard = shard * phase
    p = shard.real ** 2 + shard.imag ** 2
    idx = torch.arange(1 << L, device=device)
    w = torch.zeros(1 << L, dtype=torch.float64, device=device)
    for i, q in enumerate(sch.measured):
        P = sch.final_layout[q]
        if P < L:
            w += ((idx >> P) & 1).double() * float(1 << i)
        elif (rank >> (P - L)) & 1:
            w += float(1 << i)
    e = (w * p).sum().reshape(1)
    dist.all_reduce(e, group=group)
    return shard, float(e.item())
