"""Execution engine: tape -> ``hq_plan`` -> sm_100a kernels.

``Plan`` owns one C-ABI plan handle (``include/hq.h``) and runs it on torch
CUDA tensors (PyTorch is used for device memory and the current stream only).
``run_batch`` is what ``QuantumLayer.forward`` calls: it traces the builder
(``tracer.py``), picks or builds the plan, and returns per-sample expectations
and, when gradients are wanted, the per-sample jacobian rows the reference's
``df_x`` / ``df_p`` closures would produce at upstream 1 (``qnn.py:136-153``).

Builders that are not provably affine / batch-invariant run through
``run_per_sample``: the builder is called per sample and per shifted value,
exactly like the reference (``qnn.py:35-52``), and the resulting circuits are
simulated in batches grouped by structure — still on the GPU, with every angle
carried as a per-circuit input.
"""

from __future__ import annotations

import ctypes
import math
import os
from collections import OrderedDict

import numpy as np

from . import _native as nat
from . import tracer as tr
from .errors import CircuitError, ConfigError, DimensionError, EncodingError, NativeError

_PREC = {"c64": nat.HQ_C64, "c128": nat.HQ_C128, "complex64": nat.HQ_C64,
         "complex128": nat.HQ_C128}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: this package has no CPU execution path")
    return torch


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _arr(a, dt):
    a = np.ascontiguousarray(np.asarray(a, dtype=dt))
    return a, (a.ctypes.data if a.size else None)


class Plan:
    """One immutable device plan for a tape + gradient spec + precision."""

    def __init__(self, tape: tr.Tape, n_inputs: int, n_params: int, precision: str = "c128",
                 grad=None, shift: float = math.pi / 2, grad_scale: float = 0.5, segment: bool = False):
        if precision not in _PREC:
            raise ConfigError(f"precision must be c64 or c128, got {precision!r}")
        L = nat.lib()
        torch = _torch()
        self.device = torch.cuda.current_device()
        self.n_qubits = tape.n_qubits
        self.n_inputs, self.n_params = int(n_inputs), int(n_params)
        self.n_vars = self.n_inputs + self.n_params
        self.precision = precision
        ops = (nat.HqOp * max(1, len(tape.ops)))()
        for i, (kind, targets, slot) in enumerate(tape.ops):
            if kind == "STATEPREP":
                ops[i] = nat.HqOp(11, slot, -1, -1)
            elif len(targets) == 2:
                ops[i] = nat.HqOp(nat.KIND_CODE[kind], targets[0], targets[1], slot)
            else:
                ops[i] = nat.HqOp(nat.KIND_CODE[kind], targets[0], -1, slot)
        nnz_ptr = [0]
        var, coef = [], []
        for terms in tape.slot_terms:
            for v in sorted(terms):
                var.append(v)
                coef.append(terms[v])
            nnz_ptr.append(len(var))
        keep = []

        def a(x, dt):
            arr, p = _arr(x, dt)
            keep.append(arr)
            return p

        d = nat.HqPlanDesc()
        d.n_qubits = tape.n_qubits
        d.precision = _PREC[precision]
        d.n_ops = len(tape.ops)
        d.ops = ctypes.cast(ops, ctypes.c_void_p)
        d.n_slots = len(tape.slot_const)
        d.slot_const = a(tape.slot_const, np.float64)
        d.slot_ptr = a(nnz_ptr, np.int32)
        d.slot_var = a(var, np.int32)
        d.slot_coef = a(coef, np.float64)
        d.n_inputs, d.n_params = self.n_inputs, self.n_params
        d.n_measured = len(tape.measured)
        d.measured = a(tape.measured, np.int32)
        d.n_preps = len(tape.preps)
        pq, pp, ps0, pl = [], [0], [], []
        for qubits, first, count in tape.preps:
            pq.extend(qubits)
            pp.append(len(pq))
            ps0.append(first)
            pl.append(count)
        d.prep_ptr = a(pp, np.int32)
        d.prep_qubits = a(pq, np.int32)
        d.prep_slot0 = a(ps0, np.int32)
        d.prep_len = a(pl, np.int32)
        if grad is not None:
            mode, vslot, factor = grad
            d.grad_mode = a(mode, np.int32)
            d.grad_slot = a(vslot, np.int32)
            d.grad_factor = a(factor, np.float64)
            self.grad_mode = np.asarray(mode)
        else:
            self.grad_mode = np.zeros(self.n_vars, np.int32)
        d.shift, d.grad_scale = float(shift), float(grad_scale)
        h = ctypes.c_void_p()
        self.segment = bool(segment)
        create = L.hq_plan_create_segment if segment else L.hq_plan_create
        nat.check(create(ctypes.byref(d), ctypes.byref(h)), "plan")
        self._h = h
        self._lib = L
        self.description = L.hq_plan_describe(h).decode()
        self.measured = list(tape.measured) or list(range(tape.n_qubits))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.hq_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def stats(self, B, want_jac=True) -> dict:
        st = nat.HqStats()
        nat.check(self._lib.hq_stats(self._h, int(B), nat.HQ_WANT_JAC if want_jac else 0,
                                     ctypes.byref(st)), "stats")
        return {f: getattr(st, f) for f, _ in nat.HqStats._fields_}

    def profile(self, enable: bool) -> None:
        nat.check(self._lib.hq_profile_enable(self._h, 1 if enable else 0), "profile")

    def profile_read(self) -> dict:
        r = nat.HqProfile()
        nat.check(self._lib.hq_profile_read(self._h, ctypes.byref(r)), "profile")
        return {k: {"ms": r.ms[i], "launches": r.launches[i], "bytes": r.bytes[i]}
                for i, k in enumerate(nat.K_CLASSES)}

    def _on_device(self, *tensors):
        """Every device operand must live on the plan's GPU (kernels and the
        stream are that device's); -> the plan's current stream handle."""
        torch = _torch()
        for t in tensors:
            if t is not None and (t.device.type != "cuda" or t.device.index != self.device):
                raise DimensionError(f"tensor on {t.device} but the plan runs on cuda:{self.device}")
        return torch.cuda.current_stream(self.device).cuda_stream

    def _ws(self, B, flags):
        torch = _torch()
        n = int(self._lib.hq_workspace_bytes(self._h, int(B), int(flags)))
        return torch.empty(max(n, 256), dtype=torch.uint8, device=f"cuda:{self.device}"), n

    def forward(self, x, theta, want_jac: bool):
        """x: cuda f64 [B, ldx]; theta: cuda f64 [P] -> (out [B], jac [B, nv] | None)."""
        torch = _torch()
        B = int(x.shape[0])
        dev = f"cuda:{self.device}"
        out = torch.empty(B, dtype=torch.float64, device=dev)
        jac = torch.empty((B, self.n_vars), dtype=torch.float64, device=dev) if want_jac else None
        flags = nat.HQ_WANT_JAC if want_jac else 0
        st = self._on_device(x, theta)
        ws, nbytes = self._ws(B, flags)
        with _torch().cuda.device(self.device):
            nat.check(self._lib.hq_forward(self._h, _ptr(x), int(x.stride(0)) if x.dim() == 2 else 0,
                                           _ptr(theta), B, flags, _ptr(out), _ptr(jac), _ptr(ws),
                                           ws.numel(), st), "forward")
        return out, jac

    def vjp(self, jac, upstream, want_x=True, want_theta=True):
        torch = _torch()
        B = int(jac.shape[0])
        dev = jac.device
        gx = torch.empty((B, self.n_inputs), dtype=torch.float64, device=dev) if want_x else None
        gt = torch.empty(self.n_params, dtype=torch.float64, device=dev) if want_theta else None
        st = self._on_device(jac, upstream)
        with _torch().cuda.device(self.device):
            nat.check(self._lib.hq_vjp(self._h, _ptr(jac), _ptr(upstream), B, _ptr(gx), _ptr(gt), st),
                      "vjp")
        return gx, gt

    def state(self, x, theta, init=None):
        torch = _torch()
        B = int(x.shape[0]) if x is not None else 1
        dev = f"cuda:{self.device}"
        st_out = torch.empty((B, 1 << self.n_qubits, 2), dtype=torch.float64, device=dev)
        st = self._on_device(x, theta, init)
        ws, _ = self._ws(B, 0)
        rows = 0 if init is None else int(init.shape[0])
        with _torch().cuda.device(self.device):
            nat.check(self._lib.hq_state(self._h, _ptr(x), int(x.stride(0)) if x is not None else 0,
                                         _ptr(theta), B, _ptr(init), rows, _ptr(st_out), _ptr(ws),
                                         ws.numel(), st), "state")
        return st_out


    # -- segment plans (amplitude-sharded execution, shard.py) -------------------
    def _seg_ws(self, B):
        torch = _torch()
        n = int(self._lib.hq_seg_workspace_bytes(self._h, int(B)))
        return torch.empty(max(n, 256), dtype=torch.uint8, device=f"cuda:{self.device}")

    def _seg_check(self, psi, B):
        amp = 16 if self.precision in ("c128", "complex128") else 8
        if not psi.is_contiguous() or psi.numel() * psi.element_size() != B * amp << self.n_qubits:
            raise DimensionError(f"state rows must be contiguous [{B}, 2^{self.n_qubits}] amplitudes")

    def seg_forward(self, x, theta, psi):
        """psi (cuda, [B, 2^n] amplitudes of the plan's precision) <- U psi, in place."""
        if not self.segment:
            raise ConfigError("seg_forward needs a segment plan")
        B = int(x.shape[0])
        self._seg_check(psi, B)
        st = self._on_device(x, theta, psi)
        ws = self._seg_ws(B)
        with _torch().cuda.device(self.device):
            nat.check(self._lib.hq_seg_forward(self._h, _ptr(x), int(x.stride(0)), _ptr(theta), B, _ptr(psi),
                                               _ptr(ws), ws.numel(), st), "seg_forward")

    def seg_backward(self, x, theta, psi, lam):
        """psi <- U^-1 psi, lam <- U^† lam in place; -> jac [B, n_vars] (this segment's dots)."""
        if not self.segment:
            raise ConfigError("seg_backward needs a segment plan")
        torch = _torch()
        B = int(x.shape[0])
        self._seg_check(psi, B)
        self._seg_check(lam, B)
        st = self._on_device(x, theta, psi, lam)
        jac = torch.empty((B, self.n_vars), dtype=torch.float64, device=f"cuda:{self.device}")
        ws = self._seg_ws(B)
        with _torch().cuda.device(self.device):
            nat.check(self._lib.hq_seg_backward(self._h, _ptr(x), int(x.stride(0)), _ptr(theta), B, _ptr(psi),
                                                _ptr(lam), _ptr(jac), _ptr(ws), ws.numel(), st), "seg_backward")
        return jac

    def noisy(self, x, theta, sites, shots: int, seed: int, want_jac: bool, want_counts: bool = False):
        """NOISY trajectories (hq_noisy): -> (E [B], jac [B, nv] | None, counts [B, 2^m] | None)."""
        torch = _torch()
        B = int(x.shape[0])
        dev = f"cuda:{self.device}"
        flags = nat.HQ_WANT_JAC if want_jac else 0
        n_sites = len(sites)
        arr = (nat.HqNoiseSite * max(1, n_sites))()
        for i, (op, q, code, prm) in enumerate(sites):
            arr[i] = nat.HqNoiseSite(op, q, code, prm)
        nb = int(self._lib.hq_noisy_workspace_bytes(self._h, B, flags, n_sites))
        ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
        out = torch.empty(B, dtype=torch.float64, device=dev)
        jac = torch.empty((B, self.n_vars), dtype=torch.float64, device=dev) if want_jac else None
        m = len(self.measured)
        counts = torch.empty((B, 1 << m), dtype=torch.int64, device=dev) if want_counts else None
        st = self._on_device(x, theta)
        with _torch().cuda.device(self.device):
            nat.check(self._lib.hq_noisy(self._h, _ptr(x), int(x.stride(0)) if x.dim() == 2 else 0, _ptr(theta), B,
                                         flags, ctypes.cast(arr, ctypes.c_void_p), n_sites, int(shots),
                                         ctypes.c_uint64(int(seed) & ((1 << 64) - 1)), _ptr(out), _ptr(jac),
                                         _ptr(counts), _ptr(ws), ws.numel(), st), "noisy")
        return out, jac, counts


# ------------------------------------------------------------------------------
def tape_key(tape: tr.Tape):
    return (tape.structure_key(), tuple(tape.slot_const),
            tuple(tuple(sorted(t.items())) for t in tape.slot_terms))


class PlanCache:
    """Small LRU of plans keyed by tape + gradient spec + precision + device."""

    def __init__(self, size: int = 8):
        self.size = size
        self._d: OrderedDict = OrderedDict()

    def get(self, tape, n_inputs, n_params, precision, grad, shift, grad_scale):
        torch = _torch()
        gkey = None if grad is None else (tuple(grad[0]), tuple(grad[1]), tuple(grad[2]))
        key = (tape_key(tape), n_inputs, n_params, precision, gkey, shift, grad_scale,
               torch.cuda.current_device())
        plan = self._d.get(key)
        if plan is None:
            plan = Plan(tape, n_inputs, n_params, precision, grad, shift, grad_scale)
            self._d[key] = plan
            while len(self._d) > self.size:
                self._d.popitem(last=False)
        else:
            self._d.move_to_end(key)
        return plan


_global_cache = PlanCache(32)


def _check_preps(tape: tr.Tape, x: np.ndarray, theta: np.ndarray):
    """Host check of the reference's per-sample embedding errors (templates.py:71-75)."""
    for _, first, count in tape.preps:
        vals = np.zeros((x.shape[0], count))
        for k in range(count):
            s = first + k
            col = np.full(x.shape[0], tape.slot_const[s])
            for v, c in tape.slot_terms[s].items():
                col = col + c * (x[:, v] if v < x.shape[1] else theta[v - x.shape[1]])
            vals[:, k] = col
        if not np.all(np.isfinite(vals)):
            raise EncodingError("amplitude embedding needs a finite nonzero vector")
        if np.any(np.linalg.norm(vals, axis=1) == 0.0):
            raise EncodingError("cannot embed the zero vector")


def _check_finite(tape: tr.Tape, x: np.ndarray, theta: np.ndarray):
    """The reference raises CircuitError('<KIND> requires one finite angle')
    when it builds the GateOp of a sample whose angle is not finite
    (qsim.py:60-63); the traced path only builds probe rows, so check every
    row's gate angles here (state-load values: ``_check_preps``)."""
    d = x.shape[1]
    used = sorted({v for kind, _, slot in tape.ops if kind != "STATEPREP" and slot >= 0
                   for v in tape.slot_terms[slot]})
    ucols = [v for v in used if v < d]
    bad_rows = np.zeros(x.shape[0], bool)
    if ucols:
        bad_rows = ~np.isfinite(x[:, ucols]).all(axis=1)
    bad_theta = any(v >= d and not np.isfinite(theta[v - d]) for v in used)
    if not bad_rows.any() and not bad_theta:
        return
    row = int(np.argmax(bad_rows)) if bad_rows.any() else 0
    with np.errstate(all="ignore"):
        for kind, _, slot in tape.ops:
            if kind == "STATEPREP" or slot < 0:
                continue
            val = tape.slot_const[slot]
            for v, c in tape.slot_terms[slot].items():
                val = val + c * (x[row, v] if v < d else theta[v - d])
            if not np.isfinite(val):
                raise CircuitError(f"{kind} requires one finite angle")


def run_batch(builder, xd: np.ndarray, pd: np.ndarray, want_x: bool, want_p: bool,
              precision: str = "c128", shift: float = math.pi / 2, grad_scale: float = 0.5,
              cache: PlanCache | None = None, light_cone: bool = False):
    """Host-boundary entry: numpy in, numpy out.

    Returns ``(out [B], jac [B, d+P] | None, info)``.
    """
    B, d = xd.shape
    P = pd.shape[0]
    tape, ok = tr.trace(builder, xd, pd)
    if not ok:
        return run_per_sample(builder, xd, pd, want_x, want_p, precision, shift, grad_scale)
    torch = _torch()
    _check_finite(tape, xd, pd)
    if tape.preps:
        _check_preps(tape, xd, pd)
    if light_cone or os.environ.get("HQ_LIGHTCONE") == "1":
        # opt-in: drop gates outside the readout's backward light cone (identical E and gradients)
        tape = tr.light_cone(tape) or tape
    wanted = [want_x] * d + [want_p] * P
    grad = tr.classify(tape, d + P, wanted, shift, grad_scale) if (want_x or want_p) else None
    cache = cache or _global_cache
    try:
        plan = cache.get(tape, d, P, precision, grad, shift, grad_scale)
    except CircuitError as exc:
        if "no native lowering" in str(exc):
            return run_per_sample(builder, xd, pd, want_x, want_p, precision, shift, grad_scale)
        raise
    dev = f"cuda:{plan.device}"
    x_t = torch.from_numpy(np.ascontiguousarray(xd)).to(dev)
    p_t = torch.from_numpy(np.ascontiguousarray(pd)).to(dev)
    out, jac = plan.forward(x_t, p_t, grad is not None)
    out_h = out.cpu().numpy()
    return out_h, jac, {"plan": plan, "path": "traced"}


# ------------------------------------------------------------------------------
def _circuit_rows(circuits):
    """Group plain-float circuits by structure -> {key: (tape, [(idx, angles)])}."""
    groups = {}
    for idx, c in enumerate(circuits):
        tr.check_circuit(c)
        measured = [int(q) for q in c.measured_qubits] or list(range(c.n_qubits))
        ops, angles = [], []
        for op in c.ops:
            if op.kind == "STATEPREP":
                raise CircuitError("state loads only exist in traced builders")
            if op.angle is None:
                ops.append((op.kind, tuple(op.targets), -1))
            else:
                ops.append((op.kind, tuple(op.targets), len(angles)))
                angles.append(float(op.angle))
        key = (int(c.n_qubits), tuple(measured), tuple(ops))
        if key not in groups:
            tape = tr.Tape(int(c.n_qubits), measured, ops, [])
            tape.slot_const = [0.0] * len(angles)
            tape.slot_terms = [{s: 1.0} for s in range(len(angles))]
            groups[key] = (tape, [])
        groups[key][1].append((idx, angles))
    return groups


def evaluate_circuits(circuits, precision: str = "c128") -> np.ndarray:
    """EXACT_PROB readout of each circuit (angles carried as per-circuit inputs)."""
    torch = _torch()
    out = np.empty(len(circuits), dtype=np.float64)
    for tape, rows in _circuit_rows(circuits).values():
        A = len(tape.slot_const)
        plan = _global_cache.get(tape, A, 0, precision, None, math.pi / 2, 0.5)
        x = np.array([r[1] for r in rows], dtype=np.float64).reshape(len(rows), A)
        dev = f"cuda:{plan.device}"
        xt = torch.from_numpy(x).to(dev) if A else torch.zeros((len(rows), 1), dtype=torch.float64, device=dev)
        pt = torch.zeros(1, dtype=torch.float64, device=dev)
        e, _ = plan.forward(xt, pt, False)
        out[[r[0] for r in rows]] = e.cpu().numpy()
    return out


def final_states(circuits, precision: str = "c128", init=None) -> list:
    """Final amplitudes (complex128 numpy) of each circuit."""
    torch = _torch()
    res = [None] * len(circuits)
    for tape, rows in _circuit_rows(circuits).values():
        A = len(tape.slot_const)
        plan = _global_cache.get(tape, A, 0, precision, None, math.pi / 2, 0.5)
        dev = f"cuda:{plan.device}"
        x = np.array([r[1] for r in rows], dtype=np.float64).reshape(len(rows), A)
        xt = torch.from_numpy(x).to(dev) if A else torch.zeros((len(rows), 1), dtype=torch.float64, device=dev)
        pt = torch.zeros(1, dtype=torch.float64, device=dev)
        it = None
        if init is not None:
            z = np.ascontiguousarray(np.asarray(init, np.complex128).reshape(1, -1))
            it = torch.from_numpy(z.view(np.float64).reshape(1, -1, 2)).to(dev)
        s = plan.state(xt, pt, it).cpu().numpy()
        for k, (idx, _) in enumerate(rows):
            res[idx] = s[k, :, 0] + 1j * s[k, :, 1]
    return res


def final_state_device(circuit, init=None, precision: str = "c128"):
    """Device-resident final amplitudes of one concrete circuit: ``init`` a
    complex128 CUDA vector [2^n] (or None for |0…0⟩) -> complex128 CUDA [2^n].
    No host round trip (the amplitude-sharded executor's local segments)."""
    torch = _torch()
    (tape, rows), = _circuit_rows([circuit]).values()
    A = len(tape.slot_const)
    plan = _global_cache.get(tape, A, 0, precision, None, math.pi / 2, 0.5)
    dev = init.device if init is not None else torch.device(f"cuda:{plan.device}")
    x = (torch.tensor([rows[0][1]], dtype=torch.float64, device=dev) if A
         else torch.zeros((1, 1), dtype=torch.float64, device=dev))
    pt = torch.zeros(1, dtype=torch.float64, device=dev)
    it = None
    if init is not None:
        if init.dtype != torch.complex128 or init.numel() != (1 << tape.n_qubits):
            raise DimensionError("init must be a complex128 vector of 2^n amplitudes")
        it = torch.view_as_real(init.contiguous()).reshape(1, -1, 2)
    return torch.view_as_complex(plan.state(x, pt, it)[0])


def simulate_circuit(circuit, init=None, precision: str = "c128") -> np.ndarray:
    return final_states([circuit], precision, init)[0]


def run_per_sample(builder, xd, pd, want_x, want_p, precision, shift, grad_scale):
    """The reference's own evaluation pattern, with the simulations batched on GPU.

    One builder call per sample and per shifted value (qnn.py:35-52,131-153);
    all resulting circuits are simulated together.
    """
    from .qnn import build_circuit
    B, d = xd.shape
    P = pd.shape[0]
    circuits, index = [], []
    for i in range(B):
        circuits.append(build_circuit(builder, xd[i], pd))
        index.append(("out", i, -1, 0))
    for i in range(B):
        if want_x:
            for j in range(d):
                for sgn in (1, -1):
                    v = xd[i].copy()
                    v[j] = xd[i, j] + sgn * shift
                    circuits.append(build_circuit(builder, v, pd))
                    index.append(("x", i, j, sgn))
        if want_p:
            for j in range(P):
                for sgn in (1, -1):
                    v = pd.copy()
                    v[j] = pd[j] + sgn * shift
                    circuits.append(build_circuit(builder, xd[i], v))
                    index.append(("p", i, j, sgn))
    e = evaluate_circuits(circuits, precision)
    out = e[:B].copy()
    jac = None
    if want_x or want_p:
        jac = np.zeros((B, d + P))
        k = B
        while k < len(index):
            kind, i, j, _ = index[k]
            col = j if kind == "x" else d + j
            jac[i, col] = (e[k] - e[k + 1]) * grad_scale
            k += 2
        torch = _torch()
        jac = torch.from_numpy(jac).to(f"cuda:{torch.cuda.current_device()}")
    return out, jac, {"plan": None, "path": "per_sample"}


# ------------------------------------------------------------------------------
# SHOT_SAMPLING (qsim.py:222-248): device sampling of final states
def shard_readout(psi, n_local: int, precision: str, pos, wk, w0: float, lam=None):
    """This rank's EXACT_PROB partial Σ_j w(j)|psi_j|² (device f64 [1]) and,
    optionally, lam <- w·psi (hq_shard_readout)."""
    torch = _torch()
    L = nat.lib()
    k = len(pos)
    pa = (ctypes.c_int32 * max(k, 1))(*[int(p) for p in pos])
    wa = (ctypes.c_double * max(k, 1))(*[float(w) for w in wk])
    e = torch.empty(1, dtype=torch.float64, device=psi.device)
    ws = torch.empty(int(L.hq_shard_readout_workspace_bytes()), dtype=torch.uint8, device=psi.device)
    with torch.cuda.device(psi.device):
        nat.check(L.hq_shard_readout(_ptr(psi), _PREC[precision], int(n_local), pa, wa, k, float(w0), _ptr(e),
                                     _ptr(lam), _ptr(ws), ws.numel(),
                                     torch.cuda.current_stream(psi.device).cuda_stream), "shard_readout")
    return e


def marginal_probabilities(states, n_qubits: int, measured):
    """states: cuda f64 [rows, 2^n, 2] -> cuda f64 [rows, 2^m] (hq_marginal;
    outcome bit i = measured[i], qsim.py:194-211)."""
    torch = _torch()
    L = nat.lib()
    rows = int(states.shape[0])
    m = len(measured)
    meas = (ctypes.c_int32 * max(m, 1))(*[int(q) for q in measured])
    out = torch.empty((rows, 1 << m), dtype=torch.float64, device=states.device)
    nb = int(L.hq_marginal_workspace_bytes(rows, n_qubits, m))
    ws = torch.empty(nb, dtype=torch.uint8, device=states.device)
    st = states.contiguous()
    with torch.cuda.device(states.device):
        nat.check(L.hq_marginal(_ptr(st), rows, int(n_qubits), meas, m, _ptr(out), _ptr(ws), nb,
                                torch.cuda.current_stream(states.device).cuda_stream), "marginal")
    return out


def sample_states(states, n_qubits: int, measured, shots: int, seed: int, want_counts: bool = False):
    """states: cuda f64 [rows, 2^n, 2] -> (expectation [rows] cuda, counts [rows, 2^m] | None)."""
    torch = _torch()
    L = nat.lib()
    rows = int(states.shape[0])
    m = len(measured)
    meas = (ctypes.c_int32 * m)(*[int(q) for q in measured])
    dev = states.device
    E = torch.empty(rows, dtype=torch.float64, device=dev)
    counts = torch.empty((rows, 1 << m), dtype=torch.int64, device=dev) if want_counts else None
    nb = int(L.hq_sample_workspace_bytes(rows, n_qubits, m))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    status = L.hq_sample(_ptr(states.contiguous()), rows, n_qubits, meas, m, int(shots), int(seed) & (2**64 - 1),
                         _ptr(counts), _ptr(E), _ptr(ws), nb, st)
    nat.check(status, "sample")
    return E, counts


def shot_uniforms(seed: int, shot0: int, count: int):
    torch = _torch()
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    nat.check(nat.lib().hq_shot_uniforms(int(seed), int(shot0), int(count), _ptr(out),
                                         torch.cuda.current_stream().cuda_stream), "uniforms")
    return out


def run_batch_shots(builder, xd, pd, want_x, want_p, shots, seed, precision="c128", shift=math.pi / 2,
                    grad_scale=0.5, measured_override=None, counts_outcome=None, row_budget_bytes=2 << 30):
    """Reference SHOT_SAMPLING semantics on device: every evaluation (base rows
    and the two-point shifted ones) samples ``shots`` outcomes with the same
    seed (qnn.py:117-118, 35-52).  Params ride along as extra per-row inputs so
    shifted-θ rows are ordinary rows of one plan.

    Returns (E [B] numpy, jac [B, d+P] cuda | None); with ``counts_outcome`` the
    value is counts[outcome]/shots instead of the mean outcome (QAELayer)."""
    torch = _torch()
    B, d = xd.shape
    P = pd.shape[0]
    tape, ok = tr.trace(builder, xd, pd)
    if ok:
        _check_finite(tape, xd, pd)
    if ok and tape.preps:
        _check_preps(tape, xd, pd)
    ext = np.hstack([xd, np.broadcast_to(pd, (B, P))])
    rows = [ext]
    index = []
    if want_x or want_p:
        for j in range(d + P):
            if (j < d and not want_x) or (j >= d and not want_p):
                continue
            for sgn in (1.0, -1.0):
                r = ext.copy()
                r[:, j] = ext[:, j] + sgn * shift
                rows.append(r)
                index.append((j, sgn))
    allrows = np.concatenate(rows)
    measured = measured_override or (tape.measured if ok else None)
    if not ok:
        # per-circuit path (data-dependent / non-affine builders)
        from .qnn import build_circuit
        circuits = [build_circuit(builder, r[:d], r[d:]) for r in allrows]
        vals = []
        for c in circuits:
            amps = simulate_circuit(c, None, precision)
            stt = torch.from_numpy(np.stack([amps.real, amps.imag], -1)[None]).to("cuda")
            meas = measured_override or ([int(q) for q in c.measured_qubits] or list(range(c.n_qubits)))
            E, cnt = sample_states(stt, c.n_qubits, meas, shots, seed, counts_outcome is not None)
            vals.append(float((cnt[0, counts_outcome].double() / shots).item()) if counts_outcome is not None
                        else float(E.item()))
        vals = np.array(vals)
    else:
        plan = _global_cache.get(tape, d + P, 0, precision, None, shift, grad_scale)
        n = tape.n_qubits
        per = max(1, int(row_budget_bytes // (16 << n)))
        vals = np.empty(allrows.shape[0])
        pt = torch.zeros(1, dtype=torch.float64, device=f"cuda:{plan.device}")
        for r0 in range(0, allrows.shape[0], per):
            chunk = torch.from_numpy(np.ascontiguousarray(allrows[r0:r0 + per])).to(f"cuda:{plan.device}")
            stt = plan.state(chunk, pt)
            E, cnt = sample_states(stt, n, measured, shots, seed, counts_outcome is not None)
            v = (cnt[:, counts_outcome].double() / shots) if counts_outcome is not None else E
            vals[r0:r0 + chunk.shape[0]] = v.cpu().numpy()
    out = vals[:B]
    jac = None
    if index:
        J = np.zeros((B, d + P))
        for k in range(0, len(index), 2):
            j = index[k][0]
            ep = vals[B * (1 + k):B * (2 + k)]
            em = vals[B * (2 + k):B * (3 + k)]
            J[:, j] = (ep - em) * grad_scale
        jac = torch.from_numpy(J).to("cuda")
    return out, jac


# ------------------------------------------------------------------------------
# NOISY machine type (noise.py, qnn.py:109-111,157-166)
def _twopoint_spec(nv: int, wanted):
    return ([2 if w else 0 for w in wanted], [-1] * nv, [0.0] * nv)


def run_batch_noisy(builder, xd, pd, want_x, want_p, noise, shots, seed, shift=math.pi / 2,
                    grad_scale=0.5):
    """Per-shot noise trajectories for every sample and every shifted
    evaluation (same seed, same per-shot streams: qnn.py:35-52,109-111).
    Returns (E [B] numpy, jac [B, d+P] cuda | None)."""
    from .noise import noise_sites
    torch = _torch()
    B, d = xd.shape
    P = pd.shape[0]
    want = (want_x and d > 0) or (want_p and P > 0)
    tape, ok = tr.trace(builder, xd, pd)
    if ok:
        _check_finite(tape, xd, pd)
    if ok and not tape.preps:
        wanted = [want_x] * d + [want_p] * P
        spec = _twopoint_spec(d + P, wanted) if want else None
        plan = _global_cache.get(tape, d, P, "c128", spec, shift, grad_scale)
        dev = f"cuda:{plan.device}"
        xt = torch.from_numpy(xd).to(dev) if d else torch.zeros((B, 1), dtype=torch.float64, device=dev)
        pt = torch.from_numpy(pd).to(dev) if P else torch.zeros(1, dtype=torch.float64, device=dev)
        e, jac, _ = plan.noisy(xt, pt, noise_sites(tape.ops, noise), shots, seed, want)
        return e.cpu().numpy(), jac
    # per-circuit path (data-dependent builders / state loads): every base and
    # shifted evaluation is a concrete circuit; circuits sharing a structure
    # share one plan with their angles as per-row inputs
    from .qnn import build_circuit
    ext = np.hstack([xd, np.broadcast_to(pd, (B, P))])
    rows, index = [ext], []
    if want:
        for j in range(d + P):
            if (j < d and not want_x) or (j >= d and not want_p):
                continue
            for sgn in (1.0, -1.0):
                r = ext.copy()
                r[:, j] = ext[:, j] + sgn * shift
                rows.append(r)
                index.append(j)
    allrows = np.concatenate(rows)
    vals = noisy_circuit_values([build_circuit(builder, r[:d], r[d:]) for r in allrows], noise, shots, seed)
    jac = None
    if index:
        J = np.zeros((B, d + P))
        for k in range(0, len(index), 2):
            ep = vals[B * (1 + k):B * (2 + k)]
            em = vals[B * (2 + k):B * (3 + k)]
            J[:, index[k]] = (ep - em) * grad_scale
        jac = torch.from_numpy(J).to("cuda")
    return vals[:B], jac


def noisy_circuit_values(circuits, noise, shots, seed, want_counts=False):
    """E (and optionally counts) of concrete circuits under ``noise``."""
    from .noise import noise_sites
    torch = _torch()
    vals = np.empty(len(circuits))
    counts = [None] * len(circuits)
    for tape, rows in _circuit_rows(circuits).values():
        A = len(tape.slot_const)
        plan = _global_cache.get(tape, A, 0, "c128", None, math.pi / 2, 0.5)
        dev = f"cuda:{plan.device}"
        x = np.array([r[1] for r in rows], dtype=np.float64).reshape(len(rows), A)
        xt = torch.from_numpy(x).to(dev) if A else torch.zeros((len(rows), 1), dtype=torch.float64, device=dev)
        pt = torch.zeros(1, dtype=torch.float64, device=dev)
        e, _, cnt = plan.noisy(xt, pt, noise_sites(tape.ops, noise), shots, seed, False, want_counts)
        idx = [r[0] for r in rows]
        vals[idx] = e.cpu().numpy()
        if want_counts:
            c = cnt.cpu().numpy()
            for k, i in enumerate(idx):
                counts[i] = c[k]
    return (vals, counts) if want_counts else vals
