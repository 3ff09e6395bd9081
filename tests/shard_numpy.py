"""NumPy stand-in for the GPU segment executor of ``shard.py`` (test
infrastructure only): lets the amplitude-sharded driver — schedule, per-rank
resolution, all-to-all exchanges, readout weights, the reversed adjoint sweep
and the cross-rank reductions — run on CPU with real gloo processes.

Gate conventions follow the kernels: qubit k = bit k of the local index; RZ is
applied as diag(1, e^{iθ}) (the kernels drop the global phase e^{-iθ/2}; a
resolved CR on a rank-constant control is exactly that operator), RX/RY/H/Y
exactly.  Adjoint: for a gate G(α) with ψ, λ taken after it, dE/dα =
Im<λ|P|ψ> for exp(-iαP/2) (RX, RY) and -2 Im<λ|P1|ψ> for diag(1, e^{iα})."""

import numpy as np
import torch

from paper_2301_03251_b200 import shard as S

_H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)
_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)


def _mat(kind, a):
    if kind == "H":
        return _H
    if kind == "X":
        return _X
    if kind == "Y":
        return _Y
    if kind == "Z":
        return _Z
    c, s = np.cos(a / 2), np.sin(a / 2)
    if kind == "RX":
        return np.array([[c, -1j * s], [-1j * s, c]])
    if kind == "RY":
        return np.array([[c, -s], [s, c]], dtype=np.complex128)
    if kind == "RZ":
        return np.array([[1, 0], [0, np.exp(1j * a)]])
    raise ValueError(kind)


def _pair(v, q):
    return v.reshape(-1, 2, 1 << q)


def _apply1(v, q, M):
    p = _pair(v, q)
    a, b = p[:, 0, :].copy(), p[:, 1, :].copy()
    p[:, 0, :] = M[0, 0] * a + M[0, 1] * b
    p[:, 1, :] = M[1, 0] * a + M[1, 1] * b


def _idx(n):
    return np.arange(1 << n)


def apply(v, n, kind, t, a, inverse=False):
    if kind in ("H", "X", "Y", "Z", "RX", "RY", "RZ"):
        M = _mat(kind, a)
        _apply1(v, t[0], M.conj().T if inverse else M)
        return
    i = _idx(n)
    if kind == "CNOT":
        sel = ((i >> t[0]) & 1) == 1
        sel &= ((i >> t[1]) & 1) == 0
        j = i[sel]
        k = j | (1 << t[1])
        v[j], v[k] = v[k].copy(), v[j].copy()
    elif kind == "SWAP":
        sel = (((i >> t[0]) & 1) == 1) & (((i >> t[1]) & 1) == 0)
        j = i[sel]
        k = (j & ~(1 << t[0])) | (1 << t[1])
        v[j], v[k] = v[k].copy(), v[j].copy()
    elif kind in ("CZ", "CR"):
        sel = (((i >> t[0]) & 1) == 1) & (((i >> t[1]) & 1) == 1)
        ph = -1.0 if kind == "CZ" else np.exp(1j * a)
        v[sel] *= np.conj(ph) if inverse else ph
    else:
        raise ValueError(kind)


def _angle(sc, slot, x, theta):
    val = sc.tape.slot_const[slot]
    for var, c in sc.tape.slot_terms[slot].items():
        val += c * (x[var] if var < sc.n_inputs else theta[var - sc.n_inputs])
    return val


def _dot(v_psi, v_lam, n, kind, t):
    i = _idx(n)
    if kind in ("RX", "RY"):
        w = v_psi.copy()
        _apply1(w, t[0], _X if kind == "RX" else _Y)
        return float(np.imag(np.vdot(v_lam, w)))
    if kind == "RZ":
        sel = ((i >> t[0]) & 1) == 1
        return float(-2.0 * np.imag(np.vdot(v_lam[sel], v_psi[sel])))
    if kind == "CR":
        sel = (((i >> t[0]) & 1) == 1) & (((i >> t[1]) & 1) == 1)
        return float(-2.0 * np.imag(np.vdot(v_lam[sel], v_psi[sel])))
    raise ValueError(kind)


class NumpyExecutor:
    """Same interface as ``shard.GpuExecutor``; buffers are CPU complex128 tensors."""

    def seg_forward(self, sc, i, rank, buf, x, theta):
        v = buf.numpy()
        xs, ts = x.numpy().reshape(-1), theta.numpy().reshape(-1)
        tape, _ = sc.segment(i, rank)
        for kind, t, slot in tape.ops:
            apply(v, sc.L, kind, t, _angle(sc, slot, xs, ts) if slot >= 0 else None)

    def seg_backward(self, sc, i, rank, psi, lam, x, theta):
        p, l = psi.numpy(), lam.numpy()
        xs, ts = x.numpy().reshape(-1), theta.numpy().reshape(-1)
        tape, (mode, vslot, factor) = sc.segment(i, rank)
        var_of = {int(s): v for v, s in enumerate(vslot) if s >= 0}
        jac = np.zeros(sc.n_vars)
        for kind, t, slot in reversed(tape.ops):
            a = _angle(sc, slot, xs, ts) if slot >= 0 else None
            v = var_of.get(slot)
            if v is not None:
                jac[v] += factor[v] * _dot(p, l, sc.L, kind, t)
            apply(p, sc.L, kind, t, a, inverse=True)
            apply(l, sc.L, kind, t, a, inverse=True)
        return torch.from_numpy(jac)

    def readout(self, sc, rank, buf, lam_out):
        pos, wk, w0 = S.readout_weights(sc.sched, rank)
        i = _idx(sc.L)
        w = np.full(1 << sc.L, w0)
        for p_, k in zip(pos, wk):
            w += k * ((i >> p_) & 1)
        v = buf.numpy()
        if lam_out is not None:
            lam_out.numpy()[:] = w * v
        return torch.tensor([float(np.sum(w * np.abs(v) ** 2))], dtype=torch.float64)

    def zeros_jac(self, sc):
        return torch.zeros(sc.n_vars, dtype=torch.float64)


def virtual_exchange_cpu(bufs):
    return S.virtual_exchange(bufs)


# ---------------------------------------------------------------------------
# circuits for the sharding tests (each parameter enters exactly one
# rotation: the adjoint reproduces the reference's two-point value there)
def random_param_builder(n, depth, seed):
    rng = np.random.default_rng(seed)
    kinds = ["H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP"]
    plan, P = [], 0
    for _ in range(depth):
        k = kinds[rng.integers(len(kinds))]
        tg = tuple(int(q) for q in rng.choice(n, 2, replace=False)) if k in ("CNOT", "CZ", "CR", "SWAP") \
            else (int(rng.integers(n)),)
        if k in ("RX", "RY", "RZ", "CR"):
            plan.append((k, tg, P))
            P += 1
        else:
            plan.append((k, tg, -1))
    meas = [int(q) for q in rng.choice(n, min(n, 3), replace=False)]

    def builder(inputs, params, Circ=None):
        if Circ is None:
            from paper_2301_03251_b200.qsim import Circuit as Circ
        c = Circ(n)
        for k, tg, v in plan:
            if k == "CR":
                c.cr(tg[0], tg[1], params[v])
            elif v >= 0:
                getattr(c, k.lower())(tg[0], params[v])
            else:
                getattr(c, k.lower())(*tg)
        c.measure(*meas)
        return c
    return builder, P


def hea_builder(n, depth):
    """cfg5's shape: depth x [RY, RZ per qubit; CNOT chain]; measure(0)."""
    def builder(inputs, params, Circ=None):
        if Circ is None:
            from paper_2301_03251_b200.qsim import Circuit as Circ
        c = Circ(n)
        k = 0
        for _ in range(depth):
            for q in range(n):
                c.ry(q, params[k])
                c.rz(q, params[k + 1])
                k += 2
            for q in range(n - 1):
                c.cnot(q, q + 1)
        c.measure(0)
        return c
    return builder, 2 * n * depth


def oracle_reference(builder, theta):
    """(E, dE rows at upstream 1 [P], final state) from the CPU oracle."""
    from oracle import hq_oracle as O
    ob = lambda i, p: builder(i, p, Circ=O.Circuit)
    out, _, jp, _, _ = O.layer(ob, np.zeros((1, 0)), theta, want_x=False)
    psi = O.simulate(ob([], list(theta)))
    return float(out[0]), jp[0], psi


def sharded(builder, P, theta, g, precision="c128"):
    from paper_2301_03251_b200 import tracer as tr
    tape, ok = tr.trace(builder, np.zeros((1, 0)), np.asarray(theta))
    assert ok
    return S.ShardedCircuit(tape, 0, P, g, precision)


def same_up_to_phase(a, b, atol):
    k = int(np.argmax(np.abs(b)))
    ph = a[k] / b[k] if abs(b[k]) > 0 else 1.0
    ph = ph / abs(ph)
    np.testing.assert_allclose(a, ph * b, atol=atol)
