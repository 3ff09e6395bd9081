"""Multi-GPU execution: one process per GPU, ``torch.distributed`` for plumbing.

Batch sharding
    Samples are independent, so each rank owns a contiguous block of rows,
    runs forward + adjoint locally and contributes its partial parameter
    gradient to ONE ``all_reduce(sum)`` of the ``[P]`` f64 vector (NCCL over
    NVLink on the GPU path).  The reference sums per-sample gradients
    sequentially (``qnn.py:147-152``); here each rank sums its own rows in
    order and the ranks' partials are added by the collective — a different
    floating-point association, ~1e-16 relative.

Amplitude sharding (cfg5)
    See :mod:`paper_2301_03251_b200.shard`: one circuit whose state is split
    over ranks by its top index bits, with global-qubit swaps done as an
    all-to-all.

The functions take an ``evaluate(x_rows, theta) -> (out, jac)`` callable so the
sharding logic is testable on CPU with gloo (the tests plug in the oracle); on
GPUs :func:`plan_evaluator` wraps an :class:`engine.Plan`.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of rows for ``rank`` (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    return dist


def dp_forward_grad(evaluate, x: np.ndarray, theta: np.ndarray, upstream: np.ndarray,
                    group=None, device=None):
    """Sample-sharded forward + gradient of one batch.

    Every rank passes the full batch description (or only its shard, with
    ``x`` already sliced and ``upstream`` matching); returns the rank's
    outputs, its input-gradient rows and the all-reduced parameter gradient.
    """
    import torch
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(x.shape[0], rank, world)
    out, jac = evaluate(x[lo:hi], theta)
    jac = np.asarray(jac)
    d = x.shape[1]
    g = np.asarray(upstream, dtype=np.float64).reshape(-1)[lo:hi]
    grad_x = jac[:, :d] * g[:, None]
    grad_p = np.zeros(theta.shape[0])
    for i in range(hi - lo):                       # sample order within the shard
        grad_p += jac[i, d:] * g[i]
    if world > 1:
        t = torch.from_numpy(grad_p)
        if device is not None:
            t = t.to(device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        grad_p = t.cpu().numpy()
    return (lo, hi), np.asarray(out), grad_x, grad_p


def gather_rows(local: np.ndarray, n: int, group=None, device=None) -> np.ndarray:
    """All-gather per-rank row blocks (``shard_bounds`` layout) into ``[n, ...]``."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    sizes = [shard_bounds(n, r, world) for r in range(world)]
    width = int(np.prod(local.shape[1:])) if local.ndim > 1 else 1
    maxrows = max(hi - lo for lo, hi in sizes)
    buf = np.zeros((maxrows, width))
    buf[:local.shape[0]] = local.reshape(local.shape[0], width)
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    rows = [o.cpu().numpy()[:hi - lo] for o, (lo, hi) in zip(outs, sizes)]
    return np.concatenate(rows).reshape((n,) + local.shape[1:])


def plan_evaluator(plan, device):
    """GPU evaluator: (x_rows, theta) -> (out, jac) through the sm_100a plan."""
    import torch

    def evaluate(x_rows, theta):
        xd = torch.from_numpy(np.ascontiguousarray(x_rows, dtype=np.float64)).to(device)
        td = torch.from_numpy(np.ascontiguousarray(theta, dtype=np.float64)).to(device)
        out, jac = plan.forward(xd, td, True)
        return out.cpu().numpy(), jac.cpu().numpy()
    return evaluate


class DataParallelQuantumLayer:
    """Wrap a :class:`QuantumLayer` so its parameter gradient is all-reduced.

    Each rank calls it on its OWN local batch (DDP style); ``df_p`` returns the
    global sum over all ranks' samples.  Inputs' gradients stay rank-local.
    """

    def __init__(self, layer, group=None, device=None):
        self.layer = layer
        self.group = group
        self.device = device

    def __getattr__(self, name):
        return getattr(self.layer, name)

    def __call__(self, x):
        return self.forward(x)

    def forward(self, x):
        out = self.layer(x)
        dist = _dist()
        if not (dist.is_initialized() and dist.get_world_size(self.group) > 1):
            return out
        import torch
        group, device = self.group, self.device
        for node in out.nodes:
            if node.parent is self.layer.params:
                local_df = node.df

                def df(g, local_df=local_df):
                    t = torch.from_numpy(np.asarray(local_df(g), dtype=np.float64))
                    if device is not None:
                        t = t.to(device)
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                    return t.cpu().numpy()
                node.df = df
        return out


class LibComm:
    """The library's own NCCL communicator (``hq_comm_*`` in include/hq.h):
    one per process, rank / world taken from ``torch.distributed`` (the
    ncclUniqueId is made on rank 0 and broadcast through the process group) or
    a single-rank communicator when no group is initialised."""

    def __init__(self, device=None, group=None):
        import ctypes
        import torch
        from . import _native as nat
        self._nat = nat
        L = nat.lib()
        dist = _dist()
        if dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nid = int(L.hq_comm_id_bytes())
        buf = (ctypes.c_char * nid)()
        if self.rank == 0:
            nat.check(L.hq_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "comm id")
        if self.world > 1:
            obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=0, group=group)
            ctypes.memmove(buf, obj[0], nid)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            nat.check(L.hq_comm_init(ctypes.cast(buf, ctypes.c_void_p), self.rank, self.world, ctypes.byref(h)),
                      "comm init")
        self._h = h
        self._lib = L

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.hq_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        import torch
        return torch.cuda.current_stream(self.device).cuda_stream

    def allreduce_(self, t):
        """In-place sum over ranks of a contiguous f64 CUDA tensor."""
        import torch
        if t.dtype != torch.float64 or not t.is_contiguous() or t.device != self.device:
            raise ValueError("allreduce_ needs a contiguous float64 tensor on the communicator's device")
        self._nat.check(self._lib.hq_comm_allreduce_f64(self._h, t.data_ptr(), t.numel(), self._stream()), "allreduce")
        return t

    def alltoall(self, send, recv):
        """Chunk j of ``send`` -> rank j, chunk from rank j -> chunk j of ``recv``."""
        nbytes = send.numel() * send.element_size()
        if nbytes % self.world or recv.numel() * recv.element_size() != nbytes:
            raise ValueError("alltoall needs equal-size buffers divisible by the world size")
        self._nat.check(self._lib.hq_comm_alltoall(self._h, send.data_ptr(), recv.data_ptr(), nbytes // self.world,
                                                   self._stream()), "alltoall")
        return recv

    def backward_dp(self, plan, x, theta, upstream, want_x=False):
        """hq_backward_dp: this rank's forward + jacobian + vjp, then ONE
        all-reduce of the [P] parameter gradient.  -> (out, grad_x | None, grad_theta)."""
        import torch
        B = int(x.shape[0])
        dev = x.device
        out = torch.empty(B, dtype=torch.float64, device=dev)
        jac = torch.empty((B, plan.n_vars), dtype=torch.float64, device=dev)
        gx = torch.empty((B, plan.n_inputs), dtype=torch.float64, device=dev) if want_x else None
        gt = torch.empty(max(plan.n_params, 1), dtype=torch.float64, device=dev)
        st = plan._on_device(x, theta, upstream)
        ws, _ = plan._ws(B, self._nat.HQ_WANT_JAC)
        with torch.cuda.device(plan.device):
            self._nat.check(self._lib.hq_backward_dp(
                plan._h, x.data_ptr(), int(x.stride(0)), theta.data_ptr(), B, upstream.data_ptr(), out.data_ptr(),
                jac.data_ptr(), gx.data_ptr() if gx is not None else None, gt.data_ptr(), self._h, ws.data_ptr(),
                ws.numel(), st), "backward_dp")
        return out, gx, gt[:plan.n_params]
