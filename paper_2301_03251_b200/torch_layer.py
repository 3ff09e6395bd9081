"""Device-resident boundary for hybrid PyTorch models.

The hyqnet-compatible :class:`~paper_2301_03251_b200.qnn.QuantumLayer` takes
NumPy tensors (``qnn.py:126,154``: inputs copied to float64 on the host,
outputs cast back).  In a GPU model that would round-trip every activation
through the host.  :class:`TorchQuantumLayer` keeps everything on the device:

* forward = one ``hq_forward`` (jacobian rows produced in the same launch
  sequence when autograd needs them);
* backward = one ``hq_vjp`` (upstream-scaled input rows, sample-ordered
  parameter sum) — the reference's ``df_x`` / ``df_p`` semantics;
* the builder is traced per input width (first call with that width, using
  the batch's first/last rows and a random probe — the same checks as the host
  layer, which reject value-dependent control flow).  With ``recheck=True``
  (default) every later batch re-runs the builder once, on its own last row
  (a 1-row device->host copy), and raises ``CircuitError`` if the tape
  changed; inside CUDA-graph capture, or with ``recheck=False``, the cached
  plan runs without any host synchronisation so forward+backward can be
  captured in a CUDA graph.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine
from . import tracer as tr
from .errors import CircuitError, ConfigError, DimensionError


class _QuantumFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, theta, plan, want_x, want_p):
        x64 = x.detach().to(torch.float64).contiguous()
        th64 = theta.detach().to(device=x.device, dtype=torch.float64).contiguous()
        need = want_x or want_p
        out, jac = plan.forward(x64, th64, need)
        ctx.plan = plan
        ctx.want = (want_x, want_p)
        ctx.xdtype = x.dtype
        ctx.tdev = theta.device
        if need:
            ctx.save_for_backward(jac)
        return out.to(x.dtype).unsqueeze(1)

    @staticmethod
    def backward(ctx, g):
        (jac,) = ctx.saved_tensors
        want_x, want_p = ctx.want
        gx, gt = ctx.plan.vjp(jac, g.detach().to(torch.float64).reshape(-1).contiguous(),
                              want_x and ctx.needs_input_grad[0], want_p and ctx.needs_input_grad[1])
        return (gx.to(ctx.xdtype) if gx is not None else None,
                gt.to(ctx.tdev) if gt is not None else None, None, None, None)


class TorchQuantumLayer(torch.nn.Module):
    """``forward(x[B, d] cuda) -> [B, 1]`` with reference gradient semantics."""

    def __init__(self, circuit_builder, n_params: int, precision: str = "c128",
                 shift: float = math.pi / 2, grad_scale: float = 0.5, param_init=None,
                 device=None, recheck: bool = True):
        super().__init__()
        if n_params < 0:
            raise ConfigError("n_params must be >= 0")
        if not shift > 0:
            raise ConfigError("shift must be positive")
        if precision not in ("c64", "c128"):
            raise ConfigError(f"precision must be 'c64' or 'c128', got {precision!r}")
        self.circuit_builder = circuit_builder
        self.n_params = int(n_params)
        self.precision = precision
        self.shift = float(shift)
        self.grad_scale = float(grad_scale)
        if param_init is None:
            from .rng import default_generator
            param_init = default_generator().uniform(0, 2 * np.pi, n_params)
        param_init = np.asarray(param_init, dtype=np.float64)
        if param_init.shape != (n_params,):
            raise ConfigError(f"param_init shape {param_init.shape} != ({n_params},)")
        self.params = torch.nn.Parameter(torch.tensor(param_init, dtype=torch.float64, device=device))
        self.recheck = bool(recheck)
        self._tapes = {}          # input width -> traced tape (variable ids depend on d)
        self._plans = {}

    def _trace(self, x):
        rows = x[[0, -1]].detach().to("cpu", torch.float64).numpy()
        tape, ok = tr.trace(self.circuit_builder, rows, self.params.detach().cpu().numpy())
        if not ok:
            raise CircuitError("TorchQuantumLayer needs a batch-invariant affine builder "
                               "(use QuantumLayer for data-dependent circuits)")
        return tape

    def _plan(self, x, want_x, want_p):
        d = x.shape[1]
        tape = self._tapes.get(d)
        if tape is None:
            tape = self._tapes[d] = self._trace(x)
        elif self.recheck and not torch.cuda.is_current_stream_capturing():
            # cheap per-batch check: one traced builder call on the batch's last
            # row (a 1-row device->host copy) against the cached tape
            row = x[-1].detach().to("cpu", torch.float64).numpy()
            other = tr.traced_call(self.circuit_builder, row, self.params.detach().cpu().numpy())
            if not tape.same_as(other):
                raise CircuitError("circuit builder produced a different circuit for this batch than "
                                   "the traced one (structure or angle expressions changed)")
        if x.device.type != "cuda":
            raise DimensionError(f"TorchQuantumLayer expects CUDA inputs, got {x.device}")
        key = (want_x, want_p, d, x.device.index)
        plan = self._plans.get(key)
        if plan is None:
            grad = tr.classify(tape, d + self.n_params, [want_x] * d + [want_p] * self.n_params,
                               self.shift, self.grad_scale) if (want_x or want_p) else None
            with torch.cuda.device(x.device):
                plan = engine.Plan(tape, d, self.n_params, self.precision, grad, self.shift,
                                   self.grad_scale)
            self._plans[key] = plan
        return plan

    def forward(self, x):
        if x.dim() != 2:
            raise DimensionError(f"expected [N, d] input, got shape {tuple(x.shape)}")
        if x.shape[0] == 0:
            return x.new_zeros((0, 1))
        track = torch.is_grad_enabled()
        want_x = track and x.requires_grad
        want_p = track and self.params.requires_grad and self.n_params > 0
        plan = self._plan(x, want_x, want_p)
        return _QuantumFn.apply(x, self.params, plan, want_x, want_p)
