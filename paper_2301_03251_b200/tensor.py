"""Host tensor + dynamic autograd: only the boundary the quantum layer needs.

The reference's quantum layers hand their outputs back to a NumPy reverse-mode
graph (``pkg/src/hyqnet/tensor.py``).  This module restates that boundary so a
model written against hyqnet keeps working when the layer comes from this
package:

* ``GraphNode(parent, df)``                          — ``tensor.py:45-52``
* ``Tensor`` (data / requires_grad / grad / nodes)   — ``tensor.py:54-150``
* ``_make_result`` (nodes only when grad mode is on) — ``tensor.py:179-184``
* ``backward`` (post-order DFS, each df called once) — ``tensor.py:318-368``
* thread-local ``no_grad``                           — ``tensor.py:27-42``

Classical operators are limited to what losses around a quantum layer use
(+, -, *, /, sum, mean); conv/matmul/IO are out of scope.
:class:`paper_2301_03251_b200.qnn.QuantumLayer` also accepts reference hyqnet
tensors directly (duck-typed), so swapping only the layer is enough.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import ContractError, DimensionError

DEFAULT_DTYPE = np.float32

_mode = threading.local()


def grad_enabled() -> bool:
    return getattr(_mode, "on", True)


@contextmanager
def no_grad():
    """Evaluate without recording graph edges (per thread)."""
    saved = grad_enabled()
    _mode.on = False
    try:
        yield
    finally:
        _mode.on = saved


@dataclass
class GraphNode:
    """Edge to ``parent`` with ``df`` mapping the incoming gradient to the
    parent's contribution."""

    parent: "Tensor"
    df: Callable[[np.ndarray], np.ndarray]


class Tensor:
    """Real float32/float64 array with optional gradient tracking."""

    __array_priority__ = 100

    def __init__(self, data, requires_grad: bool = False, dtype=None):
        arr = np.asarray(data, dtype=dtype) if dtype is not None else np.asarray(data)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(dtype if dtype is not None else DEFAULT_DTYPE)
        self.data = arr
        self.requires_grad = bool(requires_grad)
        self.grad: np.ndarray | None = None
        self.nodes: list[GraphNode] = []

    shape = property(lambda self: self.data.shape)
    dtype = property(lambda self: self.data.dtype)
    size = property(lambda self: self.data.size)

    def numpy(self) -> np.ndarray:
        return self.data

    def item(self) -> float:
        return float(self.data.reshape(-1)[0])

    def detach(self) -> "Tensor":
        return Tensor(self.data, dtype=self.data.dtype)

    def zero_grad(self) -> None:
        self.grad = None

    def accumulate_grad(self, g: np.ndarray) -> None:
        if self.grad is None:
            self.grad = np.zeros_like(self.data)
        self.grad += np.asarray(g).astype(self.data.dtype, copy=False).reshape(self.data.shape)

    def backward(self, retain_graph: bool = False) -> None:
        backward(self, retain_graph=retain_graph)

    def __repr__(self):
        return f"Tensor({self.data!r}{', requires_grad=True' if self.requires_grad else ''})"

    def __add__(self, other):
        return _binary(self, other, np.add, lambda g, a, b: g, lambda g, a, b: g)

    __radd__ = __add__

    def __sub__(self, other):
        return _binary(self, other, np.subtract, lambda g, a, b: g, lambda g, a, b: -g)

    def __rsub__(self, other):
        return _binary(_wrap(other, self.dtype), self, np.subtract,
                       lambda g, a, b: g, lambda g, a, b: -g)

    def __mul__(self, other):
        return _binary(self, other, np.multiply, lambda g, a, b: g * b, lambda g, a, b: g * a)

    __rmul__ = __mul__

    def __truediv__(self, other):
        return _binary(self, other, np.divide, lambda g, a, b: g / b,
                       lambda g, a, b: -g * a / (b * b))

    def __neg__(self):
        return self * -1.0

    def sum(self):
        return tsum(self)

    def mean(self):
        return tmean(self)


def _wrap(value, dtype=None) -> Tensor:
    return value if isinstance(value, Tensor) else Tensor(value, dtype=dtype)


def _unbroadcast(g: np.ndarray, shape) -> np.ndarray:
    while g.ndim > len(shape):
        g = g.sum(axis=0)
    for axis, dim in enumerate(shape):
        if dim == 1 and g.shape[axis] != 1:
            g = g.sum(axis=axis, keepdims=True)
    return g


def _binary(a, b, op, da, db) -> Tensor:
    a = _wrap(a)
    b = _wrap(b, a.dtype)
    try:
        np.broadcast_shapes(a.shape, b.shape)
    except ValueError:
        raise DimensionError(f"cannot broadcast {a.shape} with {b.shape}") from None
    out = op(a.data, b.data)
    nodes = []
    if a.requires_grad:
        nodes.append(GraphNode(a, lambda g: _unbroadcast(da(g, a.data, b.data), a.shape)))
    if b.requires_grad:
        nodes.append(GraphNode(b, lambda g: _unbroadcast(db(g, a.data, b.data), b.shape)))
    return _make_result(np.asarray(out), nodes)


def tensor(values, shape=None, requires_grad: bool = False, dtype=None) -> Tensor:
    arr = np.asarray(values, dtype=dtype if dtype is not None else DEFAULT_DTYPE)
    if shape is not None:
        shape = tuple(int(s) for s in shape)
        if any(s < 1 for s in shape) or arr.size != int(np.prod(shape)):
            raise DimensionError(f"cannot shape {arr.size} values into {shape}")
        arr = arr.reshape(shape)
    return Tensor(arr.copy(), requires_grad=requires_grad, dtype=arr.dtype)


def _make_result(data: np.ndarray, nodes: list[GraphNode]) -> Tensor:
    out = Tensor(data, dtype=data.dtype)
    if nodes and grad_enabled():
        out.requires_grad = True
        out.nodes = nodes
    return out


def tsum(t) -> Tensor:
    t = _wrap(t)
    nodes = []
    if t.requires_grad:
        nodes.append(GraphNode(t, lambda g: np.broadcast_to(
            np.asarray(g, dtype=t.dtype), t.shape).copy()))
    return _make_result(np.asarray(t.data.sum()), nodes)


def tmean(t) -> Tensor:
    t = _wrap(t)
    n = t.size
    nodes = []
    if t.requires_grad:
        nodes.append(GraphNode(t, lambda g: np.broadcast_to(
            np.asarray(g, dtype=t.dtype) / n, t.shape).copy()))
    return _make_result(np.asarray(t.data.mean()), nodes)


def backward(loss: Tensor, retain_graph: bool = False) -> None:
    """Seed ``loss`` with 1 and push gradients to every reachable leaf.

    Same visiting discipline as the reference (``tensor.py:318-368``): a
    post-order DFS fixes a deterministic order, each ``df`` runs once per
    backward, edges are dropped afterwards unless ``retain_graph``.
    """
    if loss.size != 1:
        raise ContractError(f"backward requires a scalar loss, got shape {loss.shape}")
    if not loss.requires_grad:
        return
    order: list = []
    seen: set[int] = set()
    stack = [(loss, False)]
    while stack:
        t, done = stack.pop()
        if done:
            order.append(t)
            continue
        if id(t) in seen:
            continue
        seen.add(id(t))
        stack.append((t, True))
        for node in reversed(t.nodes):
            if id(node.parent) not in seen:
                stack.append((node.parent, False))
    pending = {id(loss): np.ones_like(loss.data)}
    for t in reversed(order):
        g = pending.pop(id(t), None)
        if g is None:
            continue
        if t.requires_grad:
            t.accumulate_grad(g)
        for node in t.nodes:
            contrib = np.asarray(node.df(g))
            if contrib.shape != node.parent.shape:
                contrib = contrib.reshape(node.parent.shape)
            key = id(node.parent)
            pending[key] = pending[key] + contrib if key in pending else contrib
        if not retain_graph:
            t.nodes = []
