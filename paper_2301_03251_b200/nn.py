"""Module tree boundary: ``Parameter`` and ``Module`` only.

Restates ``pkg/src/hyqnet/nn.py:21-83``: parameters register on attribute
assignment so ``QuantumLayer.params`` shows up in ``parameters()`` exactly
once.  The classical layers of that file (Conv2D, Linear, ...) are out of scope
 — on device, PyTorch supplies them.
"""

from __future__ import annotations

from typing import Iterator

import numpy as np

from .tensor import DEFAULT_DTYPE, Tensor


class Parameter(Tensor):
    """Trainable leaf; always requires a gradient (``nn.py:21-25``)."""

    def __init__(self, data, dtype=None):
        super().__init__(np.asarray(data, dtype=dtype or DEFAULT_DTYPE), requires_grad=True)


class Module:
    """Base calculation node (``nn.py:28-83``)."""

    def __init__(self):
        object.__setattr__(self, "_parameters", {})
        object.__setattr__(self, "_children", {})
        object.__setattr__(self, "training", True)

    def __setattr__(self, name, value):
        if isinstance(value, Parameter):
            self._parameters[name] = value
        elif isinstance(value, Module):
            self._children[name] = value
        object.__setattr__(self, name, value)

    def forward(self, *args):
        raise NotImplementedError

    def __call__(self, *args):
        return self.forward(*args)

    def _walk(self, prefix: str):
        for name, p in self._parameters.items():
            yield prefix + name, p
        for name, child in self._children.items():
            yield from child._walk(prefix + name + ".")

    def named_parameters(self, prefix: str = "") -> Iterator[tuple[str, Parameter]]:
        seen: set[int] = set()
        for name, p in self._walk(prefix):
            if id(p) not in seen:
                seen.add(id(p))
                yield name, p

    def parameters(self) -> list[Parameter]:
        return [p for _, p in self.named_parameters()]

    def children(self) -> list["Module"]:
        return list(self._children.values())

    def train(self, mode: bool = True) -> "Module":
        object.__setattr__(self, "training", mode)
        for child in self._children.values():
            child.train(mode)
        return self

    def eval(self) -> "Module":
        return self.train(False)

    def zero_grad(self) -> None:
        for p in self.parameters():
            p.zero_grad()
