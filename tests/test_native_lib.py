"""The C-ABI library (CPU-side checks, no kernel launches).

* libhq.so loads and exports every symbol include/hq.h declares;
* descriptor validation happens before any device work, so the error mapping
  (HQ_E_CIRCUIT -> CircuitError, ...) is testable without a GPU.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from paper_2301_03251_b200 import _native as nat
from paper_2301_03251_b200.errors import CircuitError, ConfigError, EncodingError


def header_symbols():
    text = open(os.path.join(REPO, "include", "hq.h")).read()
    return sorted(set(re.findall(r"\b(hq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = nat.lib()
    syms = header_symbols()
    assert set(syms) == set(nat.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.hq_abi_version() == 2


def _desc(n=2, ops=((4, 0, -1, 0),), n_slots=1, measured=(), preps=None):
    d = nat.HqPlanDesc()
    arr = (nat.HqOp * max(1, len(ops)))(*[nat.HqOp(*o) for o in ops])
    keep = [arr]
    d.n_qubits, d.precision = n, nat.HQ_C128
    d.n_ops, d.ops = len(ops), ctypes.cast(arr, ctypes.c_void_p)
    const = np.zeros(max(1, n_slots))
    ptr = np.zeros(n_slots + 1, np.int32)
    keep += [const, ptr]
    d.n_slots, d.slot_const, d.slot_ptr = n_slots, const.ctypes.data, ptr.ctypes.data
    m = np.array(measured, np.int32)
    keep.append(m)
    d.n_measured, d.measured = len(measured), (m.ctypes.data if len(measured) else None)
    d.shift, d.grad_scale = np.pi / 2, 0.5
    if preps:
        pptr, pq, s0, ln = (np.array(a, np.int32) for a in preps)
        keep += [pptr, pq, s0, ln]
        d.n_preps = len(s0)
        d.prep_ptr, d.prep_qubits = pptr.ctypes.data, pq.ctypes.data
        d.prep_slot0, d.prep_len = s0.ctypes.data, ln.ctypes.data
    return d, keep


@pytest.mark.parametrize("kw,err", [
    (dict(n=0), CircuitError),
    (dict(n=40), CircuitError),
    (dict(ops=((4, 2, -1, 0),)), CircuitError),        # target out of range
    (dict(ops=((7, 1, 1, -1),)), CircuitError),        # duplicate CNOT targets
    (dict(ops=((0, 0, -1, 0),)), CircuitError),        # H with an angle
    (dict(ops=((4, 0, -1, -1),)), CircuitError),       # RX without an angle
    (dict(ops=((42, 0, -1, -1),)), CircuitError),      # unknown kind
    (dict(measured=(0, 0)), CircuitError),             # measured twice
    (dict(measured=(5,)), CircuitError),               # measured out of range
    (dict(ops=(), n_slots=1, preps=([0, 1], [0], [0], [3])), EncodingError),
])
def test_validation_errors_map_to_reference_types(kw, err):
    d, keep = _desc(**kw)
    h = ctypes.c_void_p()
    with pytest.raises(err):
        nat.check(nat.lib().hq_plan_create(ctypes.byref(d), ctypes.byref(h)), "plan")


def test_null_descriptor_is_config_error():
    h = ctypes.c_void_p()
    with pytest.raises(ConfigError):
        nat.check(nat.lib().hq_plan_create(None, ctypes.byref(h)), "plan")
