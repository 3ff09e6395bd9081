"""ctypes binding of ``libhq.so`` (the C ABI declared in ``include/hq.h``).

There is deliberately no fallback: if the library or a CUDA device is missing
every entry point raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CircuitError, ConfigError, DimensionError, EncodingError, NativeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhq.so")

HQ_OK, HQ_E_CIRCUIT, HQ_E_CONFIG, HQ_E_DIMENSION, HQ_E_CUDA, HQ_E_OOM, HQ_E_ENCODING = range(7)
HQ_C64, HQ_C128 = 0, 1
HQ_WANT_JAC = 1
KIND_CODE = {"H": 0, "X": 1, "Y": 2, "Z": 3, "RX": 4, "RY": 5, "RZ": 6, "CNOT": 7, "CZ": 8,
             "CR": 9, "SWAP": 10, "STATEPREP": 11}

EXPORTS = ("hq_abi_version", "hq_last_error", "hq_plan_create", "hq_plan_destroy",
           "hq_plan_describe", "hq_workspace_bytes", "hq_forward", "hq_vjp", "hq_state",
           "hq_stats", "hq_profile_enable", "hq_profile_read", "hq_sample_workspace_bytes", "hq_sample",
           "hq_shot_uniforms", "hq_noisy_workspace_bytes", "hq_noisy", "hq_launch_counts",
           "hq_plan_create_segment", "hq_seg_workspace_bytes", "hq_seg_forward", "hq_seg_backward",
           "hq_shard_readout_workspace_bytes", "hq_shard_readout", "hq_comm_id_bytes", "hq_comm_unique_id",
           "hq_comm_init", "hq_comm_destroy", "hq_comm_allreduce_f64", "hq_comm_alltoall", "hq_backward_dp",
           "hq_marginal_workspace_bytes", "hq_marginal")
K_CLASSES = ("onchip", "pass_fwd", "pass_bwd", "other")


class HqOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("slot", ctypes.c_int32)]


_P = ctypes.c_void_p


class HqPlanDesc(ctypes.Structure):
    _fields_ = [
        ("n_qubits", ctypes.c_int32), ("precision", ctypes.c_int32),
        ("n_ops", ctypes.c_int32), ("ops", _P),
        ("n_slots", ctypes.c_int32), ("slot_const", _P), ("slot_ptr", _P), ("slot_var", _P),
        ("slot_coef", _P),
        ("n_inputs", ctypes.c_int32), ("n_params", ctypes.c_int32),
        ("n_measured", ctypes.c_int32), ("measured", _P),
        ("n_preps", ctypes.c_int32), ("prep_ptr", _P), ("prep_qubits", _P), ("prep_slot0", _P),
        ("prep_len", _P),
        ("grad_mode", _P), ("grad_slot", _P), ("grad_factor", _P),
        ("shift", ctypes.c_double), ("grad_scale", ctypes.c_double),
    ]


class HqNoiseSite(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("qubit", ctypes.c_int32), ("channel", ctypes.c_int32),
                ("param", ctypes.c_double)]


CHANNEL_CODE = {"bit_flip": 0, "phase_flip": 1, "depolarizing": 2, "amplitude_damping": 3}


class HqStats(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("n_passes", ctypes.c_int32),
                ("tile_bits", ctypes.c_int32), ("n_adjoint_slots", ctypes.c_int32),
                ("n_twopoint_vars", ctypes.c_int32), ("launches", ctypes.c_int64),
                ("chunk_samples", ctypes.c_int64), ("state_bytes", ctypes.c_double)]


class HqProfile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 4), ("launches", ctypes.c_int64 * 4),
                ("bytes", ctypes.c_double * 4)]


_lib = None


def lib():
    """Load libhq.so once; raise NativeError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
    h = ctypes.CDLL(LIB_PATH)
    h.hq_abi_version.restype = ctypes.c_int
    h.hq_last_error.restype = ctypes.c_char_p
    h.hq_plan_create.argtypes = [ctypes.POINTER(HqPlanDesc), ctypes.POINTER(_P)]
    h.hq_plan_create.restype = ctypes.c_int
    h.hq_plan_destroy.argtypes = [_P]
    h.hq_plan_destroy.restype = None
    h.hq_plan_describe.argtypes = [_P]
    h.hq_plan_describe.restype = ctypes.c_char_p
    h.hq_workspace_bytes.argtypes = [_P, ctypes.c_int64, ctypes.c_int32]
    h.hq_workspace_bytes.restype = ctypes.c_size_t
    h.hq_forward.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int32, _P, _P,
                             _P, ctypes.c_size_t, _P]
    h.hq_forward.restype = ctypes.c_int
    h.hq_vjp.argtypes = [_P, _P, _P, ctypes.c_int64, _P, _P, _P]
    h.hq_vjp.restype = ctypes.c_int
    h.hq_state.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, _P, ctypes.c_int64, _P, _P,
                           ctypes.c_size_t, _P]
    h.hq_state.restype = ctypes.c_int
    h.hq_stats.argtypes = [_P, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(HqStats)]
    h.hq_stats.restype = ctypes.c_int
    h.hq_profile_enable.argtypes = [_P, ctypes.c_int32]
    h.hq_profile_enable.restype = ctypes.c_int
    h.hq_profile_read.argtypes = [_P, ctypes.POINTER(HqProfile)]
    h.hq_profile_read.restype = ctypes.c_int
    h.hq_sample_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
    h.hq_sample_workspace_bytes.restype = ctypes.c_size_t
    h.hq_sample.argtypes = [_P, ctypes.c_int64, ctypes.c_int32, _P, ctypes.c_int32, ctypes.c_int64,
                            ctypes.c_uint64, _P, _P, _P, ctypes.c_size_t, _P]
    h.hq_sample.restype = ctypes.c_int
    h.hq_shot_uniforms.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _P, _P]
    h.hq_shot_uniforms.restype = ctypes.c_int
    h.hq_noisy_workspace_bytes.argtypes = [_P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
    h.hq_noisy_workspace_bytes.restype = ctypes.c_size_t
    h.hq_noisy.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int32, _P, ctypes.c_int32,
                           ctypes.c_int64, ctypes.c_uint64, _P, _P, _P, _P, ctypes.c_size_t, _P]
    h.hq_noisy.restype = ctypes.c_int
    h.hq_launch_counts.argtypes = [_P]
    h.hq_launch_counts.restype = None
    h.hq_plan_create_segment.argtypes = [ctypes.POINTER(HqPlanDesc), ctypes.POINTER(_P)]
    h.hq_plan_create_segment.restype = ctypes.c_int
    h.hq_seg_workspace_bytes.argtypes = [_P, ctypes.c_int64]
    h.hq_seg_workspace_bytes.restype = ctypes.c_size_t
    h.hq_seg_forward.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, _P, _P, ctypes.c_size_t, _P]
    h.hq_seg_forward.restype = ctypes.c_int
    h.hq_seg_backward.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_size_t,
                                  _P]
    h.hq_seg_backward.restype = ctypes.c_int
    h.hq_shard_readout_workspace_bytes.argtypes = []
    h.hq_shard_readout_workspace_bytes.restype = ctypes.c_size_t
    h.hq_shard_readout.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, _P, _P, ctypes.c_int32, ctypes.c_double,
                                   _P, _P, _P, ctypes.c_size_t, _P]
    h.hq_shard_readout.restype = ctypes.c_int
    h.hq_comm_id_bytes.argtypes = []
    h.hq_comm_id_bytes.restype = ctypes.c_size_t
    h.hq_comm_unique_id.argtypes = [_P]
    h.hq_comm_unique_id.restype = ctypes.c_int
    h.hq_comm_init.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_P)]
    h.hq_comm_init.restype = ctypes.c_int
    h.hq_comm_destroy.argtypes = [_P]
    h.hq_comm_destroy.restype = None
    h.hq_comm_allreduce_f64.argtypes = [_P, _P, ctypes.c_int64, _P]
    h.hq_comm_allreduce_f64.restype = ctypes.c_int
    h.hq_comm_alltoall.argtypes = [_P, _P, _P, ctypes.c_int64, _P]
    h.hq_comm_alltoall.restype = ctypes.c_int
    h.hq_backward_dp.argtypes = [_P, _P, ctypes.c_int64, _P, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _P,
                                 ctypes.c_size_t, _P]
    h.hq_backward_dp.restype = ctypes.c_int
    h.hq_marginal_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
    h.hq_marginal_workspace_bytes.restype = ctypes.c_size_t
    h.hq_marginal.argtypes = [_P, ctypes.c_int64, ctypes.c_int32, _P, ctypes.c_int32, _P, _P, ctypes.c_size_t, _P]
    h.hq_marginal.restype = ctypes.c_int
    if h.hq_abi_version() != 2:
        raise NativeError(f"libhq ABI {h.hq_abi_version()} != 2")
    _lib = h
    return h


def launch_counts() -> dict:
    """Process-wide kernel launches per class since the library loaded."""
    arr = (ctypes.c_int64 * 4)()
    lib().hq_launch_counts(ctypes.cast(arr, _P))
    return {k: int(arr[i]) for i, k in enumerate(K_CLASSES)}


def check(status: int, what: str) -> None:
    if status == HQ_OK:
        return
    msg = lib().hq_last_error().decode(errors="replace")
    cls = {HQ_E_CIRCUIT: CircuitError, HQ_E_CONFIG: ConfigError, HQ_E_DIMENSION: DimensionError,
           HQ_E_ENCODING: EncodingError}.get(status, NativeError)
    raise cls(f"{what}: {msg}")
