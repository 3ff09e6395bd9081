"""B200-native batched variational-circuit simulation behind the hyqnet API.

Drop-in for the hot path of VQNet 2.0 (reference package ``hyqnet``): the
``QuantumLayer`` / circuit-builder API (``pkg/src/hyqnet/__init__.py:9-31``
re-exports the same names), executed by hand-written sm_100a kernels through
the C ABI in ``include/hq.h``.  See DESIGN.md.
"""

from .errors import (AdapterError, CircuitError, ConfigError, ContractError, DimensionError,
                     EncodingError, FormatError, HyqnetError, NativeError)
from .tensor import (GraphNode, Tensor, backward, no_grad, tensor, tmean, tsum)
from .rng import manual_seed
from .nn import Module, Parameter
from .qsim import (MAX_QUBITS, Circuit, Counts, GateOp, StatePrepOp, StateVector, apply_gate,
                   format_circuit_text, gate_matrix, parse_circuit_text, probabilities, simulate)
from .templates import (amplitude_embedding, angle_embedding, basis_embedding, ccz, cry, crz,
                        cswap, toffoli)
from .qnn import (EXACT_PROB, NOISY, SHOT_SAMPLING, NoiseQuantumLayer, QAELayer, QuantumLayer,
                  expectation_from_counts, measure_shots, parameter_shift_grad, shot_rng)
from .noise import (CHANNEL_NAMES, Channel, NoiseModel, amplitude_damping, apply_channel, bit_flip,
                    depolarizing, phase_flip, run_trajectory, simulate_noisy)

__version__ = "0.1.0"
