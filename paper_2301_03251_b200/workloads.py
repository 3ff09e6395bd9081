"""The five benchmark circuits of SURVEY.md §8(d), written once against any
hyqnet-compatible module pair so the identical builder drives the reference
(golden vectors), the oracle and the GPU path.

``make_builder(cfg, qsim, templates)`` returns ``builder(inputs, params)``;
``inputs_for(cfg, batch)`` / ``params_for(cfg)`` give the seeded synthetic
data (``np.random.default_rng(0)`` for inputs, ``default_rng(1)`` for params).
"""

from __future__ import annotations

import math

import numpy as np

# name -> (n_qubits, n_inputs, n_params, default batch, primary precision)
CONFIGS = {
    "cfg1": (4, 4, 24, 64, "c128"),
    "cfg2": (10, 10, 60, 256, "c64"),
    "cfg3": (12, 512, 108, 1024, "c128"),
    "cfg4": (20, 20, 400, 4096, "c64"),
    "cfg5": (32, 0, 1280, 1, "c128"),
}


def make_builder(cfg: str, qsim, templates):
    Circuit = qsim.Circuit
    if cfg in ("cfg1", "cfg2"):
        n = CONFIGS[cfg][0]

        def vqc(inputs, params):
            # angle encoding; 2 x [RX RY RZ per qubit; CNOT ring]; P(q0 = 1)
            c = Circuit(n)
            for q in range(n):
                c.ry(q, inputs[q])
            k = 0
            for _ in range(2):
                for q in range(n):
                    c.rx(q, params[k])
                    c.ry(q, params[k + 1])
                    c.rz(q, params[k + 2])
                    k += 3
                for q in range(n):
                    c.cnot(q, (q + 1) % n)
            c.measure(0)
            return c
        return vqc
    if cfg == "cfg3":
        train = list(range(3, 12))

        def qae(inputs, params):
            # aux 0 | reference {1,2} | training {3..11}; HEA depth 6; SWAP test
            c = Circuit(12)
            c.extend(templates.amplitude_embedding(inputs, qubits=train))
            k = 0
            for _ in range(6):
                for q in train:
                    c.ry(q, params[k])
                    c.rz(q, params[k + 1])
                    k += 2
                for q in train[:-1]:
                    c.cnot(q, q + 1)
            c.h(0)
            for t, r in ((10, 1), (11, 2)):
                c.extend(templates.cswap(0, t, r))
            c.h(0)
            c.measure(0)
            return c
        return qae
    if cfg in ("cfg4", "cfg5"):
        n = CONFIGS[cfg][0]
        depth = 10 if cfg == "cfg4" else 20
        encode = cfg == "cfg4"

        def hea(inputs, params):
            # [RY(x) per qubit;] depth x [RY RZ per qubit; CNOT chain]; P(q0 = 1)
            c = Circuit(n)
            if encode:
                for q in range(n):
                    c.ry(q, inputs[q])
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
        return hea
    raise KeyError(cfg)


def qae_vectors(count: int, dim: int, support: int, seed: int = 0) -> np.ndarray:
    """Unit vectors on the first ``support`` coordinates (restates data.py:151-159)."""
    rng = np.random.default_rng(seed)
    out = np.zeros((count, dim), dtype=np.float64)
    block = rng.normal(size=(count, support))
    out[:, :support] = block / np.linalg.norm(block, axis=1, keepdims=True)
    return out


def inputs_for(cfg: str, batch: int | None = None) -> np.ndarray:
    n, d, _, b0, _ = CONFIGS[cfg]
    b = b0 if batch is None else batch
    if cfg == "cfg3":
        return qae_vectors(max(b, 1), 512, 128, seed=0)[:b]
    if d == 0:
        return np.zeros((b, 0))
    return np.random.default_rng(0).uniform(-math.pi, math.pi, (b, d))


def params_for(cfg: str) -> np.ndarray:
    return np.random.default_rng(1).uniform(0.0, 2 * math.pi, CONFIGS[cfg][2])


def gate_counts(cfg: str):
    """(R, D, total gates): non-permutation 1q gates, differentiated angle
    occurrences, all gates — the SURVEY.md §8(d) flop-model inputs."""
    n, d, P, _, _ = CONFIGS[cfg]
    if cfg in ("cfg1", "cfg2"):
        R = n + 2 * 3 * n
        return R, R, R + 2 * n
    if cfg == "cfg3":
        # 6 x 9 x 2 rotations + 2 cswap (each 2 H inside toffoli) + 2 H
        return 108 + 4 + 2, 108, 108 + 6 * 8 + 2 * 9 + 2
    if cfg == "cfg4":
        return n + 10 * 2 * n, 10 * 2 * n, n + 10 * (2 * n + n - 1)
    return 20 * 2 * n, 20 * 2 * n, 20 * (2 * n + n - 1)
