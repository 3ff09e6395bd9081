"""Pass-kernel generator on the CPU host (no GPU): NVRTC compiles the
specialised sm_100a kernels of a small multi-pass plan (compile-only mode, the
same path build() uses to precompile), and the deferred-RZ phase table is in
the generated source exactly when enabled."""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import math, sys
sys.path.insert(0, sys.argv[1])
from paper_2301_03251_b200 import engine, qsim, tracer as tr
class _C:
    @staticmethod
    def current_device(): return 0
class _T:
    cuda = _C
engine._torch = lambda: _T
n = 11
def b(inputs, params):
    c = qsim.Circuit(n)
    k = 0
    for _ in range(3):
        for q in range(n):
            c.ry(q, params[k]); c.rz(q, params[k + 1]); k += 2
        for q in range(n - 1):
            c.cnot(q, q + 1)
    c.cz(0, 5)
    c.measure(0)
    return c
import numpy as np
P = 6 * n
tape, ok = tr.trace(b, np.zeros((2, 0)), np.linspace(0.1, 2.0, P))
try:
    engine.Plan(tape, 0, P, "c64", tr.classify(tape, P, [True] * P, math.pi / 2, 0.5))
except Exception:
    pass   # expected without a GPU: the cubins are already on disk
"""


def _nvrtc_available():
    import ctypes
    for name in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
        try:
            ctypes.CDLL(name)
            return True
        except OSError:
            pass
    return False


@pytest.mark.skipif(not os.path.exists(os.path.join(REPO, "paper_2301_03251_b200", "libhq.so")),
                    reason="libhq.so not built")
@pytest.mark.skipif(not _nvrtc_available(), reason="no NVRTC")
@pytest.mark.parametrize("defer", ["1", "0"])
def test_pass_kernels_compile_for_sm100a(tmp_path, defer):
    env = dict(os.environ, HQ_JIT_COMPILE_ONLY="1", HQ_JIT_CACHE=str(tmp_path / "cache"),
               HQ_JIT_DUMP=str(tmp_path / "src.cu"), HQ_FORCE_STREAM="1", HQ_TILE_BITS="9",
               HQ_DEFER_RZ=defer)
    subprocess.run([sys.executable, "-c", SCRIPT, REPO], env=env, check=True, timeout=600,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    cubins = list((tmp_path / "cache").glob("*.sm_100a.cubin"))
    assert cubins, "NVRTC produced no sm_100a cubin"
    src = (tmp_path / "src.cu").read_text()
    assert "extern \"C\" __global__" in src and "hq_b0" in src and "hq_f0" in src
    assert ("ptab_[" in src) == (defer == "1")
