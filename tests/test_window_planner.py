"""Register-window planner invariants on the host (no GPU): every window the
planner emits for the cfg4 benchmark plans -- backward windows, the 4-bit
complex128 forward windows and the schedule search's trial windows -- maps
each tile qubit to exactly one register or thread bit, keeps the lanes on
every shared-memory bank class the window's thread bits offer, and (with the
warp-slot DP) keeps warp-index slots across most transitions.

Plans are built with HQ_PLAN_ONLY (planner only, stops before the JIT) and
HQ_WIN_DEBUG (one line per window: R = register bits, S = thread bits,
lanes first)."""

import os
import re
import subprocess
import sys

import pytest

from conftest import REPO

GEN = r"""
import sys, math
sys.path.insert(0, %r)
from paper_2301_03251_b200 import engine, qsim, tracer as tr, workloads as wl, templates as T
class _C:
    @staticmethod
    def current_device(): return 0
class _T: cuda = _C
engine._torch = lambda: _T
cfg, prec = sys.argv[1], sys.argv[2]
n, d, P, _, _ = wl.CONFIGS[cfg]
b = wl.make_builder(cfg, qsim, T)
tape, ok = tr.trace(b, wl.inputs_for(cfg, 2), wl.params_for(cfg))
grad = tr.classify(tape, d + P, [False] * d + [True] * P, math.pi / 2, 0.5)
try:
    engine.Plan(tape, d, P, prec, grad)
except Exception as e:
    print("stopped:", str(e)[:80])
""" % REPO


def windows(prec, **env):
    e = dict(os.environ, HQ_PLAN_ONLY="1", HQ_WIN_DEBUG="1", HQ_JIT_COMPILE_ONLY="1", **env)
    r = subprocess.run([sys.executable, "-c", GEN, "cfg4", prec], env=e, capture_output=True, text=True, timeout=600)
    out = []
    for line in r.stderr.splitlines():
        m = re.match(r"win ops=(\d+) (\w+) R=([\d,]*) S=([\d,]*)", line)
        if m:
            out.append(([int(v) for v in m.group(3).split(",") if v], [int(v) for v in m.group(4).split(",") if v]))
    return out


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_every_window_is_a_valid_bit_assignment(prec):
    ws = windows(prec)
    assert len(ws) > 50
    for R, S in ws:
        q = len(R) + len(S)
        assert sorted(R + S) == list(range(q)), (R, S)
        lanes = S[:5]
        offered = {b & 3 for b in S}
        assert {b & 3 for b in lanes} == offered or len(lanes) < len(offered), (R, S)


def kept_fraction(ws):
    kept = total = 0
    for (R0, S0), (R1, S1) in zip(ws, ws[1:]):
        if len(R0) != len(R1) or len(S0) != len(S1) or len(S0) <= 5:
            continue
        total += 1
        kept += sum(a == b for a, b in zip(S0[5:], S1[5:]))
    return kept, total


def test_warp_slot_dp_keeps_more_warp_slots():
    # the final plan's windows only (no schedule-search trials): kept warp
    # slots between consecutive windows, DP vs the round-1 placement
    # (measured 124 vs 74 slots over 79 transitions)
    on = kept_fraction(windows("c128", HQ_PLAN_SEARCH="0"))
    off = kept_fraction(windows("c128", HQ_PLAN_SEARCH="0", HQ_KEEP_WARPS="0"))
    assert on[1] == off[1] > 0
    assert on[0] >= 1.4 * off[0], (on, off)
