"""Warp-group barrier ids of the window transitions (csrc/hq_internal.h,
hq::group_barrier_base / group_barrier_mask), checked on the host.

The generator's transitions are correct by construction only if
  * every named-barrier id in 1..15 belongs to exactly ONE warp group (one
    kept-slot pattern and one value of those slots) with one thread count, so
    a warp running ahead can never join a barrier another group still uses;
  * the pattern a transition synchronises on is a subset of the slots it
    actually keeps (a coarser group is a superset of the exchanging warps);
  * the planner's score over patterns is monotone (its DP relies on it).
Compiled with g++ against the header the JIT generator and planner use."""

import os
import shutil
import subprocess

import pytest

from conftest import REPO

SRC = r"""
#include <cstdio>
#include "hq_internal.h"
int main() {
  for (int nwarp = 0; nwarp <= 5; ++nwarp) {
    const unsigned full = (1u << nwarp) - 1u;
    int owner_pattern[16], owner_value[16], owner_count[16];
    for (int i = 0; i < 16; ++i) owner_pattern[i] = -1;
    for (unsigned m = 0; m <= full; ++m) {
      const int base = hq::group_barrier_base(nwarp, m);
      if (m == 0 || m == full) { if (base) { std::printf("FAIL base for trivial pattern\n"); return 1; } continue; }
      if (!base) continue;
      const int k = __builtin_popcount(m);
      for (int v = 0; v < (1 << k); ++v) {
        const int id = base + v;
        const int count = 32 << (nwarp - k);
        if (id < 1 || id > 15) { std::printf("FAIL id %d out of range\n", id); return 1; }
        if (owner_pattern[id] >= 0) { std::printf("FAIL id %d shared\n", id); return 1; }
        owner_pattern[id] = (int)m; owner_value[id] = v; owner_count[id] = count;
      }
    }
    for (unsigned m = 0; m <= full; ++m) {
      const unsigned g = hq::group_barrier_mask(nwarp, m);
      if ((g & ~m) != 0) { std::printf("FAIL mask not a subset\n"); return 1; }
      if (m == full && g != full) { std::printf("FAIL full pattern\n"); return 1; }
      if (g && g != full && !hq::group_barrier_base(nwarp, g)) { std::printf("FAIL mask without ids\n"); return 1; }
      for (unsigned s = m; s; s = (s - 1) & m)   // monotone score over sub-patterns
        if (__builtin_popcount(hq::group_barrier_mask(nwarp, s)) > __builtin_popcount(g)) {
          std::printf("FAIL not monotone\n"); return 1; }
    }
    int used = 0;
    for (int i = 1; i < 16; ++i) used += owner_pattern[i] >= 0;
    std::printf("nwarp %d ids %d\n", nwarp, used);
  }
  std::printf("OK\n");
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_group_barrier_ids_unique_and_monotone(tmp_path):
    src = tmp_path / "ids.cpp"
    src.write_text(SRC)
    exe = tmp_path / "ids"
    csrc = os.path.join(REPO, "paper_2301_03251_b200", "csrc")
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", csrc, "-I", cuda_inc, str(src), "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True).stdout
    assert out.strip().endswith("OK"), out
    # three warp bits (256-thread tiles): pairs on every 2-slot pattern + one 4-warp pattern
    assert "nwarp 3 ids 14" in out
