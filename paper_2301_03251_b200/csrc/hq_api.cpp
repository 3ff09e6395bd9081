// C ABI + host planner of the batched circuit simulator (see include/hq.h).
//
// Plan creation validates the tape the way the reference validates circuits
// (GateOp.__post_init__ qsim.py:54-71, Circuit.add qsim.py:109-113,
// Circuit.measure qsim.py:132-140), decides the execution path, and for the
// HBM path schedules gates into passes:
//
//   * a pass = one read + one write of the state, tile = 2^q amplitudes over q
//     "local" qubits, the low f qubits always local (contiguous 128 B runs);
//   * a gate joins the current pass when no earlier unscheduled gate shares a
//     qubit with it and its exchange qubits (targets of non-diagonal kinds) are
//     local; diagonal kinds and controls may sit on non-local qubits because
//     their bit is constant over a tile;
//   * each pass's tile and each register window's register set are chosen by
//     lookahead (the subset admitting the most upcoming gates);
//   * leading single-qubit gates fold into an analytic initial product state
//     (their gradients come from λ at the circuit start, k_fold_grad).
//
// Everything device-side of a plan lives in one cudaMalloc.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "hq_internal.h"
#include "hq_launch.h"
#include "hq_jit.h"

namespace {

thread_local std::string g_err;

hq_status fail(hq_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

constexpr int kMaxQubits = 34;
constexpr int kMaxPreps = 32;
constexpr size_t kMaxPassOps = 2048;   // bounds the per-pass trig cache in shared memory
constexpr size_t kC128PassOps = 140;   // complex128 candidate cap (see the plan builder)

bool takes_angle(int k) {
  return k == HQ_GATE_RX || k == HQ_GATE_RY || k == HQ_GATE_RZ || k == HQ_GATE_CR;
}
bool two_qubit(int k) {
  return k == HQ_GATE_CNOT || k == HQ_GATE_CZ || k == HQ_GATE_CR || k == HQ_GATE_SWAP;
}
const char* kind_name(int k) {
  static const char* names[] = {"H", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "CR", "SWAP", "STATEPREP"};
  return (k >= 0 && k <= 11) ? names[k] : "?";
}

uint64_t op_mask(const hq_op& op) {
  uint64_t m = 1ull << op.q0;
  if (two_qubit(op.kind)) m |= 1ull << op.q1;
  return m;
}
// qubits that must be resident in a tile (pairs are exchanged along them)
uint64_t exch_mask(const hq_op& op) {
  switch (op.kind) {
    case HQ_GATE_H: case HQ_GATE_X: case HQ_GATE_Y: case HQ_GATE_RX: case HQ_GATE_RY:
      return 1ull << op.q0;
    case HQ_GATE_CNOT:
      return 1ull << op.q1;
    case HQ_GATE_SWAP:
      return (1ull << op.q0) | (1ull << op.q1);
    default:
      return 0;
  }
}
int popc(uint64_t m) { return __builtin_popcountll(m); }

size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

int onchip_max_qubits(int precision) {
  if (const char* e = std::getenv("HQ_ONCHIP_MAX")) return std::atoi(e);   // test hook
  return precision == HQ_C64 ? 13 : 12;
}
int tile_bits_for(int precision) { return precision == HQ_C64 ? 12 : 11; }
int fixed_bits_for(int precision) {
  if (const char* e = std::getenv("HQ_FIXED_BITS")) return std::atoi(e);   // test hook
  // 128-byte runs: whole L2 lines per tile visit (measured: forward passes
  // 4.6 -> 5.3 TB/s on cfg4 despite 17 instead of 15 passes).  complex128
  // plans with dense passes drop to 2 fixed bits at schedule time (below).
  return precision == HQ_C64 ? 4 : 3;
}

// Streaming workspace budget (ψ checkpoints + λ per chunk of samples): larger
// chunks mean more CTAs per launch (smaller tail wave) and fewer launches —
// cfg4 B=4096: 24 GiB 4,450 -> 64 GiB 4,567 samples/s.  Default min(64 GiB,
// 35% of the device's memory), HQ_WS_BUDGET_MB overrides.
int64_t ws_budget() {
  static const int64_t dflt = [] {
    size_t fr = 0, tot = 0;
    int64_t mb = 64 * 1024;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && tot > 0)
      mb = std::min<int64_t>(mb, (int64_t)(tot * 0.35) >> 20);
    else
      cudaGetLastError();
    return std::max<int64_t>(mb, 1024);
  }();
  const char* e = std::getenv("HQ_WS_BUDGET_MB");
  int64_t mb = e ? std::atoll(e) : dflt;
  if (mb < 64) mb = 64;
  return mb << 20;
}

struct Layout {
  int64_t V = 0;
  size_t tp = 0, dpart = 0, psi = 0, lam = 0, rpart = 0, lamN = 0, locpart = 0, scratch = 0, total = 0;
  int32_t n_parts = 1;
  hq::StreamWs sws;
};

Layout layout_for(const hq_plan_s* pl, int64_t B, int32_t flags, bool need_state_only = false) {
  Layout L;
  const bool jac = (flags & HQ_WANT_JAC) != 0;
  L.V = B + (jac ? B * 2 * pl->n_tp : 0);
  const size_t amp = pl->precision == HQ_C64 ? 8 : 16;
  size_t off = 0;
  if (pl->onchip) {
    L.n_parts = hq::onchip_parts(pl);
  } else {
    const int64_t n_tiles = 1ll << (pl->n_qubits - pl->tile_bits);
    const bool adj = jac && pl->n_adj > 0;
    const int64_t per = (int64_t)amp << pl->n_qubits;
    // adjoint with specialised kernels: forward passes keep ψ checkpoints so the
    // backward passes never write ψ back (3 instead of 4 vector transfers)
    const int np = (int)pl->passes.size();
    const char* nock = std::getenv("HQ_NO_CKPT");
    if (adj && pl->jit.ok && np >= 2 && !(nock && nock[0] == '1') &&
        (int64_t)np * per <= ws_budget())
      L.sws.ckpt = np - 1;
    int64_t cs = ws_budget() / (per * (L.sws.ckpt ? L.sws.ckpt + 1 : (adj ? 2 : 1)));
    if (cs < 1) cs = 1;
    if (cs > L.V) cs = L.V;
    if (cs < 1) cs = 1;
    // equal launches instead of a small tail chunk
    if (L.V > cs) {
      const int64_t nl = (L.V + cs - 1) / cs;
      cs = (L.V + nl - 1) / nl;
    }
    int64_t want = (1184 + cs - 1) / cs;  // >= ~8 CTAs per SM per launch
    int64_t nc = 16;
    while (nc < want) nc <<= 1;
    if (nc > n_tiles) nc = n_tiles;
    L.sws.chunk_samples = cs;
    L.sws.n_chunks = (int32_t)nc;
    L.n_parts = (int32_t)nc;
    L.psi = off; off = align_up(off + (size_t)cs * per * (L.sws.ckpt ? L.sws.ckpt : 1));
    if (adj) { L.lam = off; off = align_up(off + (size_t)cs * per); }
    L.rpart = off; off = align_up(off + (size_t)cs * nc * 8);
    if (adj && pl->fold_grad) { L.lamN = off; off = align_up(off + (size_t)cs * n_tiles * 16); }
    if (adj && !pl->fold_local.empty()) {
      L.locpart = off;
      off = align_up(off + (size_t)cs * nc * pl->fold_local.size() * 32);
    }
  }
  (void)need_state_only;
  L.scratch = off; off = align_up(off + (size_t)B * 8 + 8);   // readout sink for hq_state
  if (jac) {
    L.tp = off; off = align_up(off + (size_t)B * 2 * pl->n_tp * 8 + 8);
    L.dpart = off; off = align_up(off + (size_t)B * pl->n_adj * L.n_parts * 8 + 8);
  }
  L.total = off + 256;
  return L;
}

}  // namespace

namespace hq {
hq_status fail_status(hq_status s, const std::string& msg) { return fail(s, msg); }
static std::atomic<int64_t> g_launch_count[HQ_K_CLASSES];
void count_launch(int cls) {
  if (cls >= 0 && cls < HQ_K_CLASSES) g_launch_count[cls].fetch_add(1, std::memory_order_relaxed);
}
}  // namespace hq

extern "C" void hq_launch_counts(int64_t* out) {
  for (int k = 0; k < HQ_K_CLASSES; ++k) out[k] = hq::g_launch_count[k].load(std::memory_order_relaxed);
}

extern "C" int hq_abi_version(void) { return HQ_ABI_VERSION; }
extern "C" const char* hq_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------------------
static hq_status validate(const hq_plan_desc* d) {
  if (!d) return fail(HQ_E_CONFIG, "null plan descriptor");
  if (d->n_qubits < 1 || d->n_qubits > kMaxQubits)
    return fail(HQ_E_CIRCUIT, "n_qubits must be in 1.." + std::to_string(kMaxQubits) + ", got " +
                                  std::to_string(d->n_qubits));
  if (d->precision != HQ_C64 && d->precision != HQ_C128) return fail(HQ_E_CONFIG, "unknown precision");
  if (d->n_ops < 0 || (d->n_ops > 0 && !d->ops)) return fail(HQ_E_CONFIG, "bad op array");
  if (d->n_slots < 0 || (d->n_slots > 0 && (!d->slot_const || !d->slot_ptr)))
    return fail(HQ_E_CONFIG, "bad slot table");
  if (d->n_inputs < 0 || d->n_params < 0) return fail(HQ_E_CONFIG, "negative variable count");
  const int nvars = d->n_inputs + d->n_params;
  if (d->n_slots > 0) {
    if (d->slot_ptr[0] != 0) return fail(HQ_E_CONFIG, "slot_ptr[0] must be 0");
    for (int s = 0; s < d->n_slots; ++s) {
      if (d->slot_ptr[s + 1] < d->slot_ptr[s]) return fail(HQ_E_CONFIG, "slot_ptr not monotone");
      for (int k = d->slot_ptr[s]; k < d->slot_ptr[s + 1]; ++k)
        if (d->slot_var[k] < 0 || d->slot_var[k] >= nvars) return fail(HQ_E_CONFIG, "slot variable out of range");
    }
  }
  if (d->n_preps < 0 || d->n_preps > kMaxPreps) return fail(HQ_E_CONFIG, "too many state loads");
  for (int p = 0; p < d->n_preps; ++p) {
    const int q0 = d->prep_ptr[p], q1 = d->prep_ptr[p + 1];
    if (q1 <= q0) return fail(HQ_E_CIRCUIT, "empty state load");
    uint64_t m = 0;
    for (int k = q0; k < q1; ++k) {
      const int q = d->prep_qubits[k];
      if (q < 0 || q >= d->n_qubits) return fail(HQ_E_CIRCUIT, "state-load qubit out of range");
      if (m & (1ull << q)) return fail(HQ_E_CIRCUIT, "duplicate qubit in state load");
      m |= 1ull << q;
    }
    if (d->prep_len[p] < 1 || (int64_t)d->prep_len[p] > (1ll << (q1 - q0)))
      return fail(HQ_E_ENCODING, "state-load vector exceeds its qubits");
    if (d->prep_slot0[p] < 0 || d->prep_slot0[p] + d->prep_len[p] > d->n_slots)
      return fail(HQ_E_CONFIG, "state-load slots out of range");
  }
  for (int i = 0; i < d->n_ops; ++i) {
    const hq_op& op = d->ops[i];
    if (op.kind < 0 || op.kind > HQ_GATE_STATEPREP)
      return fail(HQ_E_CIRCUIT, "unknown gate kind " + std::to_string(op.kind));
    if (op.kind == HQ_GATE_STATEPREP) {
      if (op.q0 < 0 || op.q0 >= d->n_preps) return fail(HQ_E_CONFIG, "bad state-load index");
      continue;
    }
    if (op.q0 < 0 || op.q0 >= d->n_qubits)
      return fail(HQ_E_CIRCUIT, std::string(kind_name(op.kind)) + " targets exceed " +
                                    std::to_string(d->n_qubits) + " qubits");
    if (two_qubit(op.kind)) {
      if (op.q1 < 0 || op.q1 >= d->n_qubits)
        return fail(HQ_E_CIRCUIT, std::string(kind_name(op.kind)) + " targets exceed " +
                                      std::to_string(d->n_qubits) + " qubits");
      if (op.q1 == op.q0) return fail(HQ_E_CIRCUIT, std::string("duplicate targets in ") + kind_name(op.kind));
    }
    if (takes_angle(op.kind)) {
      if (op.slot < 0 || op.slot >= d->n_slots) return fail(HQ_E_CIRCUIT, std::string(kind_name(op.kind)) + " requires one finite angle");
    } else if (op.slot >= 0) {
      return fail(HQ_E_CIRCUIT, std::string(kind_name(op.kind)) + " takes no angle");
    }
  }
  if (d->n_measured < 0 || (d->n_measured > 0 && !d->measured)) return fail(HQ_E_CONFIG, "bad measured list");
  uint64_t mm = 0;
  for (int i = 0; i < d->n_measured; ++i) {
    const int q = d->measured[i];
    if (q < 0 || q >= d->n_qubits) return fail(HQ_E_CIRCUIT, "measured qubit " + std::to_string(q) + " out of range");
    if (mm & (1ull << q)) return fail(HQ_E_CIRCUIT, "qubit " + std::to_string(q) + " measured twice");
    mm |= 1ull << q;
  }
  if (d->grad_mode) {
    for (int v = 0; v < nvars; ++v) {
      const int m = d->grad_mode[v];
      if (m < HQ_GRAD_ZERO || m > HQ_GRAD_TWOPOINT) return fail(HQ_E_CONFIG, "bad gradient mode");
      if (m == HQ_GRAD_ADJOINT && (d->grad_slot[v] < 0 || d->grad_slot[v] >= d->n_slots))
        return fail(HQ_E_CONFIG, "adjoint variable without a slot");
    }
  }
  if (!(d->shift > 0.0)) return fail(HQ_E_CONFIG, "shift must be positive");
  return HQ_OK;
}

namespace {

// Greedy pass scheduler (see file comment).
// excl0: qubits that must stay out of the first pass's tile (their folded
// gates' gradients are read from λ contracted over that tile)
std::vector<hq::Pass> schedule_passes(const std::vector<hq_op>& ops, int n, int q, int f, uint64_t excl0 = 0,
                                      size_t op_cap = kMaxPassOps, size_t first_cap = 0) {
  std::vector<hq::Pass> passes;
  std::vector<char> done(ops.size(), 0);
  size_t left = ops.size();
  const uint64_t fixed = (f >= 64) ? ~0ull : ((1ull << f) - 1);
  // Tile choice by lookahead (HQ_PASS_LOOKAHEAD=0: first-come greedy + lowest-
  // qubit top-up): cfg4 17 -> 8 passes, 4,676 -> 5,646 samples/s
  size_t max_ops = op_cap;   // HQ_MAX_PASS_OPS: test hook (code size per pass kernel)
  if (const char* e = std::getenv("HQ_MAX_PASS_OPS")) max_ops = std::max<size_t>(8, std::min<size_t>(kMaxPassOps, std::atoll(e)));
  // HQ_FIRST_PASS_OPS: cap of the first pass only (its kernels are the largest)
  size_t first_ops = first_cap ? std::min(first_cap, max_ops) : max_ops;
  // HQ_PASS_CAPS="c0,c1,...": per-pass op caps (planner experiments; 0 = none)
  std::vector<size_t> pass_caps;
  if (const char* e = std::getenv("HQ_PASS_CAPS")) {
    std::string v(e);
    size_t p0 = 0;
    while (p0 <= v.size()) {
      const size_t p1 = v.find(',', p0);
      pass_caps.push_back((size_t)std::atoll(v.substr(p0, p1 == std::string::npos ? std::string::npos : p1 - p0).c_str()));
      if (p1 == std::string::npos) break;
      p0 = p1 + 1;
    }
    if (!pass_caps.empty() && pass_caps[0]) first_ops = pass_caps[0];
  }
  if (const char* e = std::getenv("HQ_FIRST_PASS_OPS")) first_ops = std::max<size_t>(8, std::min<size_t>(max_ops, std::atoll(e)));
  const char* pla = std::getenv("HQ_PASS_LOOKAHEAD");
  const bool lookahead = !(pla && pla[0] == '0');
  const bool depth2 = pla && pla[0] == '2';
  const int need = q - popc(fixed);
  const uint64_t allq = n >= 64 ? ~0ull : ((1ull << n) - 1);
  // ops admitted by tile Lc given the finished set d (first-come blocking)
  auto admit = [&](uint64_t Lc, std::vector<char>& d, bool mark) {
    long cnt = 0;
    uint64_t blocked = 0;
    for (size_t k = 0; k < ops.size() && blocked != allq; ++k) {
      if (d[k]) continue;
      const uint64_t qs = op_mask(ops[k]);
      if (qs & blocked) { blocked |= qs; continue; }
      if ((exch_mask(ops[k]) & ~Lc) == 0) {
        ++cnt;
        if (mark) d[k] = 1;
      } else {
        blocked |= qs;
      }
    }
    return cnt;
  };
  // every candidate tile (fixed + (q-f)-subset of the next ops' exchange qubits,
  // up to 16 candidates) with its admitted count, best first
  auto tiles = [&](std::vector<char>& d, uint64_t ex0) {
    std::vector<std::pair<long, uint64_t>> out;
    uint64_t cand = 0;
    for (size_t k = 0; k < ops.size() && popc(cand) < 16; ++k) {
      if (d[k]) continue;
      const uint64_t ex = exch_mask(ops[k]) & ~fixed & ~ex0;
      if (popc(cand | ex) > 16) break;
      cand |= ex;
    }
    std::vector<int> cb;
    for (int b = 0; b < n; ++b)
      if (cand >> b & 1ull) cb.push_back(b);
    const int nc = (int)cb.size();
    if (nc <= need || nc > 18) return out;
    std::vector<int> idx(need);
    for (int i = 0; i < need; ++i) idx[i] = i;
    while (true) {
      uint64_t Lc = fixed;
      for (int i : idx) Lc |= 1ull << cb[i];
      out.push_back({admit(Lc, d, false), Lc});
      int i = need - 1;
      while (i >= 0 && idx[i] == nc - need + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int j = i + 1; j < need; ++j) idx[j] = idx[j - 1] + 1;
    }
    std::stable_sort(out.begin(), out.end(), [](const std::pair<long, uint64_t>& x,
                                                 const std::pair<long, uint64_t>& y) { return x.first > y.first; });
    return out;
  };
  // Beam search over whole tile sequences (width 4, 6 expansions per state):
  // the schedule with the fewest passes wins.
  std::vector<uint64_t> beam_tiles;
  // opt-in (HQ_PASS_BEAM=1): on cfg4 / cfg5 it finds the greedy lookahead's
  // schedule again at 1.5-2.5x the planning time
  const char* pb = std::getenv("HQ_PASS_BEAM");
  if (lookahead && pb && pb[0] == '1' && max_ops >= ops.size()) {
    struct St { std::vector<char> d; size_t left; std::vector<uint64_t> t; };
    std::vector<St> beam{St{done, left, {}}};
    bool ok = true;
    for (int level = 0; ok && level < 64; ++level) {
      bool all_done = true;
      std::vector<St> nxt;
      for (auto& st : beam) {
        if (st.left == 0) { nxt.push_back(st); continue; }
        all_done = false;
        auto cands = tiles(st.d, level == 0 ? excl0 : 0);
        if (cands.empty()) { ok = false; break; }
        for (size_t c = 0; c < cands.size() && c < 6; ++c) {
          St ns{st.d, st.left, st.t};
          ns.left -= (size_t)admit(cands[c].second, ns.d, true);
          ns.t.push_back(cands[c].second);
          nxt.push_back(std::move(ns));
        }
      }
      if (!ok || all_done) break;
      std::stable_sort(nxt.begin(), nxt.end(), [](const St& a, const St& b) { return a.left < b.left; });
      beam.clear();
      for (auto& st : nxt) {
        bool dup = false;
        for (auto& b2 : beam) dup |= b2.d == st.d;
        if (!dup) beam.push_back(std::move(st));
        if (beam.size() == 4) break;
      }
    }
    if (ok) {
      size_t bi = 0;
      for (size_t i = 0; i < beam.size(); ++i)
        if (beam[i].left == 0 && (beam[bi].left != 0 || beam[i].t.size() < beam[bi].t.size())) bi = i;
      if (beam[bi].left == 0) beam_tiles = beam[bi].t;
    }
  }
  while (left > 0) {
    uint64_t L = fixed;
    hq::Pass ps;
    bool progress = true;
    bool first_scan = true;
    if (passes.size() < beam_tiles.size()) {
      L = beam_tiles[passes.size()];
      first_scan = false;
    } else if (lookahead) {
      // tile = fixed bits + the candidate subset admitting the most ops; depth 2
      // (HQ_PASS_LOOKAHEAD=2) adds the best follow-up pass's count for the top 6
      const uint64_t excl = passes.empty() ? excl0 : 0;
      auto lv1 = tiles(done, excl);
      if (!lv1.empty()) {
        long best = lv1[0].first;
        uint64_t bestL = lv1[0].second;
        if (depth2) {
          long best_tot = -1;
          for (size_t c = 0; c < lv1.size() && c < 6; ++c) {
            std::vector<char> d2 = done;
            const long s1 = admit(lv1[c].second, d2, true);
            long s2 = 0;
            for (const auto& t : tiles(d2, 0)) s2 = std::max(s2, t.first);
            if (s1 + s2 > best_tot) { best_tot = s1 + s2; best = s1; bestL = lv1[c].second; }
          }
        }
        if (best > 0) { L = bestL; first_scan = false; }
      }
    }
    while (progress) {
      progress = false;
      uint64_t blocked = 0;
      for (size_t k = 0; k < ops.size(); ++k) {
        if (done[k]) continue;
        const uint64_t qs = op_mask(ops[k]);
        if (qs & blocked) { blocked |= qs; continue; }
        const uint64_t ex = exch_mask(ops[k]);
        if (ps.op_ids.size() >= (passes.empty() ? first_ops : (passes.size() < pass_caps.size() && pass_caps[passes.size()]
                                                                   ? pass_caps[passes.size()] : max_ops))) {
          blocked |= qs;
          continue;
        }
        const uint64_t excl = passes.empty() ? excl0 : 0;
        if (!(ex & excl) && ((ex & ~L) == 0 || popc(L | ex) <= q)) {
          L |= ex;
          done[k] = 1;
          --left;
          ps.op_ids.push_back((int32_t)k);
          progress = true;
        } else {
          blocked |= qs;
        }
      }
      if (first_scan) {
        // top up the tile with the lowest remaining qubits, then rescan
        for (int b = 0; b < n && popc(L) < q; ++b)
          if (!((passes.empty() ? excl0 : 0) >> b & 1ull)) L |= 1ull << b;
        first_scan = false;
        progress = true;
      }
    }
    for (int b = 0; b < n; ++b)
      if (L & (1ull << b)) ps.local.push_back(b);
    passes.push_back(std::move(ps));
  }
  if (passes.empty()) {
    hq::Pass ps;
    for (int b = 0; b < q; ++b) ps.local.push_back(b);
    passes.push_back(std::move(ps));
  }
  return passes;
}

// register bits per thread in the streaming kernels (must match hq_stream.cu RBits)
int reg_bits_for(int precision) { return precision == HQ_C64 ? 4 : 3; }
#define RBITS(p) reg_bits_for(p)

uint16_t swz_host(uint32_t j) { return (uint16_t)(j ^ (((j >> 4) ^ (j >> 8)) & 15u)); }

// Split one pass's ops (tile-bit operands) into register windows (see
// hq_window.cuh): same greedy as the pass scheduler, capacity kRegBits, over
// the exchange qubits; controls / diagonal qubits may be thread bits.
void plan_windows(hq::Pass& ps, const std::vector<hq::DOp>& ops, int q, int RB, int fixed, bool rollout = true,
                  bool warp_local = false) {
  auto exch = [](const hq::DOp& o) -> uint32_t {
    switch (o.kind) {
      case HQ_GATE_H: case HQ_GATE_X: case HQ_GATE_Y: case HQ_GATE_RX: case HQ_GATE_RY:
        return 1u << o.a;
      case HQ_GATE_CNOT:
        return 1u << o.b;
      default:
        return 0u;
    }
  };
  auto qmask = [](const hq::DOp& o) -> uint32_t {
    uint32_t m = 0;
    if (o.a >= 0) m |= 1u << o.a;
    if (o.b >= 0) m |= 1u << o.b;
    return m;
  };
  std::vector<int> dl(ops.size(), -1);
  int ndl = 0;
  for (size_t k = 0; k < ops.size(); ++k)
    if (ops[k].dslot >= 0) dl[k] = ndl++;
  std::vector<char> done(ops.size(), 0);
  size_t left = ops.size();
  const uint32_t all = (q >= 32) ? ~0u : ((1u << q) - 1);
  // Register set of a window: every RB-subset of the exchange qubits the next
  // ops need is tried and the one that admits the most ops wins (first-come
  // greedy as the fallback: HQ_WIN_GREEDY=1).  Sets that would take every tile
  // bit of a bank class out of the thread bits are skipped.
  const char* wg = std::getenv("HQ_WIN_GREEDY");
  const bool lookahead = !(wg && wg[0] == '1');
  // Shuffle transitions (generator: hq_jit.cpp): a window whose register bits
  // differ from the previous window's only by qubits that were LANE bits there
  // is reached with warp shuffles (each swapped bit moves half of a thread's
  // amplitudes to the partner lane; no shared-memory round trip, no barrier).
  // The lookahead prefers such register sets by kShflBonus score points
  // (= half an admitted op each).
  const bool shfl = hq::shfl_enabled();
  // (default for both precisions: complex64 -2.8% with the warp-group
  // transitions, measured with one compiler -- profiles/r02_compiler_ab.log)
  bool keep_warps = warp_local;
  if (const char* e = std::getenv("HQ_KEEP_WARPS")) keep_warps = std::atoi(e) != 0;
  int shfl_bonus = 3;
  if (const char* e = std::getenv("HQ_SHFL_BONUS")) shfl_bonus = std::atoi(e);
  std::vector<int> pR, pS;            // previous window's register / thread bits
  bool have_prev = false;
  const int n_lanes = std::min(5, q - RB);
  auto lane_mask_prev = [&]() {
    uint32_t m = 0;
    for (int s2 = 0; s2 < n_lanes && s2 < (int)pS.size(); ++s2) m |= 1u << pS[s2];
    return m;
  };
  auto reg_mask_prev = [&]() {
    uint32_t m = 0;
    for (int b : pR) m |= 1u << b;
    return m;
  };
  auto shfl_able = [&](uint32_t R) {
    return shfl && have_prev && (R & ~reg_mask_prev() & ~lane_mask_prev()) == 0;
  };
  auto class_ok = [&](uint32_t m) {
    for (int cls = 0; cls < 4; ++cls) {
      int c = 0, tot = 0;
      for (int b = 0; b < q; ++b)
        if ((b & 3) == cls) { ++tot; if (!(m >> b & 1u)) ++c; }
      if (tot > 0 && c == 0) return false;
    }
    return true;
  };
  auto admitted_in = [&](uint32_t R, const std::vector<char>& dn) {
    int cnt = 0;
    uint32_t blocked = 0;
    for (size_t k = 0; k < ops.size(); ++k) {
      if (dn[k]) continue;
      const uint32_t qs = qmask(ops[k]);
      if (qs & blocked) { blocked |= qs; continue; }
      if ((exch(ops[k]) & ~R) == 0) ++cnt;
      else blocked |= qs;
    }
    return cnt;
  };
  auto admitted = [&](uint32_t R) { return admitted_in(R, done); };
  const uint32_t fmask_all = fixed >= 32 ? ~0u : ((1u << fixed) - 1u);
  // lookahead candidates: (score, register set), best first
  auto candidates = [&](const std::vector<char>& dn, bool with_shfl) {
    std::vector<std::pair<int, uint32_t>> out;
    uint32_t cand = 0;
    int seen = 0;
    for (size_t k = 0; k < ops.size() && seen < 48; ++k)
      if (!dn[k]) { cand |= exch(ops[k]); ++seen; }
    std::vector<int> cb;
    for (int b = 0; b < q; ++b)
      if (cand >> b & 1u) cb.push_back(b);
    if ((int)cb.size() <= RB || cb.size() > 16) return out;
    const int nc = (int)cb.size();
    for (uint32_t sel = 0; sel < (1u << nc); ++sel) {
      if (popc(sel) != RB) continue;
      uint32_t R = 0;
      for (int i = 0; i < nc; ++i)
        if (sel >> i & 1u) R |= 1u << cb[i];
      if (!class_ok(R)) continue;
      const int sc = 2 * admitted_in(R, dn) + ((R & fmask_all) ? 0 : 1) + (with_shfl && shfl_able(R) ? shfl_bonus : 0);
      if (sc > 1) out.push_back({sc, R});
    }
    std::stable_sort(out.begin(), out.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    return out;
  };
  auto class_left_of = [&](uint32_t m, int cls) {
    int c = 0;
    for (int b = 0; b < q; ++b)
      if (!(m >> b & 1u) && (b & 3) == cls) ++c;
    return c;
  };
  // admit ops into a window with register set Rm (scan, top-up, rescan) — the
  // rollout's copy of the main loop below, without emitting anything
  auto admit_sim = [&](uint32_t Rm, std::vector<char>& dn) {
    bool progress = true, first_scan = true;
    size_t n_adm = 0;
    while (progress) {
      progress = false;
      uint32_t blocked = 0;
      for (size_t k = 0; k < ops.size(); ++k) {
        if (dn[k]) continue;
        const uint32_t qs = qmask(ops[k]);
        if (qs & blocked) { blocked |= qs; continue; }
        const uint32_t ex = exch(ops[k]);
        if ((ex & ~Rm) == 0 || popc(Rm | ex) <= RB) { Rm |= ex; dn[k] = 1; ++n_adm; progress = true; }
        else blocked |= qs;
      }
      if (first_scan) {
        for (int pass2 = 0; pass2 < 2; ++pass2)
          for (int b = q - 1; b >= 0 && popc(Rm) < RB; --b)
            if (!(Rm >> b & 1u) && (pass2 == 1 || class_left_of(Rm, b & 3) > 1)) Rm |= 1u << b;
        first_scan = false;
        progress = true;
      }
    }
    return n_adm;
  };
  // windows the greedy lookahead needs to finish from state dn
  auto rollout_windows = [&](std::vector<char> dn) {
    int w = 0;
    for (;;) {
      bool any = false;
      for (char c : dn) if (!c) { any = true; break; }
      if (!any) return w;
      auto cs = candidates(dn, false);
      if (admit_sim(cs.empty() ? 0u : cs[0].second, dn) == 0) return w + 1000;   // no progress: give up
      ++w;
    }
  };
  // Window rollouts (opt-in, HQ_WIN_ROLLOUT = number of candidates): the best
  // few lookahead register sets are each followed by a greedy rollout of the
  // rest of the pass and the one finishing in the fewest windows wins.  On
  // cfg4 the lookahead is already at the rollout optimum (c128: same 53
  // windows with 4 or 8 candidates; c64: 34 -> 33), so it stays off.
  int n_roll = 0;
  if (const char* e = std::getenv("HQ_WIN_ROLLOUT")) n_roll = std::atoi(e);
  if (!rollout || shfl) n_roll = 0;
  struct WinTmp {
    uint32_t Rm = 0, ctl = 0;
    std::vector<int> R, S;
    std::vector<size_t> exec;
    bool shuffled = false;
  };
  std::vector<WinTmp> wins;
  // thread bits of a window: lanes first (one per bank class, the fixed bits
  // in their own slots, CNOT controls kept for the warp bits), then the warp
  // bits -- the set W when given (ascending, so equal sets get equal slots)
  auto thread_bits = [&](const WinTmp& wt, const std::vector<int>& W) {
    uint32_t Wm = 0;
    for (int b : W) Wm |= 1u << b;
    std::vector<int> S, rest;
    for (int b = 0; b < q; ++b)
      if (!(wt.Rm >> b & 1u)) rest.push_back(b);
    std::vector<char> used(rest.size(), 0);
    for (size_t i = 0; i < rest.size(); ++i) used[i] = (Wm >> rest[i] & 1u) ? 1 : 0;
    auto pick = [&](int cls) {   // lane bit of bank class cls (-1: any class)
      int best = -1;
      for (size_t i = 0; i < rest.size(); ++i) {
        if (used[i] || (cls >= 0 && (rest[i] & 3) != cls)) continue;
        if (rest[i] < fixed) { best = (int)i; break; }
        const bool c = wt.ctl >> rest[i] & 1u;
        if (best < 0 || (!c && (wt.ctl >> rest[best] & 1u))) best = (int)i;
        if (!c) break;
      }
      if (best >= 0) { S.push_back(rest[best]); used[best] = 1; }
    };
    for (int cls = 0; cls < 4 && (int)S.size() < 5; ++cls) pick(cls);
    while ((int)S.size() < 5 && S.size() < rest.size()) {
      const size_t before = S.size();
      pick(-1);
      if (S.size() == before) break;
    }
    for (size_t i = 0; i < rest.size(); ++i)
      if (!used[i]) S.push_back(rest[i]);
    S.insert(S.end(), W.begin(), W.end());
    return S;
  };
  do {
    uint32_t Rm = 0;
    if (lookahead && n_roll > 1) {
      auto cs = candidates(done, false);
      int best_w = 1 << 30, best_sc = -1;
      for (int c = 0; c < (int)cs.size() && c < n_roll; ++c) {
        std::vector<char> dn(done);
        if (admit_sim(cs[c].second, dn) == 0) continue;
        const int w = 1 + rollout_windows(dn);
        if (w < best_w || (w == best_w && cs[c].first > best_sc)) { best_w = w; best_sc = cs[c].first; Rm = cs[c].second; }
      }
    } else if (lookahead) {
      uint32_t cand = 0;
      int seen = 0;
      for (size_t k = 0; k < ops.size() && seen < 48; ++k)
        if (!done[k]) { cand |= exch(ops[k]); ++seen; }
      std::vector<int> cb;
      for (int b = 0; b < q; ++b)
        if (cand >> b & 1u) cb.push_back(b);
      if ((int)cb.size() > RB && cb.size() <= 16) {
        int best = -1;
        uint32_t bestR = 0;
        const int nc = (int)cb.size();
        for (uint32_t sel = 0; sel < (1u << nc); ++sel) {
          if (popc(sel) != RB) continue;
          uint32_t R = 0;
          for (int i = 0; i < nc; ++i)
            if (sel >> i & 1u) R |= 1u << cb[i];
          if (!class_ok(R)) continue;
          // ties: keep the fixed low bits (HBM-contiguous lanes) out of the registers
          const uint32_t fmask = fixed >= 32 ? ~0u : ((1u << fixed) - 1u);
          const int sc = 2 * admitted(R) + ((R & fmask) ? 0 : 1) + (shfl_able(R) ? shfl_bonus : 0);
          if (sc > best) { best = sc; bestR = R; }
        }
        if (best > 1) Rm = bestR;
      }
    }
    std::vector<size_t> exec;
    bool progress = true, first_scan = true;
    while (progress) {
      progress = false;
      uint32_t blocked = 0;
      for (size_t k = 0; k < ops.size(); ++k) {
        if (done[k]) continue;
        const uint32_t qs = qmask(ops[k]);
        if (qs & blocked) { blocked |= qs; continue; }
        const uint32_t ex = exch(ops[k]);
        if ((ex & ~Rm) == 0 || popc(Rm | ex) <= RB) {
          Rm |= ex;
          done[k] = 1;
          --left;
          exec.push_back(k);
          progress = true;
        } else {
          blocked |= qs;
        }
      }
      if (first_scan) {
        // top up the register bits, keeping at least one thread bit in each of
        // the 4 bank classes (b & 3) so window loads/stores stay conflict-free
        auto class_left = [&](uint32_t m, int cls) {
          int c = 0;
          for (int b = 0; b < q; ++b)
            if (!(m >> b & 1u) && (b & 3) == cls) ++c;
          return c;
        };
        // (shuffle transitions: the previous window's register bits first,
        // then its lane bits, so the transition stays a set of lane swaps)
        if (shfl && have_prev) {
          const uint32_t pref[2] = {reg_mask_prev(), lane_mask_prev()};
          for (uint32_t pm : pref)
            for (int b = q - 1; b >= 0 && popc(Rm) < RB; --b)
              if ((pm >> b & 1u) && !(Rm >> b & 1u) && class_left(Rm, b & 3) > 1) Rm |= 1u << b;
        }
        for (int pass2 = 0; pass2 < 2; ++pass2)
          for (int b = q - 1; b >= 0 && popc(Rm) < RB; --b)
            if (!(Rm >> b & 1u) && (pass2 == 1 || class_left(Rm, b & 3) > 1)) Rm |= 1u << b;
        first_scan = false;
        progress = true;
      }
    }
    // register bits, then thread bits: lanes first, covering all 4 bank
    // classes.  Controls of CNOTs whose control is not a register bit go to
    // warp bits where possible (warp-uniform branch instead of FSEL swaps);
    // bits below `fixed` keep their lane slots (direct HBM windows).
    WinTmp wt;
    wt.Rm = Rm;
    wt.exec = exec;
    for (size_t k : exec)
      if (ops[k].kind == HQ_GATE_CNOT && ops[k].a >= 0 && !(Rm >> ops[k].a & 1u)) wt.ctl |= 1u << ops[k].a;
    for (int b = 0; b < q; ++b)
      if (Rm >> b & 1u) wt.R.push_back(b);
    if (shfl_able(Rm)) {
      // keep the previous thread-bit slots; each qubit entering the registers
      // from lane slot s hands that slot to a qubit leaving the registers
      std::vector<int> S2(pS), out;
      for (int b : pR)
        if (!(Rm >> b & 1u)) out.push_back(b);
      size_t oi = 0;
      for (int s2 = 0; s2 < n_lanes; ++s2)
        if (Rm >> S2[s2] & 1u) S2[s2] = out[oi++];
      int cls = 0;
      for (int s2 = 0; s2 < n_lanes; ++s2) cls |= 1 << (S2[s2] & 3);
      if (oi == out.size() && (cls == 15 || q - RB < 5)) {
        wt.S = S2;
        wt.shuffled = true;
      }
    }
    if (!wt.shuffled && (shfl || !keep_warps)) wt.S = thread_bits(wt, {});
    pR = wt.R;
    pS = wt.S;
    have_prev = true;
    wins.push_back(wt);
  } while (left > 0);

  // Warp-local transitions (complex128 default; HQ_KEEP_WARPS=0/1 overrides):
  // the warp-index bits of each window are chosen over the whole pass so that
  // consecutive windows keep as many of them as possible in the same warp-bit
  // slots.  The shared-memory exchange between two windows then only crosses
  // warps that differ in the changed slots: all kept -> inside each warp
  // (__syncwarp), some kept -> within groups of 2 or 4 warps (named barriers),
  // none -> the whole CTA (hq_jit.cpp, post_store_sync).  DP over the window
  // sequence: state = the ordered warp-bit tuple W (disjoint from the window's
  // register bits and the fixed bits, leaving lanes that still cover every
  // bank class); score per transition 16·kept/nwarp + the CNOT controls W
  // covers (warp-uniform branches).
  if (!shfl && keep_warps && !wins.empty() && q - RB > n_lanes) {
    const int nwarp = q - RB - n_lanes;
    std::vector<int> free_bits;
    for (int b = 0; b < q; ++b)
      if (!(fmask_all >> b & 1u)) free_bits.push_back(b);
    // ordered tuples (sorted sets only when there would be too many)
    size_t n_ord = 1;
    for (int i = 0; i < nwarp; ++i) n_ord *= (free_bits.size() > (size_t)i ? free_bits.size() - i : 0);
    const bool ordered = n_ord <= 1500;
    std::vector<std::vector<int>> cand;
    std::vector<int> cur;
    std::function<void(uint32_t)> gen = [&](uint32_t usedm) {
      if ((int)cur.size() == nwarp) { cand.push_back(cur); return; }
      for (int b : free_bits) {
        if (usedm >> b & 1u) continue;
        if (!ordered && !cur.empty() && b < cur.back()) continue;
        cur.push_back(b);
        gen(usedm | 1u << b);
        cur.pop_back();
      }
    };
    gen(0u);
    auto classes = [&](uint32_t m) {
      int c = 0;
      for (int b = 0; b < q; ++b)
        if (m >> b & 1u) c |= 1 << (b & 3);
      return c;
    };
    const size_t K = wins.size(), C = cand.size();
    std::vector<uint32_t> cmask(C, 0u);
    for (size_t c = 0; c < C; ++c)
      for (int b : cand[c]) cmask[c] |= 1u << b;
    const int NEG = -(1 << 28);
    std::vector<std::vector<int>> dp(K, std::vector<int>(C, NEG)), from(K, std::vector<int>(C, -1));
    // transition score by the exactly-kept slot pattern (via the barrier group
    // it can use); the previous windows' best per (pattern, kept qubits) makes
    // each step O(C · 2^nwarp) instead of O(C²)
    const uint32_t nmask = 1u << nwarp;
    std::vector<int> score(nmask, 0);
    for (uint32_t m = 0; m < nmask; ++m) score[m] = 16 * popc(hq::group_barrier_mask(nwarp, m)) / nwarp;
    auto key = [&](size_t c, uint32_t m) {
      uint32_t k2 = 0;
      for (int i = 0; i < nwarp; ++i)
        if (m >> i & 1u) k2 = k2 * 32u + (uint32_t)cand[c][i] + 1u;
      return k2;
    };
    for (size_t k = 0; k < K; ++k) {
      const uint32_t restm = all & ~wins[k].Rm;
      // best previous value per (sub-pattern m, its qubits): a previous tuple
      // agreeing with c on at least m's slots scores at least score[m], and
      // score is monotone over sub-patterns, so the max over m is exact
      std::vector<std::unordered_map<uint32_t, std::pair<int, int>>> best(nmask);
      if (k > 0)
        for (size_t c2 = 0; c2 < C; ++c2) {
          if (dp[k - 1][c2] <= NEG) continue;
          for (uint32_t m = 0; m < nmask; ++m) {
            auto& e = best[m].try_emplace(key(c2, m), NEG, -1).first->second;
            if (dp[k - 1][c2] > e.first) e = {dp[k - 1][c2], (int)c2};
          }
        }
      for (size_t c = 0; c < C; ++c) {
        if ((cmask[c] & wins[k].Rm) || classes(restm & ~cmask[c]) != classes(restm)) continue;
        const int own = popc(cmask[c] & wins[k].ctl);
        if (k == 0) { dp[k][c] = own; continue; }
        int v = NEG, f = -1;
        for (uint32_t m = 0; m < nmask; ++m) {
          auto it = best[m].find(key(c, m));
          if (it == best[m].end() || it->second.second < 0) continue;
          if (it->second.first + score[m] > v) { v = it->second.first + score[m]; f = it->second.second; }
        }
        if (f < 0) { dp[k][c] = own; continue; }   // previous window had no valid tuple: restart
        dp[k][c] = v + own;
        from[k][c] = f;
      }
    }
    // backtrack; a chain break (a window without any valid tuple) falls back
    // to the default placement there and restarts from the best earlier state
    std::vector<std::vector<int>> Wsel(K);
    int c = -1;
    for (size_t k = K; k-- > 0;) {
      if (c < 0) {
        int bv = NEG;
        for (size_t i = 0; i < C; ++i)
          if (dp[k][i] > bv) { bv = dp[k][i]; c = (int)i; }
      }
      if (c < 0) continue;
      Wsel[k] = cand[c];
      c = from[k][c];
    }
    for (size_t k = 0; k < K; ++k) wins[k].S = thread_bits(wins[k], Wsel[k]);
  }
  // no warp-index bits (one warp per tile): the default placement
  for (WinTmp& wt : wins)
    if (wt.S.empty()) wt.S = thread_bits(wt, {});

  for (const WinTmp& wt : wins) {
    const std::vector<int>& R = wt.R;
    const std::vector<int>& S = wt.S;
    if (std::getenv("HQ_WIN_DEBUG")) {
      std::fprintf(stderr, "win ops=%zu %s R=", wt.exec.size(), wt.shuffled ? "shfl" : "smem");
      for (int b : R) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, " S=");
      for (int b : S) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, "\n");
    }
    hq::WinHost w{};
    w.op0 = (int16_t)ps.wops.size();
    for (int i = 0; i < RB && i < 6; ++i) w.pr[i] = swz_host(1u << R[i]);
    for (size_t s2 = 0; s2 < S.size() && s2 < 10; ++s2) w.ps[s2] = swz_host(1u << S[s2]);
    auto code = [&](int x) -> int8_t {
      if (x < 0) return (int8_t)(64 + ~x);
      for (int i = 0; i < RB; ++i) if (R[i] == x) return (int8_t)i;
      for (size_t i = 0; i < S.size(); ++i) if (S[i] == x) return (int8_t)(16 + i);
      return (int8_t)-1;
    };
    for (size_t k : wt.exec) {
      const hq::DOp& o = ops[k];
      hq::WOp wo{};
      wo.kind = (int8_t)o.kind;
      wo.a = code(o.a);
      wo.b = o.b == -1 && o.kind != HQ_GATE_CNOT && o.kind != HQ_GATE_CZ && o.kind != HQ_GATE_CR
                 ? (int8_t)-1 : code(o.b);
      wo.slot = (int16_t)o.slot;
      wo.dl = (int16_t)dl[k];
      ps.wops.push_back(wo);
    }
    w.op1 = (int16_t)ps.wops.size();
    ps.hwins.push_back(w);
    if (RB <= 4) {   // the device copy (generic kernels) holds 4 register bits
      hq::WinDev d{};
      d.op0 = w.op0;
      d.op1 = w.op1;
      for (int i = 0; i < 4; ++i) d.pr[i] = w.pr[i];
      for (int i = 0; i < 10; ++i) d.ps[i] = w.ps[i];
      ps.wins.push_back(d);
    }
  }
}

template <typename T>
void put(std::vector<char>& blob, size_t& off, const T* src, size_t count, const T*& dst_dev_rel) {
  off = align_up(off, 16);
  if (blob.size() < off + count * sizeof(T)) blob.resize(off + count * sizeof(T));
  if (count) std::memcpy(blob.data() + off, src, count * sizeof(T));
  dst_dev_rel = reinterpret_cast<const T*>(off);
  off += count * sizeof(T);
}

template <typename T>
const T* rebase(const T* rel, char* base) {
  return reinterpret_cast<const T*>(base + reinterpret_cast<size_t>(rel));
}

}  // namespace

// opts: kNoFold (no folded prefixes), kOnchipOk (small circuits may use the
// shared-memory interpreter when the specialised kernels are unavailable)
// kSegment: a segment plan of the amplitude-sharded executor (in-place passes
// on a caller-owned state, no readout, no folding, specialised kernels only)
enum { kNoFold = 1, kPreferOnchip = 2, kSmallPasses = 4, kSegment = 8 };
static hq_status plan_create_impl(const hq_plan_desc* d, hq_plan* out, int opts);

extern "C" hq_status hq_plan_create(const hq_plan_desc* d, hq_plan* out) {
  return plan_create_impl(d, out, 0);
}

extern "C" hq_status hq_plan_create_segment(const hq_plan_desc* d, hq_plan* out) {
  return plan_create_impl(d, out, kSegment | kNoFold);
}

namespace {
// Owning copy of a plan description (the unfolded twin is built lazily).
struct DescCopy {
  hq_plan_desc d{};
  std::vector<hq_op> ops;
  std::vector<double> sconst, scoef, gfactor;
  std::vector<int32_t> sptr, svar, meas, pptr, pq, ps0, plen, gmode, gslot;
  explicit DescCopy(const hq_plan_desc* s) : d(*s) {
    const int nv = s->n_inputs + s->n_params;
    const int nnz = s->n_slots ? s->slot_ptr[s->n_slots] : 0;
    const int npq = s->n_preps ? s->prep_ptr[s->n_preps] : 0;
    ops.assign(s->ops, s->ops + s->n_ops);
    sconst.assign(s->slot_const, s->slot_const + s->n_slots);
    if (s->n_slots) sptr.assign(s->slot_ptr, s->slot_ptr + s->n_slots + 1);
    svar.assign(s->slot_var, s->slot_var + nnz);
    scoef.assign(s->slot_coef, s->slot_coef + nnz);
    if (s->n_measured) meas.assign(s->measured, s->measured + s->n_measured);
    if (s->n_preps) {
      pptr.assign(s->prep_ptr, s->prep_ptr + s->n_preps + 1);
      pq.assign(s->prep_qubits, s->prep_qubits + npq);
      ps0.assign(s->prep_slot0, s->prep_slot0 + s->n_preps);
      plen.assign(s->prep_len, s->prep_len + s->n_preps);
    }
    if (s->grad_mode) {
      gmode.assign(s->grad_mode, s->grad_mode + nv);
      gslot.assign(s->grad_slot, s->grad_slot + nv);
      gfactor.assign(s->grad_factor, s->grad_factor + nv);
    }
    d.ops = ops.data();
    d.slot_const = sconst.data();
    d.slot_ptr = sptr.data();
    d.slot_var = svar.data();
    d.slot_coef = scoef.data();
    d.measured = meas.empty() ? nullptr : meas.data();
    d.prep_ptr = pptr.data();
    d.prep_qubits = pq.data();
    d.prep_slot0 = ps0.data();
    d.prep_len = plen.data();
    d.grad_mode = s->grad_mode ? gmode.data() : nullptr;
    d.grad_slot = s->grad_mode ? gslot.data() : nullptr;
    d.grad_factor = s->grad_mode ? gfactor.data() : nullptr;
  }
};
bool single_qubit(int k) {
  return k == HQ_GATE_H || k == HQ_GATE_X || k == HQ_GATE_Y || k == HQ_GATE_Z || k == HQ_GATE_RX ||
         k == HQ_GATE_RY || k == HQ_GATE_RZ;
}
constexpr int kMaxFoldPerQubit = 32;
}  // namespace

static hq_status plan_create_impl(const hq_plan_desc* d, hq_plan* out, int opts) {
  const bool seg = (opts & kSegment) != 0;
  const bool allow_fold = !(opts & kNoFold) && !seg;
  if (!out) return fail(HQ_E_CONFIG, "null output");
  *out = nullptr;
  hq_status st = validate(d);
  if (st != HQ_OK) return st;
  if (seg && d->n_preps > 0) return fail(HQ_E_CONFIG, "segment plans take no state loads");
  if (seg && d->grad_mode)
    for (int v = 0; v < d->n_inputs + d->n_params; ++v)
      if (d->grad_mode[v] == HQ_GRAD_TWOPOINT) return fail(HQ_E_CONFIG, "segment plans differentiate by adjoint only");
  auto pl = new hq_plan_s();
  pl->seg = seg;
  const int n = d->n_qubits;
  const int nvars = d->n_inputs + d->n_params;
  pl->n_qubits = n;
  pl->precision = d->precision;
  pl->n_inputs = d->n_inputs;
  pl->n_params = d->n_params;
  pl->n_slots = d->n_slots;
  for (int i = 0; i < d->n_measured; ++i) pl->host_measured.push_back(d->measured[i]);
  if (pl->host_measured.empty())
    for (int qb = 0; qb < n; ++qb) pl->host_measured.push_back(qb);

  // ---- state loads must precede every gate on their qubits ----------------
  std::vector<hq_op> gates;
  uint64_t touched = 0, prep_mask = 0;
  for (int i = 0; i < d->n_ops; ++i) {
    const hq_op& op = d->ops[i];
    if (op.kind == HQ_GATE_STATEPREP) {
      uint64_t m = 0;
      for (int k = d->prep_ptr[op.q0]; k < d->prep_ptr[op.q0 + 1]; ++k) m |= 1ull << d->prep_qubits[k];
      if ((m & touched) || (m & prep_mask)) {
        delete pl;
        return fail(HQ_E_CIRCUIT, "state load after gates on its qubits has no native lowering");
      }
      prep_mask |= m;
      continue;
    }
    touched |= op_mask(op);
    gates.push_back(op);
  }
  // ---- readout-invariant diagonal gates: a diagonal gate (Z, RZ, CZ, CR)
  // that commutes to the end of the circuit — past gates on other qubits,
  // other diagonals, and monomial gates (X, Y, CNOT, SWAP), which keep it
  // diagonal while widening its support (CNOT with a target in the support
  // adds the control; SWAP moves it) — acts before a permutation-with-phases
  // and the diagonal EXACT_PROB readout, so it changes neither E nor any other
  // derivative (|P D ψ|² is |ψ|² permuted).  It is dropped; the derivatives of
  // variables that enter only dropped gates are 0, which is also the
  // reference's two-point value (E does not depend on them).  hq_state
  // (amplitudes) runs on the unfolded twin, which keeps every gate.
  std::vector<char> dropped_slot(d->n_slots > 0 ? d->n_slots : 1, 0);
  if (allow_fold && !std::getenv("HQ_NO_DROP")) {
    auto diag = [](int k) { return k == HQ_GATE_Z || k == HQ_GATE_RZ || k == HQ_GATE_CZ || k == HQ_GATE_CR; };
    std::vector<char> drop(gates.size(), 0);
    size_t nd = 0;
    for (size_t k = 0; k < gates.size(); ++k) {
      if (!diag(gates[k].kind)) continue;
      uint64_t S = op_mask(gates[k]);
      bool ok = true;
      for (size_t j = k + 1; j < gates.size() && ok; ++j) {
        const hq_op& g = gates[j];
        const uint64_t m = op_mask(g);
        if (!(m & S) || diag(g.kind) || g.kind == HQ_GATE_X || g.kind == HQ_GATE_Y) continue;
        if (g.kind == HQ_GATE_CNOT) {
          if (S >> g.q1 & 1ull) S |= 1ull << g.q0;
        } else if (g.kind == HQ_GATE_SWAP) {
          const uint64_t a = 1ull << g.q0, b = 1ull << g.q1;
          const bool ha = S & a, hb = S & b;
          S &= ~(a | b);
          if (ha) S |= b;
          if (hb) S |= a;
        } else {
          ok = false;   // H / RX / RY on the support: not readout-invariant
        }
      }
      if (ok) { drop[k] = 1; ++nd; }
    }
    if (nd > 0 && nd < gates.size()) {
      std::vector<hq_op> kept;
      for (size_t k = 0; k < gates.size(); ++k) {
        if (!drop[k]) { kept.push_back(gates[k]); continue; }
        if (gates[k].slot >= 0) dropped_slot[gates[k].slot] = 1;
      }
      gates.swap(kept);
      pl->dropped = (int32_t)nd;
    }
  }
  pl->has_preps = d->n_preps > 0;
  std::vector<int32_t> prep_off(d->n_preps);
  for (int p = 0; p < d->n_preps; ++p) { prep_off[p] = pl->prep_total; pl->prep_total += d->prep_len[p]; }

  // ---- gradient bookkeeping -------------------------------------------------
  std::vector<int32_t> var_mode(nvars, HQ_GRAD_ZERO), var_dsl(nvars, -1), var_tp(nvars, -1), tp_var;
  std::vector<double> var_factor(nvars, 0.0);
  std::map<int, int> dsl_of_slot;
  if (d->grad_mode) {
    for (int v = 0; v < nvars; ++v) {
      var_mode[v] = d->grad_mode[v];
      if (var_mode[v] == HQ_GRAD_ADJOINT && dropped_slot[d->grad_slot[v]]) var_mode[v] = HQ_GRAD_ZERO;
      if (var_mode[v] == HQ_GRAD_ADJOINT) {
        const int s = d->grad_slot[v];
        auto it = dsl_of_slot.find(s);
        if (it == dsl_of_slot.end()) it = dsl_of_slot.emplace(s, (int)dsl_of_slot.size()).first;
        var_dsl[v] = it->second;
        var_factor[v] = d->grad_factor[v];
      } else if (var_mode[v] == HQ_GRAD_TWOPOINT) {
        var_tp[v] = (int32_t)tp_var.size();
        tp_var.push_back(v);
      }
    }
  }
  pl->n_adj = (int32_t)dsl_of_slot.size();
  pl->n_tp = (int32_t)tp_var.size();
  pl->host_var_mode = var_mode;
  std::vector<int> slot_users(d->n_slots, 0);
  for (const auto& g : gates) if (g.slot >= 0) slot_users[g.slot]++;
  for (const auto& kv : dsl_of_slot) {
    if (slot_users[kv.first] != 1) {
      delete pl;
      return fail(HQ_E_CONFIG, "adjoint slot must feed exactly one gate");
    }
  }
  auto dslot_of = [&](const hq_op& g) -> int {
    if (g.slot < 0) return -1;
    auto it = dsl_of_slot.find(g.slot);
    return it == dsl_of_slot.end() ? -1 : it->second;
  };

  // ---- execution path ---------------------------------------------------------
  // HQ_FORCE_STREAM / HQ_TILE_BITS: test hooks that push small circuits through
  // the multi-pass HBM path (parity of the pass planner against the oracle)
  const char* force = std::getenv("HQ_FORCE_STREAM");
  const char* tb_env = std::getenv("HQ_TILE_BITS");
  // Shared-memory interpreter (k_onchip) only for circuits too small for the
  // specialised streaming kernels (tile >= 2^(RB+5) amplitudes): from 9 (c64) /
  // 8 (c128) qubits the whole state is one tile of a single fused
  // forward+backward kernel, 3-7x faster than the interpreter (n = 9..13,
  // tools/onchip_vs_stream.py).  Without NVRTC the interpreter takes over.
  const int stream_min = reg_bits_for(d->precision) + 5;
  pl->onchip = !seg && n <= onchip_max_qubits(d->precision) && !(force && force[0] == '1') &&
               (n < stream_min || (opts & kPreferOnchip));
  std::vector<int32_t> pass_slots, pass_dlist, pass_local;
  if (pl->onchip) {
    pl->tile_bits = n;
    for (const auto& g : gates) {
      hq::DOp o{};
      o.kind = g.kind;
      o.a = g.q0;
      o.b = two_qubit(g.kind) ? g.q1 : -1;
      o.slot = g.slot;
      o.dslot = dslot_of(g);
      pl->dops.push_back(o);
    }
    if (hq::onchip_smem_bytes(pl) > 220 * 1024) pl->onchip = false;
  }
  if (!pl->onchip) {
    pl->dops.clear();
    pl->tile_bits = tile_bits_for(d->precision);
    if (tb_env) pl->tile_bits = std::max(3, std::min(14, std::atoi(tb_env)));
    if (n < pl->tile_bits) pl->tile_bits = n;   // whole state in one tile
    // the generic window kernels run at most 256 threads per tile
    if ((opts & kSmallPasses) && pl->tile_bits - reg_bits_for(d->precision) > 8)
      pl->tile_bits = reg_bits_for(d->precision) + 8;
    if (pl->tile_bits < 2) {
      delete pl;
      return fail(HQ_E_CONFIG, "circuit too small for the streaming path");
    }
    int f = std::min(fixed_bits_for(d->precision), pl->tile_bits - 2);
    pl->fixed_bits = f;
    // SWAP(a,b) = CNOT(a,b) CNOT(b,a) CNOT(a,b): register windows only permute along one bit
    std::vector<hq_op> g2;
    for (const auto& g : gates) {
      if (g.kind == HQ_GATE_SWAP) {
        g2.push_back(hq_op{HQ_GATE_CNOT, g.q0, g.q1, -1});
        g2.push_back(hq_op{HQ_GATE_CNOT, g.q1, g.q0, -1});
        g2.push_back(hq_op{HQ_GATE_CNOT, g.q0, g.q1, -1});
      } else {
        g2.push_back(g);
      }
    }
    gates.swap(g2);
    int RB = reg_bits_for(d->precision);
    if (const char* e = std::getenv("HQ_REG_BITS")) RB = std::max(2, std::min(4, std::atoi(e)));
    pl->reg_bits = RB;
    if (pl->tile_bits - RB < 5 || pl->tile_bits - RB > 10) {
      delete pl;
      return fail(HQ_E_CONFIG, "tile must hold 2^9..2^14 amplitudes");
    }
    // ---- trailing X / CNOT gates: a basis permutation P applied to the
    // readout instead of the state (E = Σ_j w(P j)|ψ_j|², λ = w(P·) ψ) ----
    const char* noperm = std::getenv("HQ_NO_PERM");
    if (allow_fold && !(noperm && noperm[0] == '1')) {
      size_t cut = gates.size();
      while (cut > 1 && (gates[cut - 1].kind == HQ_GATE_X || gates[cut - 1].kind == HQ_GATE_CNOT)) --cut;
      if (cut < gates.size()) {
        pl->perm_mask.assign(n, 0);
        pl->perm_const.assign(n, 0);
        for (int qb = 0; qb < n; ++qb) pl->perm_mask[qb] = 1ull << qb;
        for (size_t k = cut; k < gates.size(); ++k) {
          const hq_op& g = gates[k];
          if (g.kind == HQ_GATE_X) {
            pl->perm_const[g.q0] ^= 1;
          } else {
            pl->perm_mask[g.q1] ^= pl->perm_mask[g.q0];
            pl->perm_const[g.q1] ^= pl->perm_const[g.q0];
          }
        }
        pl->perm = true;
        pl->perm_ops = (int32_t)(gates.size() - cut);
        gates.resize(cut);
      }
    }
    // generic kernels: shared-memory tables per pass.  complex128 pass kernels
    // run at 2 CTAs/SM with 128 registers: a schedule capped at 140 ops per
    // pass is kept when it needs strictly fewer passes than the uncapped one
    // (cfg4 c128: 9 -> 8 passes, first pass 184 -> 140 ops, forward+backward
    // 426.8 -> 381.1 ms at B=1024).  With equal counts the capped schedule lost
    // (cfg5 adjoint 8.09 -> 9.00 s), and complex64 gets slower with any cap
    // (profiles/r01_c128_pass_cap.log).
    const size_t op_cap = (opts & kSmallPasses) ? 48 : kMaxPassOps;
    const bool try_cap = !(opts & kSmallPasses) && d->precision == HQ_C128;
    // register windows a schedule needs (plan_windows on each pass's ops)
    auto count_windows = [&](const std::vector<hq::Pass>& sched) {
      size_t w = 0;
      for (const auto& ps : sched) {
        int pos[kMaxQubits];
        for (int b = 0; b < n; ++b) pos[b] = ~b;
        for (int i = 0; i < (int)ps.local.size(); ++i) pos[ps.local[i]] = i;
        std::vector<hq::DOp> pops;
        for (int k : ps.op_ids) {
          const hq_op& g = gates[k];
          hq::DOp o{};
          o.kind = g.kind;
          o.a = pos[g.q0];
          o.b = two_qubit(g.kind) ? pos[g.q1] : -1;
          o.slot = -1;
          o.dslot = -1;
          pops.push_back(o);
        }
        hq::Pass tmp = ps;
        plan_windows(tmp, pops, pl->tile_bits, RB, f, false);
        w += tmp.hwins.size();
      }
      return w;
    };
    // Schedule search: the first pass's op cap (and, for complex128, the
    // 140-op cap of every pass) is chosen by a cost model over register
    // windows and passes — each window transition and each HBM sweep costs
    // about the same in the complex128 kernels (cfg4, B=1024: ~2.4 ms each),
    // while complex64 passes are ~8x a window (HBM-bound sweeps): cost =
    // windows + k·passes, k = 1 (c128) / 8 (c64).  cfg4 c128: first pass
    // 140 -> 120 ops, 57 -> 53 windows, 379.6 -> 369.8 ms forward+adjoint
    // (profiles/r02_firstpass.log).  HQ_PLAN_SEARCH=0: the round-1 rule.
    const char* ps_env = std::getenv("HQ_PLAN_SEARCH");
    const bool search = !(ps_env && ps_env[0] == '0') && !(opts & kSmallPasses) && !std::getenv("HQ_FIRST_PASS_OPS");
    const size_t pass_w = d->precision == HQ_C64 ? 8 : 1;
    auto schedule = [&](uint64_t excl0) {
      auto best = schedule_passes(gates, n, pl->tile_bits, f, excl0, op_cap);
      if (try_cap) {
        auto capped = schedule_passes(gates, n, pl->tile_bits, f, excl0, kC128PassOps);
        if (capped.size() < best.size()) best.swap(capped);
      }
      const size_t first = best.empty() ? 0 : best[0].op_ids.size();
      // small plans: nothing to gain; long ones (cfg5: 59 passes) gain nothing
      // measurable from the first pass's cap and pay ~10 s of window counting
      const bool force = ps_env && ps_env[0] == '2';   // HQ_PLAN_SEARCH=2: also long plans
      if (!search || best.size() < 4 || (best.size() > 24 && !force) || first < 64) return best;
      size_t best_cost = count_windows(best) + pass_w * best.size();
      const size_t oc = (try_cap && best[0].op_ids.size() <= kC128PassOps) ? kC128PassOps : op_cap;
      for (int pct : {95, 91, 87, 83, 79, 75}) {
        auto cand = schedule_passes(gates, n, pl->tile_bits, f, excl0, oc, first * pct / 100);
        const size_t cost = count_windows(cand) + pass_w * cand.size();
        if (cost < best_cost) { best_cost = cost; best.swap(cand); }
      }
      return best;
    };
    // complex128 with dense passes: 64-byte runs (2 fixed bits).  Its pass
    // kernels are FP64-bound when a pass carries many gates, and the freer
    // tile choice needs fewer passes (cfg4: 8 -> 6, 336.9 -> 335.9 ms forward
    // + adjoint at B=1024; bench 3,019 -> 3,052 samples/s), while sparse
    // passes stay HBM-bound and want whole 128-byte lines (cfg5, ~32 gates
    // per pass: forward 1.86 s with 3 fixed bits, 2.09 s with 2;
    // profiles/r02_compiler_ab.log).  Rule: >= 4 passes of >= 48 gates each
    // on average with 3 fixed bits.  HQ_FIXED_BITS overrides.
    if (d->precision == HQ_C128 && !std::getenv("HQ_FIXED_BITS") && f == 3 && !(opts & kSmallPasses)) {
      const auto probe = schedule_passes(gates, n, pl->tile_bits, f, 0, op_cap);
      if (probe.size() >= 4 && gates.size() >= 48 * probe.size()) {
        f = 2;
        pl->fixed_bits = f;
      }
    }
    pl->passes = schedule(0);

    // ---- fold leading single-qubit gates into the initial product state ----
    // Qubits outside the first pass's tile: their whole single-qubit prefix
    // (its gradients come from λ at the first pass's start, contracted over
    // the tile: k_fold_grad).  Tile qubits: only the leading undifferentiated
    // gates (the first backward pass differentiates the rest as usual).
    const char* nofold = std::getenv("HQ_NO_FOLD");
    // differentiated prefixes of tile qubits fold too with HQ_FOLD_LOCAL=1
    const char* fl_env = std::getenv("HQ_FOLD_LOCAL");
    // (opt-in: on cfg4 the first backward pass got 2 more register windows and
    // ran slower, 3.31 -> 3.49 ms, than with those gates kept)
    const bool fold_local_grad = fl_env && fl_env[0] == '1';
    if (allow_fold && !pl->has_preps && !(nofold && nofold[0] == '1')) {
      uint64_t L0 = 0;
      for (int b : pl->passes[0].local) L0 |= 1ull << b;
      std::vector<char> open(n, 1), fold_it(gates.size(), 0);
      std::vector<int> cnt(n, 0);
      uint64_t excl = 0;
      for (size_t k = 0; k < gates.size(); ++k) {
        const hq_op& g = gates[k];
        if (!single_qubit(g.kind)) {
          for (int qb : {g.q0, g.q1})
            if (qb >= 0) open[qb] = 0;
          continue;
        }
        const int qb = g.q0;
        if (!open[qb]) continue;
        const bool local0 = L0 >> qb & 1ull;
        if (cnt[qb] >= kMaxFoldPerQubit || (local0 && dslot_of(g) >= 0 && !fold_local_grad)) {
          open[qb] = 0;
          continue;
        }
        fold_it[k] = 1;
        ++cnt[qb];
        if (dslot_of(g) >= 0) excl |= 1ull << qb;
      }
      std::vector<hq_op> kept;
      pl->fold_ptr.assign(n + 1, 0);
      for (int qb = 0; qb < n; ++qb) pl->fold_ptr[qb + 1] = pl->fold_ptr[qb] + cnt[qb];
      pl->fold_kind.assign(pl->fold_ptr[n], 0);
      pl->fold_slot.assign(pl->fold_ptr[n], -1);
      pl->fold_dslot.assign(pl->fold_ptr[n], -1);
      std::vector<int> fill(n, 0);
      for (size_t k = 0; k < gates.size(); ++k) {
        if (!fold_it[k]) { kept.push_back(gates[k]); continue; }
        const hq_op& g = gates[k];
        const int at = pl->fold_ptr[g.q0] + fill[g.q0]++;
        pl->fold_kind[at] = g.kind;
        pl->fold_slot[at] = g.slot;
        pl->fold_dslot[at] = dslot_of(g);
      }
      if (pl->fold_ptr[n] > 0 && !kept.empty()) {
        pl->fold = true;
        pl->fold_grad = excl != 0;
        pl->fold_ops = pl->fold_ptr[n];
        gates.swap(kept);
        // folded qubits with gradients: outside the first tile through λ contracted
        // over the tile (lamN), inside it through the tile-level contraction (locpart)
        pl->passes = schedule(fold_local_grad ? 0 : excl);
        for (int b : pl->passes[0].local)
          if (excl >> b & 1ull) {
            if (!fold_local_grad) {
              delete pl;
              return fail(HQ_E_CONFIG, "internal: folded qubit inside the first pass");
            }
            pl->fold_local.push_back(b);
          }
      } else {
        pl->fold_ptr.clear();
        pl->fold_kind.clear();
        pl->fold_slot.clear();
        pl->fold_dslot.clear();
      }
    }
    for (auto& ps : pl->passes) {
      int pos[kMaxQubits];
      for (int b = 0; b < n; ++b) pos[b] = ~b;
      for (int i = 0; i < (int)ps.local.size(); ++i) pos[ps.local[i]] = i;
      std::map<int, int> local_slot;
      ps.first_dop = (int32_t)pl->dops.size();
      ps.first_dlist = (int32_t)pass_dlist.size();
      std::vector<hq::DOp> pops;
      for (int k : ps.op_ids) {
        const hq_op& g = gates[k];
        hq::DOp o{};
        o.kind = g.kind;
        o.a = pos[g.q0];
        o.b = two_qubit(g.kind) ? pos[g.q1] : -1;
        o.slot = -1;
        if (g.slot >= 0) {
          auto it = local_slot.find(g.slot);
          if (it == local_slot.end()) {
            it = local_slot.emplace(g.slot, (int)ps.slots.size()).first;
            ps.slots.push_back(g.slot);
          }
          o.slot = it->second;
        }
        o.dslot = dslot_of(g);
        if (o.dslot >= 0) pass_dlist.push_back(o.dslot);
        pl->dops.push_back(o);
        pops.push_back(o);
      }
      plan_windows(ps, pops, pl->tile_bits, RB, f, true, true);
      // complex128 forward kernels: one more register bit (HQ_FWD_RB=0: off)
      {
        bool split = pl->precision == HQ_C128;
        if (const char* e = std::getenv("HQ_FWD_RB")) split = std::atoi(e) != 0;
        split = split && pl->tile_bits - (RB + 1) >= 5 && RB + 1 <= 5;
        if (split) {
          hq::Pass tmp;
          plan_windows(tmp, pops, pl->tile_bits, RB + 1, f, true, true);
          ps.f_rb = RB + 1;
          ps.fwins = std::move(tmp.hwins);
          ps.fwops = std::move(tmp.wops);
        }
      }
      ps.n_dops = (int32_t)ps.op_ids.size();
      ps.n_dslots_pass = (int32_t)pass_dlist.size() - ps.first_dlist;
      ps.first_slotlist = (int32_t)pass_slots.size();
      pass_slots.insert(pass_slots.end(), ps.slots.begin(), ps.slots.end());
      // local qubits then non-local, in increasing order
      std::vector<int32_t> row(ps.local.begin(), ps.local.end());
      for (int b = 0; b < n; ++b)
        if (pos[b] < 0) row.push_back(b);
      pass_local.insert(pass_local.end(), row.begin(), row.end());
      pl->max_pass_slots = std::max(pl->max_pass_slots, (int32_t)ps.slots.size());
      pl->max_pass_dl = std::max(pl->max_pass_dl, ps.n_dslots_pass);
    }
  }

  // gates whose dropped global phase / sign hq_state restores (folded gates are exact)
  std::vector<int32_t> rz_slots, rot_slots;
  for (const auto& g : gates) {
    if (g.kind == HQ_GATE_RZ) rz_slots.push_back(g.slot);
    if (g.kind == HQ_GATE_RX || g.kind == HQ_GATE_RY) rot_slots.push_back(g.slot);
  }

  if (pl->onchip && n <= 4 && !pl->has_preps) {
    // one-thread-per-sample specialised kernel; the interpreter stays for
    // initial states, amplitude output or without NVRTC
    std::string why;
    if (hq::jit_build(pl, why) != HQ_OK) pl->jit.small = nullptr;
  }
  if (!pl->onchip && std::getenv("HQ_PLAN_WINDOWS")) {
    if (std::getenv("HQ_PLAN_ONLY")) {   // planner experiments: print and stop before the JIT
      std::fprintf(stderr, "hq windows:");
      for (const auto& ps2 : pl->passes) std::fprintf(stderr, " %d/%zu", ps2.n_dops, ps2.wins.size());
      std::fprintf(stderr, "\n");
      delete pl;
      return fail(HQ_E_CONFIG, "plan-only");
    }
    std::fprintf(stderr, "hq windows:");
    for (const auto& ps : pl->passes) std::fprintf(stderr, " %d/%zu", ps.n_dops, ps.wins.size());
    std::fprintf(stderr, "\n");
    if (std::getenv("HQ_PLAN_WINDOWS")[0] == '2')
      for (const auto& ps : pl->passes) {
        std::fprintf(stderr, "  local:");
        for (int b : ps.local) std::fprintf(stderr, " %d", b);
        std::fprintf(stderr, "  ops:");
        for (int k : ps.op_ids) {
          const hq_op& g = gates[k];
          std::fprintf(stderr, " %d(%d%s%d)", k, g.kind, two_qubit(g.kind) ? "," : "", two_qubit(g.kind) ? g.q1 : g.q0);
        }
        std::fprintf(stderr, "\n");
      }
  }
  if (!pl->onchip) {
    std::string why;
    const hq_status js = hq::jit_build(pl, why);
    if (js != HQ_OK && seg) {
      delete pl;
      return fail(js, "segment plans need the specialised kernels: " + why);
    }
    if (js != HQ_OK && pl->reg_bits != reg_bits_for(d->precision)) {
      delete pl;
      return fail(HQ_E_CONFIG, "HQ_REG_BITS needs the specialised kernels: " + why);
    }
    if (js != HQ_OK && !(opts & kPreferOnchip) && (pl->fold || pl->perm || n <= onchip_max_qubits(d->precision))) {
      // folding needs the specialised kernels; small circuits fall back to the interpreter
      delete pl;
      if (std::getenv("HQ_JIT_COMPILE_ONLY")) return fail(HQ_E_CONFIG, why);
      return plan_create_impl(d, out, opts | kNoFold | kPreferOnchip);
    }
    if (js != HQ_OK && !(opts & kSmallPasses)) {
      // the generic window kernels keep per-pass tables in shared memory
      size_t need = 0;
      for (int i = 0; i < (int)pl->passes.size(); ++i)
        need = std::max(need, std::max(hq::stream_smem_bytes(pl, i, false), hq::stream_smem_bytes(pl, i, true)));
      if (need > 220 * 1024 || pl->tile_bits - pl->reg_bits > 8) {
        delete pl;
        return plan_create_impl(d, out, opts | kSmallPasses | kNoFold);
      }
    }
    if (js != HQ_OK) {
      pl->jit.ok = false;
      pl->jit.why = why;
      if (!(std::getenv("HQ_JIT") && std::getenv("HQ_JIT")[0] == '0'))
        std::fprintf(stderr, "hq: pass specialisation unavailable (%s); using the generic window kernels\n",
                     why.c_str());
    }
  }

  std::ostringstream os;
  os << (seg ? "segment " : "") << "n=" << n << " " << (d->precision == HQ_C64 ? "c64" : "c128") << " gates=" << gates.size()
     << " slots=" << d->n_slots << " preps=" << d->n_preps << " adjoint_slots=" << pl->n_adj
     << " twopoint_vars=" << pl->n_tp;
  if (pl->onchip) {
    os << " path=onchip smem=" << hq::onchip_smem_bytes(pl) << (pl->jit.small ? " kernel=small-jit" : "");
  } else {
    os << " path=stream kernels=" << (pl->jit.ok ? "jit" : "generic") << " tile_bits=" << pl->tile_bits
       << " reg_bits=" << pl->reg_bits << " folded=" << pl->fold_ops << (pl->fold_grad ? "(grad)" : "")
       << " dropped_diag=" << pl->dropped
       << " readout_perm=" << pl->perm_ops
       << " passes=" << pl->passes.size() << " [";
    for (size_t i = 0; i < pl->passes.size(); ++i)
      os << (i ? "," : "") << pl->passes[i].n_dops << "/" << pl->passes[i].wins.size() << "w";
    os << "]";
    if (std::getenv("HQ_PLAN_VERBOSE")) {
      auto bit = [](uint16_t m) { return 31 - __builtin_clz((unsigned)m); };
      for (size_t i = 0; i < pl->passes.size(); ++i) {
        os << "\n pass " << i << " local=";
        for (int b : pl->passes[i].local) os << b << ",";
        for (const auto& w : pl->passes[i].wins) {
          os << "\n   win ops=" << (w.op1 - w.op0) << " R=";
          for (int k = 0; k < pl->reg_bits; ++k) os << bit(w.pr[k]) << ",";
          os << " S=";
          for (int k = 0; k < pl->tile_bits - pl->reg_bits; ++k) os << bit(w.ps[k]) << ",";
        }
      }
    }
  }
  pl->description = os.str();
  if (std::getenv("HQ_PLAN_VERBOSE")) std::fprintf(stderr, "%s\n", pl->description.c_str());

  // ---- upload -------------------------------------------------------------
  std::vector<char> blob;
  size_t off = 0;
  hq::DevPlan dv{};
  const hq::DOp* r_ops;
  const int32_t *r_sptr, *r_svar, *r_meas, *r_pptr, *r_pq, *r_ps0, *r_plen, *r_tp, *r_vm, *r_vd, *r_vt;
  const int32_t *r_pslots, *r_pdl, *r_ploc, *r_poff;
  const double *r_sconst, *r_scoef, *r_vf;
  std::vector<int32_t> sptr(d->slot_ptr, d->slot_ptr + (d->n_slots ? d->n_slots + 1 : 0));
  const int nnz = d->n_slots ? d->slot_ptr[d->n_slots] : 0;
  std::vector<int32_t> meas(d->measured, d->measured + d->n_measured);
  if (meas.empty())
    for (int qb = 0; qb < n; ++qb) meas.push_back(qb);
  put(blob, off, pl->dops.data(), pl->dops.size(), r_ops);
  put(blob, off, d->slot_const, (size_t)d->n_slots, r_sconst);
  put(blob, off, sptr.data(), sptr.size(), r_sptr);
  put(blob, off, d->slot_var, (size_t)nnz, r_svar);
  put(blob, off, d->slot_coef, (size_t)nnz, r_scoef);
  put(blob, off, meas.data(), meas.size(), r_meas);
  std::vector<int32_t> pptr(d->prep_ptr, d->prep_ptr + (d->n_preps ? d->n_preps + 1 : 0));
  const int npq = d->n_preps ? d->prep_ptr[d->n_preps] : 0;
  put(blob, off, pptr.data(), pptr.size(), r_pptr);
  put(blob, off, d->prep_qubits, (size_t)npq, r_pq);
  put(blob, off, d->prep_slot0, (size_t)d->n_preps, r_ps0);
  put(blob, off, d->prep_len, (size_t)d->n_preps, r_plen);
  put(blob, off, prep_off.data(), prep_off.size(), r_poff);
  put(blob, off, tp_var.data(), tp_var.size(), r_tp);
  put(blob, off, var_mode.data(), var_mode.size(), r_vm);
  put(blob, off, var_dsl.data(), var_dsl.size(), r_vd);
  put(blob, off, var_tp.data(), var_tp.size(), r_vt);
  put(blob, off, var_factor.data(), var_factor.size(), r_vf);
  put(blob, off, pass_slots.data(), pass_slots.size(), r_pslots);
  put(blob, off, pass_dlist.data(), pass_dlist.size(), r_pdl);
  put(blob, off, pass_local.data(), pass_local.size(), r_ploc);
  std::vector<hq::WinDev> all_wins;
  std::vector<hq::WOp> all_wops;
  for (auto& ps : pl->passes) {
    ps.first_win = (int32_t)all_wins.size();
    ps.first_wop = (int32_t)all_wops.size();
    all_wins.insert(all_wins.end(), ps.wins.begin(), ps.wins.end());
    all_wops.insert(all_wops.end(), ps.wops.begin(), ps.wops.end());
  }
  const hq::WinDev* r_wins;
  const hq::WOp* r_wops;
  put(blob, off, all_wins.data(), all_wins.size(), r_wins);
  put(blob, off, all_wops.data(), all_wops.size(), r_wops);
  const hq_op* r_tape;
  put(blob, off, d->ops, (size_t)d->n_ops, r_tape);
  const int32_t *r_rz, *r_rot, *r_fptr, *r_fkind, *r_fslot, *r_fdsl, *r_fnl;
  put(blob, off, rz_slots.data(), rz_slots.size(), r_rz);
  put(blob, off, rot_slots.data(), rot_slots.size(), r_rot);
  std::vector<int32_t> fold_nl;
  if (pl->fold)
    for (int b = 0; b < n; ++b)
      if (std::find(pl->passes[0].local.begin(), pl->passes[0].local.end(), b) == pl->passes[0].local.end())
        fold_nl.push_back(b);
  put(blob, off, pl->fold_ptr.data(), pl->fold_ptr.size(), r_fptr);
  put(blob, off, pl->fold_kind.data(), pl->fold_kind.size(), r_fkind);
  put(blob, off, pl->fold_slot.data(), pl->fold_slot.size(), r_fslot);
  put(blob, off, pl->fold_dslot.data(), pl->fold_dslot.size(), r_fdsl);
  put(blob, off, fold_nl.data(), fold_nl.size(), r_fnl);
  const int32_t* r_floc;
  put(blob, off, pl->fold_local.data(), pl->fold_local.size(), r_floc);
  const uint64_t* r_pmask;
  const int32_t* r_pconst;
  put(blob, off, pl->perm_mask.data(), pl->perm_mask.size(), r_pmask);
  put(blob, off, pl->perm_const.data(), pl->perm_const.size(), r_pconst);
  blob.resize(align_up(std::max<size_t>(blob.size(), 16)));
  cudaError_t ce = cudaMalloc(&pl->dmem, blob.size());
  if (ce != cudaSuccess) {
    delete pl;
    return fail(ce == cudaErrorMemoryAllocation ? HQ_E_OOM : HQ_E_CUDA,
                std::string("plan upload: ") + cudaGetErrorString(ce));
  }
  ce = cudaMemcpy(pl->dmem, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    cudaFree(pl->dmem);
    delete pl;
    return fail(HQ_E_CUDA, std::string("plan upload: ") + cudaGetErrorString(ce));
  }
  char* base = static_cast<char*>(pl->dmem);
  dv.n_qubits = n;
  dv.n_slots = d->n_slots;
  dv.n_inputs = d->n_inputs;
  dv.n_params = d->n_params;
  dv.n_vars = nvars;
  dv.n_measured = (int32_t)meas.size();
  dv.n_preps = d->n_preps;
  dv.n_tp = pl->n_tp;
  dv.n_adj = pl->n_adj;
  dv.shift = d->shift;
  dv.grad_scale = d->grad_scale;
  dv.slot_const = rebase(r_sconst, base);
  dv.slot_ptr = rebase(r_sptr, base);
  dv.slot_var = rebase(r_svar, base);
  dv.slot_coef = rebase(r_scoef, base);
  dv.measured = rebase(r_meas, base);
  dv.prep_ptr = rebase(r_pptr, base);
  dv.prep_qubits = rebase(r_pq, base);
  dv.prep_slot0 = rebase(r_ps0, base);
  dv.prep_len = rebase(r_plen, base);
  dv.tp_var = rebase(r_tp, base);
  dv.var_mode = rebase(r_vm, base);
  dv.var_dsl = rebase(r_vd, base);
  dv.var_tp = rebase(r_vt, base);
  dv.var_factor = rebase(r_vf, base);
  pl->d_ops = rebase(r_ops, base);
  pl->d_pass_slots = rebase(r_pslots, base);
  pl->d_pass_dlist = rebase(r_pdl, base);
  pl->d_pass_local = rebase(r_ploc, base);
  pl->d_prep_off = rebase(r_poff, base);
  pl->d_wins = rebase(r_wins, base);
  dv.n_rz = (int32_t)rz_slots.size();
  dv.rz_slots = rebase(r_rz, base);
  dv.n_rot = (int32_t)rot_slots.size();
  dv.rot_slots = rebase(r_rot, base);
  dv.n_fold = pl->fold ? (int32_t)pl->fold_ops : 0;
  dv.fold_ptr = rebase(r_fptr, base);
  dv.fold_kind = rebase(r_fkind, base);
  dv.fold_slot = rebase(r_fslot, base);
  dv.fold_dslot = rebase(r_fdsl, base);
  dv.fold_nonlocal = rebase(r_fnl, base);
  dv.n_fold_nonlocal = (int32_t)fold_nl.size();
  dv.fold_local = rebase(r_floc, base);
  dv.n_fold_local = (int32_t)pl->fold_local.size();
  dv.perm = pl->perm ? 1 : 0;
  dv.perm_mask = rebase(r_pmask, base);
  dv.perm_const = rebase(r_pconst, base);
  pl->dev = dv;
  pl->d_tape = rebase(r_tape, base);
  pl->n_tape = d->n_ops;
  if (pl->fold || pl->dropped > 0) pl->desc_copy = std::make_shared<DescCopy>(d);
  pl->d_wops = rebase(r_wops, base);

  *out = pl;
  return HQ_OK;
}

extern "C" void hq_plan_destroy(hq_plan pl) {
  if (!pl) return;
  if (pl->twin) hq_plan_destroy(pl->twin);
  for (auto& r : pl->prof.recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : pl->prof.pool) cudaEventDestroy(e);
  if (pl->dmem) cudaFree(pl->dmem);
  delete pl;
}

extern "C" const char* hq_plan_describe(hq_plan pl) { return pl ? pl->description.c_str() : ""; }

extern "C" size_t hq_workspace_bytes(hq_plan pl, int64_t batch, int32_t flags) {
  if (!pl || batch < 0) return 0;
  return layout_for(pl, batch, flags).total;
}

static hq_status run(hq_plan pl, const double* x, int64_t ldx, const double* theta, int64_t batch,
                     int32_t flags, double* out, double* jac, double* state, const double* init,
                     int64_t init_rows, void* ws, size_t ws_bytes, void* stream) {
  if (!pl) return fail(HQ_E_CONFIG, "null plan");
  if (batch < 0) return fail(HQ_E_DIMENSION, "negative batch");
  if (batch == 0) return HQ_OK;
  if (pl->n_inputs > 0 && (!x || ldx < pl->n_inputs))
    return fail(HQ_E_DIMENSION, "input rows narrower than the circuit's inputs");
  if (pl->n_params > 0 && !theta) return fail(HQ_E_DIMENSION, "missing parameters");
  if (init && pl->has_preps) return fail(HQ_E_CIRCUIT, "initial state and state loads are exclusive");
  if ((init && pl->fold) || (state && pl->dropped > 0)) {
    // a caller-provided initial state replaces the folded product state, and
    // amplitudes need the dropped trailing diagonal gates: run the same tape
    // unfolded (same workspace layout for hq_state)
    hq_plan tw = nullptr;
    {
      std::lock_guard<std::mutex> lk(pl->twin_mu);
      if (!pl->twin) {
        const hq_status st = plan_create_impl(&static_cast<DescCopy*>(pl->desc_copy.get())->d, &pl->twin, kNoFold);
        if (st != HQ_OK) return st;
      }
      tw = pl->twin;
    }
    return run(tw, x, ldx, theta, batch, flags, out, jac, state, init, init_rows, ws, ws_bytes, stream);
  }
  const Layout L = layout_for(pl, batch, flags);
  if (ws_bytes < L.total || (!ws && L.total > 256)) return fail(HQ_E_CONFIG, "workspace too small");
  char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  hq::LaunchIn in;
  in.x = x;
  in.ldx = ldx;
  in.theta = theta;
  in.B = batch;
  in.V = L.V;
  in.out = out;
  in.jac = (flags & HQ_WANT_JAC) ? jac : nullptr;
  in.tp = reinterpret_cast<double*>(w + L.tp);
  in.dpart = reinterpret_cast<double*>(w + L.dpart);
  in.n_parts = L.n_parts;
  in.want_adj = (flags & HQ_WANT_JAC) ? 1 : 0;
  in.state = state;
  in.init = init;
  in.init_rows = init_rows;
  in.sws = L.sws;
  if (!pl->onchip) {
    in.sws.psi = w + L.psi;
    in.sws.lam = L.lam ? w + L.lam : nullptr;
    in.sws.rpart = reinterpret_cast<double*>(w + L.rpart);
    in.sws.lamN = L.lamN ? w + L.lamN : nullptr;
    in.sws.locpart = L.locpart ? w + L.locpart : nullptr;
  }
  cudaError_t e = hq::launch_forward(pl, in, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(HQ_E_CUDA, std::string("forward launch: ") + cudaGetErrorString(e));
  return HQ_OK;
}

extern "C" hq_status hq_forward(hq_plan pl, const double* x, int64_t ldx, const double* theta,
                                int64_t batch, int32_t flags, double* out, double* jac, void* ws,
                                size_t ws_bytes, void* stream) {
  if (!out && batch > 0) return fail(HQ_E_CONFIG, "null output");
  if ((flags & HQ_WANT_JAC) && !jac && batch > 0) return fail(HQ_E_CONFIG, "null jacobian output");
  return run(pl, x, ldx, theta, batch, flags, out, jac, nullptr, nullptr, 0, ws, ws_bytes, stream);
}

extern "C" hq_status hq_state(hq_plan pl, const double* x, int64_t ldx, const double* theta,
                              int64_t batch, const double* init, int64_t init_rows, double* state,
                              void* ws, size_t ws_bytes, void* stream) {
  if (!pl) return fail(HQ_E_CONFIG, "null plan");
  if (!state && batch > 0) return fail(HQ_E_CONFIG, "null state output");
  if (init && init_rows != 1 && init_rows != batch) return fail(HQ_E_DIMENSION, "init rows must be 1 or batch");
  // the readout still runs; route it into the workspace's scratch row
  const Layout L = layout_for(pl, batch, 0);
  if (ws_bytes < L.total) return fail(HQ_E_CONFIG, "workspace too small");
  char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  double* out = reinterpret_cast<double*>(w + L.scratch);
  return run(pl, x, ldx, theta, batch, 0, out, nullptr, state, init, init_rows, ws, ws_bytes, stream);
}

// ---- segment plans (amplitude-sharded executor) ----------------------------
static int32_t seg_chunks(const hq_plan_s* pl, int64_t B) {
  const int64_t n_tiles = 1ll << (pl->n_qubits - pl->tile_bits);
  const int64_t want = (1184 + B - 1) / B;   // >= ~8 CTAs per SM per launch
  int64_t nc = 16;
  while (nc < want) nc <<= 1;
  return (int32_t)std::min<int64_t>(nc, n_tiles);
}

extern "C" size_t hq_seg_workspace_bytes(hq_plan pl, int64_t batch) {
  if (!pl || batch <= 0) return 256;
  return align_up((size_t)batch * (size_t)std::max(pl->n_adj, 1) * (size_t)seg_chunks(pl, batch) * 8) + 512;
}

static hq_status seg_run(hq_plan pl, const double* x, int64_t ldx, const double* theta, int64_t batch, void* psi,
                         void* lam, double* jac, void* ws, size_t ws_bytes, void* stream) {
  if (!pl) return fail(HQ_E_CONFIG, "null plan");
  if (!pl->seg) return fail(HQ_E_CONFIG, "not a segment plan (hq_plan_create_segment)");
  if (batch < 0) return fail(HQ_E_DIMENSION, "negative batch");
  if (batch == 0) return HQ_OK;
  if (!psi) return fail(HQ_E_CONFIG, "null state");
  if (pl->n_inputs > 0 && (!x || ldx < pl->n_inputs))
    return fail(HQ_E_DIMENSION, "input rows narrower than the circuit's inputs");
  if (pl->n_params > 0 && !theta) return fail(HQ_E_DIMENSION, "missing parameters");
  if (ws_bytes < hq_seg_workspace_bytes(pl, batch)) return fail(HQ_E_CONFIG, "workspace too small");
  double* dpart = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  const cudaError_t e = hq::launch_segment(pl, x, ldx, theta, batch, psi, lam, dpart, seg_chunks(pl, batch), jac,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(HQ_E_CUDA, std::string("segment launch: ") + cudaGetErrorString(e));
  return HQ_OK;
}

extern "C" hq_status hq_seg_forward(hq_plan pl, const double* x, int64_t ldx, const double* theta, int64_t batch,
                                    void* psi, void* ws, size_t ws_bytes, void* stream) {
  return seg_run(pl, x, ldx, theta, batch, psi, nullptr, nullptr, ws, ws_bytes, stream);
}

extern "C" hq_status hq_seg_backward(hq_plan pl, const double* x, int64_t ldx, const double* theta, int64_t batch,
                                     void* psi, void* lam, double* jac, void* ws, size_t ws_bytes, void* stream) {
  if (!lam || !jac) return fail(HQ_E_CONFIG, "null adjoint state / jacobian output");
  return seg_run(pl, x, ldx, theta, batch, psi, lam, jac, ws, ws_bytes, stream);
}

extern "C" hq_status hq_vjp(hq_plan pl, const double* jac, const double* upstream, int64_t batch,
                            double* grad_x, double* grad_theta, void* stream) {
  if (!pl) return fail(HQ_E_CONFIG, "null plan");
  if (batch <= 0) return HQ_OK;
  if (!jac || !upstream) return fail(HQ_E_CONFIG, "null jacobian / upstream");
  cudaError_t e = hq::launch_vjp(pl, jac, upstream, batch, grad_x, grad_theta, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(HQ_E_CUDA, std::string("vjp launch: ") + cudaGetErrorString(e));
  return HQ_OK;
}

extern "C" hq_status hq_stats(hq_plan pl, int64_t batch, int32_t flags, hq_plan_stats* out) {
  if (!pl || !out) return fail(HQ_E_CONFIG, "null plan / output");
  const Layout L = layout_for(pl, batch, flags);
  hq_plan_stats s{};
  s.path = pl->onchip ? 0 : 1;
  s.n_passes = pl->onchip ? 1 : (int32_t)pl->passes.size();
  s.tile_bits = pl->tile_bits;
  s.n_adjoint_slots = pl->n_adj;
  s.n_twopoint_vars = pl->n_tp;
  s.state_bytes = (double)(pl->precision == HQ_C64 ? 8 : 16) * (double)(1ll << pl->n_qubits);
  const bool jac = (flags & HQ_WANT_JAC) != 0;
  int64_t launches = 0;
  if (batch > 0) {
    if (pl->onchip) {
      launches = 1;
    } else {
      const int64_t np = (int64_t)pl->passes.size();
      const int64_t cs = L.sws.chunk_samples;
      const int64_t real_chunks = (batch + cs - 1) / cs;
      const int64_t shifted = L.V - batch;
      const int64_t sh_chunks = (shifted + cs - 1) / cs;
      const bool adj = jac && pl->n_adj > 0;
      const bool fused = adj && pl->jit.ok && pl->jit.fused != nullptr;
      launches = real_chunks * (np + 1 + (adj ? (fused ? np - 1 : np) + (pl->fold_grad ? 1 : 0) : 0)) + sh_chunks * (np + 1);
      s.chunk_samples = cs;
    }
    if (jac && (int64_t)batch * (pl->n_inputs + pl->n_params) > 0) launches += 1;
  }
  s.launches = launches;
  *out = s;
  return HQ_OK;
}

extern "C" hq_status hq_profile_enable(hq_plan pl, int32_t enable) {
  if (!pl) return fail(HQ_E_CONFIG, "null plan");
  pl->prof.on = enable != 0;
  return HQ_OK;
}

extern "C" hq_status hq_profile_read(hq_plan pl, hq_profile_result* out) {
  if (!pl || !out) return fail(HQ_E_CONFIG, "null plan / output");
  hq_profile_result r{};
  const char* dump = std::getenv("HQ_PROFILE_DUMP");
  int idx = 0;
  for (auto& rec : pl->prof.recs) {
    cudaError_t e = cudaEventSynchronize(rec.b);
    if (e != cudaSuccess) return fail(HQ_E_CUDA, std::string("profile: ") + cudaGetErrorString(e));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, rec.a, rec.b);
    r.ms[rec.cls] += ms;
    r.launches[rec.cls] += 1;
    r.bytes[rec.cls] += rec.bytes;
    if (dump && dump[0] == '1')
      std::fprintf(stderr, "hq_prof %d cls=%d ms=%.4f bytes=%.0f GBps=%.1f\n", idx, rec.cls, ms, rec.bytes,
                   ms > 0 ? rec.bytes / (ms * 1e6) : 0.0);
    ++idx;
    pl->prof.pool.push_back(rec.a);
    pl->prof.pool.push_back(rec.b);
  }
  pl->prof.recs.clear();
  *out = r;
  return HQ_OK;
}
