// Internal structures shared by the host planner (hq_api.cpp) and the sm_100a
// kernels (hq_kernels.cu).  Nothing here crosses the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hq.h"
#include "hq_pod.h"

namespace hq {

// One op as a kernel sees it.  Qubit operands are TILE bit positions when >= 0;
// a negative value ~g (= -1-g) names a global qubit g that is not resident in
// the tile, whose bit is constant over the tile (only legal as a control or as
// the qubit of a diagonal gate — the planner guarantees it).
struct DOp {
  int32_t kind;
  int32_t a;      // target for 1q kinds; control for CNOT/CZ/CR; first qubit of SWAP
  int32_t b;      // target of CNOT/CZ/CR, second qubit of SWAP, unused otherwise
  int32_t slot;   // angle slot or -1
  int32_t dslot;  // index among the adjoint variables whose derivative this op yields, or -1
  int32_t pad[3];
};

// One op of a register window (streaming path).  Operand codes:
//   0..15 register bit, 16 + s thread-index bit s, 64 + g global qubit g
//   outside the tile (constant over the tile).
struct WOp {
  int8_t kind;
  int8_t a;        // target / control / first qubit
  int8_t b;        // second operand or -1
  int8_t pad0;
  int16_t slot;    // pass-local trig slot or -1
  int16_t dl;      // pass-local derivative index or -1
};

// A register window: which tile qubits are register bits (pr, swizzled masks)
// and thread bits (ps), and its op range in the pass's WOp list.
struct WinDev {
  int16_t op0, op1;
  uint16_t pr[4];   // swz(1 << R[i])
  uint16_t ps[10];  // swz(1 << S[s]); thread-index bit s <-> tile qubit S[s]
};

// Host-side window (the JIT generator): up to 6 register bits (forward
// kernels with one more register bit than the device struct carries).
struct WinHost {
  int16_t op0 = 0, op1 = 0;
  uint16_t pr[6] = {};
  uint16_t ps[10] = {};
};

// One HBM pass of the streaming path: tile = 2^q amplitudes gathered from the
// global qubits local[0..q).
struct Pass {
  std::vector<int32_t> local;      // tile bit i <-> global qubit local[i]
  std::vector<int32_t> op_ids;     // tape ops applied in this pass, in order
  std::vector<int32_t> slots;      // distinct angle slots those ops read
  int32_t first_dop = 0;           // offset of this pass's DOps in the device array
  int32_t n_dops = 0;
  int32_t first_slotlist = 0;      // offset into the device slot-list array
  int32_t n_dslots_pass = 0;       // ops in this pass that yield a derivative
  int32_t first_dlist = 0;         // offset into device list of dslot ids of this pass
  std::vector<WinDev> wins;        // register windows of this pass
  std::vector<WOp> wops;           // ops in window order
  int32_t first_win = 0, first_wop = 0;
  // forward-only kernels of complex128 plans: windows of f_rb (= reg_bits + 1)
  // register bits (ψ alone fits 16 amplitudes per thread; fewer windows, less
  // shared-memory traffic); 0 = the kernels share wins / wops
  int32_t f_rb = 0;
  std::vector<WinHost> fwins;
  std::vector<WOp> fwops;
  std::vector<WinHost> hwins;      // wins as the generator reads them
};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double bytes;
};

struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    cudaEvent_t e;
    if (!pool.empty()) { e = pool.back(); pool.pop_back(); return e; }
    cudaEventCreate(&e);
    return e;
  }
};

}  // namespace hq

namespace hq {
// sets hq_last_error() and returns s (for entry points outside hq_api.cpp)
hq_status fail_status(hq_status s, const std::string& msg);
// process-wide launch counters per kernel class (hq_launch_counts)
void count_launch(int cls);
// warp-shuffle register-window transitions (plan_windows / the JIT generator),
// opt-in with HQ_SHFL=1: measured slower on cfg4 (complex128 backward 286 ->
// 294 ms, complex64 124 -> 145 ms at B=1024, profiles/r02_shfl.log): the
// shuffle-friendly register sets need more windows, and transitions are only
// ~22% (c128) / ~4% (c64) of the backward passes (HQ_ABLATE=1)
inline bool shfl_enabled() {
  const char* e = std::getenv("HQ_SHFL");
  return e && e[0] == '1';
}
// Named-barrier ids of the warp-group window transitions (hq_jit.cpp
// post_store_sync; chosen for by plan_windows).  A transition that keeps the
// warp-index slots in `kept` (bit j = slot 5 + j of nwarp) synchronises each
// group of warps agreeing on those slots with barrier base + (their values).
// Every id always belongs to the SAME group of warps with the same count --
// otherwise a warp running ahead could join a barrier another group still
// uses.  Ids 1..15 are handed to kept-slot patterns, most slots kept first;
// returns the base id, or 0 when the pattern has no ids (full CTA barrier).
inline int group_barrier_base(int nwarp, uint32_t kept) {
  const uint32_t full = (1u << nwarp) - 1u;
  if (kept == 0 || kept == full || nwarp > 5) return 0;
  int next = 1;
  for (int sz = nwarp - 1; sz >= 1; --sz)
    for (uint32_t m = full; m >= 1; --m) {   // fixed order: high slots first
      if (__builtin_popcount(m) != sz) continue;
      if (next + (1 << sz) > 16) return 0;
      if (m == kept) return next;
      next += 1 << sz;
    }
  return 0;
}
// The warp slots a transition keeping `kept` synchronises on: all of them
// (warp-local) when every slot is kept, else the largest sub-pattern that owns
// barrier ids (a coarser group -- a superset of the warps that exchange data
// -- is still correct), else 0 (CTA barrier).
inline uint32_t group_barrier_mask(int nwarp, uint32_t kept) {
  const uint32_t full = (1u << nwarp) - 1u;
  if (kept == full) return full;
  uint32_t best = 0;
  for (uint32_t m = kept; m; m = (m - 1) & kept)
    if (group_barrier_base(nwarp, m) && __builtin_popcount(m) > __builtin_popcount(best)) best = m;
  return best;
}
}  // namespace hq

struct hq_plan_s {
  int32_t n_qubits = 0;
  int32_t precision = HQ_C128;
  int32_t n_inputs = 0, n_params = 0;
  bool onchip = true;
  bool seg = false;                       // segment plan (hq_plan_create_segment): in-place passes, no readout
  int32_t tile_bits = 0;                  // streaming path
  int32_t fixed_bits = 0;                 // low qubits always in the tile (contiguous HBM runs)
  int32_t reg_bits = 0;                   // amplitudes per thread = 2^reg_bits (register windows)
  int32_t n_adj = 0, n_tp = 0;
  std::vector<hq::DOp> dops;              // on-chip: the whole tape; streaming: per pass
  std::vector<hq::Pass> passes;
  std::vector<int32_t> host_var_mode;
  int32_t n_slots = 0;
  int32_t max_pass_slots = 0;
  int32_t max_pass_dl = 0;
  bool has_preps = false;
  int32_t prep_total = 0;                 // Σ prep_len
  std::string description;
  // device memory (one allocation, carved)
  void* dmem = nullptr;
  hq::DevPlan dev{};
  const hq::DOp* d_ops = nullptr;
  const int32_t* d_pass_slots = nullptr;
  const int32_t* d_pass_dlist = nullptr;
  const int32_t* d_pass_local = nullptr;  // [n_passes][n] (local then nonlocal)
  const int32_t* d_prep_off = nullptr;    // [n_preps]
  const hq_op* d_tape = nullptr;          // the plan's tape as given (NOISY trajectories)
  std::vector<int32_t> host_measured;     // readout qubits (host copy)
  int32_t n_tape = 0;
  const hq::WinDev* d_wins = nullptr;
  const hq::WOp* d_wops = nullptr;
  mutable hq::Prof prof;                  // live per-launch timing (bench / profiling)
  // leading single-qubit gates folded into the initial product state
  // (fold_ptr[q]..fold_ptr[q+1] index fold_kind/slot/dslot); fold_grad: some
  // folded gate is differentiated (gradient from λ at the first pass's start)
  bool fold = false, fold_grad = false;
  std::vector<int32_t> fold_ptr, fold_kind, fold_slot, fold_dslot;
  std::vector<int32_t> fold_local;        // first-tile qubits with differentiated folded gates
  // trailing X/CNOT gates folded into the readout: output bit q of the final
  // basis permutation = parity(index & perm_mask[q]) ^ perm_const[q]
  bool perm = false;
  std::vector<uint64_t> perm_mask;
  std::vector<int32_t> perm_const;
  int32_t perm_ops = 0;
  int32_t dropped = 0;                    // trailing diagonal gates dropped (readout-invariant)
  int64_t fold_ops = 0;
  // hq_state with a caller-provided initial state runs on an unfolded twin
  std::shared_ptr<void> desc_copy;
  hq_plan_s* twin = nullptr;
  std::mutex twin_mu;                     // plans are shared across threads; the twin is built once
  struct Jit {
    bool ok = false;
    std::string why;                      // why the static kernels run instead
    std::vector<cudaKernel_t> fwd, bwd;   // per pass
    cudaKernel_t fused = nullptr;         // last forward pass + its backward
    // launch geometry fixed when the kernels were generated (threads per CTA,
    // dynamic shared memory), per pass and mode (0 fwd, 1 bwd, 2 fused): later
    // changes of the environment knobs cannot desynchronise a launch from
    // the code's shared-memory carve-up
    std::vector<int> block[3];
    std::vector<size_t> smem[3];
    cudaKernel_t small = nullptr;         // on-chip plans up to 4 qubits: one thread per sample
  } jit;
};
