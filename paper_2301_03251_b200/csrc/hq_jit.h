// NVRTC-specialised streaming passes (see hq_jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "hq_internal.h"

namespace hq {

struct JitLayout {
  size_t lut, trig, extra, extra2, fz, fred, total;   // fz: first pass of a folding plan, [n][2] initial factors
  bool per_thread;  // bwd: per-thread derivative accumulators (group == 32)
  int group;        // bwd: derivative partials kept per group of 32/group lanes (1 = per warp)
  int slot_stride;  // bwd: floats between derivative slots' partials (padded in group mode: no bank conflicts)
  bool pp;          // ping-pong: two tile groups per CTA alternating math / transition phases
  int block;        // threads per CTA (T, or 2T in ping-pong kernels)
};

// ping-pong backward kernels (HQ_PINGPONG=1): see gen_pass
bool pingpong_for(const hq_plan_s* pl, int pass, bool bwd, bool fused);

JitLayout jit_layout(const hq_plan_s* pl, int pass, bool bwd, bool fused = false);
// compile (or fetch from the in-process / on-disk cache) the plan's pass kernels
hq_status jit_build(hq_plan_s* pl, std::string& err);
// mode 0 forward, 1 backward, 2 fused last-forward + first-backward
// one-thread-per-sample kernel of a small on-chip plan (readout + gradients)
cudaError_t jit_launch_small(const hq_plan_s* pl, const KArgs& a, cudaStream_t st);
cudaError_t jit_launch_pass(const hq_plan_s* pl, int pass, int mode, const KArgs& a, const JPass& ps,
                            unsigned grid, cudaStream_t st);

}  // namespace hq
