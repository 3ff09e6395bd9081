// NVRTC-specialised streaming passes (see hq_jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "hq_internal.h"

namespace hq {

struct JitLayout {
  size_t lut, trig, extra, total;
  bool per_thread;  // bwd: per-thread derivative accumulators (else per warp)
};

JitLayout jit_layout(const hq_plan_s* pl, int pass, bool bwd);
// compile (or fetch from the in-process / on-disk cache) the plan's pass kernels
hq_status jit_build(hq_plan_s* pl, std::string& err);
cudaError_t jit_launch_pass(const hq_plan_s* pl, int pass, bool bwd, const KArgs& a, const JPass& ps,
                            unsigned grid, cudaStream_t st);

}  // namespace hq
