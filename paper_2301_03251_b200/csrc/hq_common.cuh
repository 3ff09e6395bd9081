// Kernel arguments and device helpers shared by the on-chip and streaming
// kernels, plus the host-side launch profiler.
#pragma once

#include <cuda_runtime.h>

#include "hq_internal.h"
#include "hq_launch.h"
#include "hq_tile.cuh"

namespace hq {

// Bracket one launch with events when the plan is being profiled.
struct ProfScope {
  const hq_plan_s* pl;
  cudaStream_t st;
  ProfRec r;
  ProfScope(const hq_plan_s* p, cudaStream_t s, int cls, double bytes) : pl(p), st(s) {
    count_launch(cls);
    if (!pl->prof.on) return;
    r.cls = cls;
    r.bytes = bytes;
    r.a = pl->prof.get();
    r.b = pl->prof.get();
    cudaEventRecord(r.a, st);
  }
  ~ProfScope() {
    if (!pl->prof.on) return;
    cudaEventRecord(r.b, st);
    pl->prof.recs.push_back(r);
  }
};


cudaError_t run_stream(const hq_plan_s* pl, const KArgs& a, const StreamWs& ws, cudaStream_t st);
cudaError_t run_segment(const hq_plan_s* pl, const KArgs& a, void* psi, void* lam, int32_t n_chunks, bool backward,
                        cudaStream_t st);

// E per virtual sample from per-chunk readout partials (fixed order)
__global__ void k_readout_fold(const double* __restrict__ rpart, int64_t v0, int64_t nv,
                               int32_t n_chunks, int64_t B, double* out, double* tp);

}  // namespace hq
