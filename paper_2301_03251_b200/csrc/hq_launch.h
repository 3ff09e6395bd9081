// Host-side launch interface between hq_api.cpp and hq_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include "hq_internal.h"

namespace hq {

// Carved workspace of the HBM-streaming path.
struct StreamWs {
  void* psi = nullptr;        // [chunk_samples, 2^n] amplitudes
  void* lam = nullptr;        // same, adjoint vector
  double* rpart = nullptr;    // [chunk_samples, n_chunks]
  int64_t chunk_samples = 0;  // virtual samples resident per launch
  int32_t n_chunks = 1;       // CTAs per sample per pass
  int32_t ckpt = 0;           // >0: forward passes write ψ checkpoints C_1..C_ckpt out of place
  void* lamN = nullptr;       // fold_grad: [chunk_samples, 2^(n-q)] complex128 (k_fold_grad input)
  void* locpart = nullptr;    // [chunk_samples, n_chunks, n_fold_local, 2] complex128
};

struct LaunchIn {
  const double* x = nullptr;
  int64_t ldx = 0;
  const double* theta = nullptr;
  int64_t B = 0, V = 0;
  double* out = nullptr;
  double* tp = nullptr;
  double* dpart = nullptr;
  int32_t n_parts = 1;
  int32_t want_adj = 0;
  double* jac = nullptr;
  double* state = nullptr;
  const double* init = nullptr;
  int64_t init_rows = 0;
  StreamWs sws;
};

size_t onchip_smem_bytes(const hq_plan_s* pl);
size_t stream_smem_bytes(const hq_plan_s* pl, int pass, bool bwd);   // generic window kernels
int onchip_parts(const hq_plan_s* pl);
cudaError_t launch_forward(const hq_plan_s* pl, const LaunchIn& in, cudaStream_t st);
cudaError_t launch_segment(const hq_plan_s* pl, const double* x, int64_t ldx, const double* theta, int64_t B,
                           void* psi, void* lam, double* dpart, int32_t n_chunks, double* jac, cudaStream_t st);
cudaError_t launch_vjp(const hq_plan_s* pl, const double* jac, const double* up, int64_t B,
                       double* gx, double* gt, cudaStream_t st);

}  // namespace hq
