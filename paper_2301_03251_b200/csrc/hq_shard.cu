// Readout of one amplitude shard (amplitude-sharded execution).
//
// The EXACT_PROB readout E = Σ_j w(j)|ψ_j|² with w(j) = Σ_i 2^i·bit(j,
// measured[i]) (qnn.py:107-116) splits over ranks: the measured qubits that
// are rank bits contribute a per-rank constant w0, the local ones a weight per
// local index bit.  hq_shard_readout forms this rank's partial sum with a
// fixed-order two-stage reduction (bit-reproducible for a given n) and, for
// the adjoint, λ = w·ψ in the same sweep over the shard.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "hq_internal.h"

namespace hq {
namespace {

constexpr int kMaxW = 64;
constexpr int kParts = 2048;
constexpr int kThreads = 256;

struct WArgs {
  int32_t k;
  int32_t pos[kMaxW];
  double wk[kMaxW];
  double w0;
};

template <typename R>
__global__ void __launch_bounds__(kThreads) k_shard_readout(const R* __restrict__ psi, R* __restrict__ lam,
                                                            uint64_t count, WArgs w, double* __restrict__ part) {
  // block b owns the contiguous index range [b·per, (b+1)·per); threads stride it
  const uint64_t per = (count + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = (uint64_t)blockIdx.x * per;
  const uint64_t hi = lo + per < count ? lo + per : count;
  double s = 0.0;
  for (uint64_t j = lo + threadIdx.x; j < hi; j += kThreads) {
    double wj = w.w0;
    for (int i = 0; i < w.k; ++i)
      if ((j >> w.pos[i]) & 1ull) wj += w.wk[i];
    const R re = psi[2 * j], im = psi[2 * j + 1];
    s += wj * ((double)re * (double)re + (double)im * (double)im);
    if (lam) {
      lam[2 * j] = (R)wj * re;
      lam[2 * j + 1] = (R)wj * im;
    }
  }
  __shared__ double red[kThreads];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(kThreads) k_fold_parts(const double* __restrict__ part, int n, double* out) {
  __shared__ double red[kThreads];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace
}  // namespace hq

extern "C" size_t hq_shard_readout_workspace_bytes(void) { return (size_t)hq::kParts * 8 + 256; }

extern "C" hq_status hq_shard_readout(const void* psi, int32_t precision, int32_t n_local, const int32_t* pos,
                                      const double* wk, int32_t k, double w0, double* e_out, void* lam, void* ws,
                                      size_t ws_bytes, void* stream) {
  if (!psi || !e_out) return hq::fail_status(HQ_E_CONFIG, "hq_shard_readout: null state / output");
  if (n_local < 1 || n_local > 40) return hq::fail_status(HQ_E_DIMENSION, "hq_shard_readout: bad shard size");
  if (k < 0 || k > hq::kMaxW || (k > 0 && (!pos || !wk)))
    return hq::fail_status(HQ_E_CONFIG, "hq_shard_readout: bad weight list");
  if (precision != HQ_C64 && precision != HQ_C128) return hq::fail_status(HQ_E_CONFIG, "hq_shard_readout: precision");
  if (!ws || ws_bytes < hq_shard_readout_workspace_bytes())
    return hq::fail_status(HQ_E_CONFIG, "hq_shard_readout: workspace too small");
  hq::WArgs w{};
  w.k = k;
  w.w0 = w0;
  for (int i = 0; i < k; ++i) {
    if (pos[i] < 0 || pos[i] >= n_local) return hq::fail_status(HQ_E_DIMENSION, "hq_shard_readout: weight bit");
    w.pos[i] = pos[i];
    w.wk[i] = wk[i];
  }
  const uint64_t count = 1ull << n_local;
  const int parts = (int)(count / hq::kThreads < (uint64_t)hq::kParts ? (count + hq::kThreads - 1) / hq::kThreads
                                                                      : (uint64_t)hq::kParts);
  double* part = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hq::count_launch(HQ_K_OTHER);
  if (precision == HQ_C128)
    hq::k_shard_readout<double><<<parts, hq::kThreads, 0, st>>>(static_cast<const double*>(psi),
                                                                static_cast<double*>(lam), count, w, part);
  else
    hq::k_shard_readout<float><<<parts, hq::kThreads, 0, st>>>(static_cast<const float*>(psi),
                                                               static_cast<float*>(lam), count, w, part);
  hq::count_launch(HQ_K_OTHER);
  hq::k_fold_parts<<<1, hq::kThreads, 0, st>>>(part, parts, e_out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HQ_OK
                          : hq::fail_status(HQ_E_CUDA, std::string("hq_shard_readout launch: ") + cudaGetErrorString(e));
}
