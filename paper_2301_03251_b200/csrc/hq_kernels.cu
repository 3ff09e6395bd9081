// sm_100a kernels of the batched circuit simulator.
//
//   k_onchip      whole state resident in shared memory (n <= 13 c64 / 12 c128):
//                 slot trig -> state init -> all gates -> readout -> (λ = wψ ->
//                 reverse sweep with fused derivative dots).  One CTA per
//                 (virtual) sample; replaces the serial loop qnn.py:131-132 and
//                 the 2·(d+P) re-simulations per sample of qnn.py:136-153.
//   k_pass_fwd /  HBM-streaming passes for larger n: each CTA gathers tiles of
//   k_pass_bwd    2^q amplitudes (the pass's local qubits, low qubits always
//                 included so 64 B segments stay contiguous), applies every op
//                 the planner assigned to the pass, and writes the tile back.
//   k_jac         per-sample jacobian rows from derivative partials / two-point
//                 pairs (fixed-order reductions).
//   k_vjp         upstream scaling + sequential batch sum (qnn.py:137-152).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "hq_common.cuh"
#include "hq_jit.h"

namespace hq {

// ---------------------------------------------------------------------------
// the op list is staged in shared memory when it fits (one dependent global
// load per gate step otherwise dominated small circuits: cfg1 48 us/step)
constexpr size_t kOnchipOpsSmem = 32 * 1024;
__host__ __device__ inline bool onchip_ops_in_smem(int n_ops) { return (size_t)n_ops * sizeof(DOp) <= kOnchipOpsSmem; }

template <typename R>
__global__ void __launch_bounds__(256) k_onchip(KArgs a, const DOp* __restrict__ ops, int n_ops) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevPlan& p = a.p;
  const int n = p.n_qubits;
  const int A = p.n_slots;
  const int T = blockDim.x, tid = threadIdx.x, nw = T >> 5;
  const uint32_t N = 1u << n;
  double2* trig = reinterpret_cast<double2*>(smem);
  double* sval = reinterpret_cast<double*>(trig + A);
  double* red = sval + ((a.prep_total + 1) & ~1);
  double* inv = red + 32;
  C* psi = reinterpret_cast<C*>(inv + 32);
  C* lam = psi + N;
  if (onchip_ops_in_smem(n_ops)) {
    DOp* sops = reinterpret_cast<DOp*>(lam + N);
    for (int k = tid; k < n_ops; k += T) sops[k] = ops[k];
    ops = sops;
    __syncthreads();
  }

  for (int64_t v = blockIdx.x; v < a.V; v += gridDim.x) {
    const VSample vs = decode_vsample(p, v, a.B);
    load_slots(a, vs, nullptr, A, trig, sval, p.n_preps > 0, tid, T);
    __syncthreads();
    if (p.n_preps > 0) prep_norms(a, sval, inv, tid);
    __syncthreads();
    if (a.init) {
      const double* src = a.init + (a.init_rows > 1 ? v : 0) * (int64_t)N * 2;
      for (uint32_t i = tid; i < N; i += T) psi[i] = cmake<C, R>((R)src[2 * i], (R)src[2 * i + 1]);
    } else if (p.n_preps > 0) {
      for (uint32_t i = tid; i < N; i += T) {
        const double2 z = init_amp(a, sval, inv, i);
        psi[i] = cmake<C, R>((R)z.x, (R)z.y);
      }
    } else {
      for (uint32_t i = tid; i < N; i += T) psi[i] = cmake<C, R>((R)(i == 0), (R)0);
    }
    __syncthreads();
    for (int k = 0; k < n_ops; ++k) {
      const DOp op = ops[k];
      tile_apply<R, false>(psi, n, op, trig, 0ull, tid, T);
      __syncthreads();
    }
    // readout E = Σ w(idx)|ψ(idx)|²
    double e = 0.0;
    for (uint32_t i = tid; i < N; i += T) {
      const C z = psi[i];
      e += weight_of(p, i) * (double)(z.x * z.x + z.y * z.y);
    }
    e = block_sum<R>(e, red, tid, T);
    if (tid == 0) {
      if (vs.u < 0) a.out[v] = e;
      else a.tp[vs.u] = e;
    }
    if (a.state) {
      double* dst = a.state + v * (int64_t)N * 2;
      for (uint32_t i = tid; i < N; i += T) { dst[2 * i] = (double)psi[i].x; dst[2 * i + 1] = (double)psi[i].y; }
    }
    if (a.want_adj && vs.u < 0 && p.n_adj > 0) {
      for (uint32_t i = tid; i < N; i += T) {
        const R w = (R)weight_of(p, i);
        lam[i] = cmake<C, R>(w * psi[i].x, w * psi[i].y);
      }
      __syncthreads();
      for (int k = n_ops - 1; k >= 0; --k) {
        const DOp op = ops[k];
        const double d = tile_adjoint_step<R>(psi, lam, n, op, trig, 0ull, tid, T);
        if (op.dslot >= 0) {
          const double ws = warp_sum<R>(d);
          if ((tid & 31) == 0)
            a.dpart[((int64_t)v * p.n_adj + op.dslot) * a.n_parts + (tid >> 5)] = ws;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  (void)nw;
}

// ---------------------------------------------------------------------------
__global__ void k_readout_fold(const double* __restrict__ rpart, int64_t v0, int64_t nv,
                               int32_t n_chunks, int64_t B, double* out, double* tp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  double s = 0.0;
  for (int c = 0; c < n_chunks; ++c) s += rpart[i * n_chunks + c];
  const int64_t v = v0 + i;
  if (v < B) out[v] = s;
  else tp[v - B] = s;
}

// jac[b, var] from derivative partials (adjoint) or E± pairs (two-point).
__global__ void k_jac(DevPlan p, int64_t B, const double* __restrict__ dpart, int32_t n_parts,
                      const double* __restrict__ tp, double* jac) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * p.n_vars) return;
  const int64_t b = i / p.n_vars;
  const int var = (int)(i - b * p.n_vars);
  const int mode = p.var_mode[var];
  double g = 0.0;
  if (mode == HQ_GRAD_ADJOINT) {
    const double* src = dpart + (b * p.n_adj + p.var_dsl[var]) * n_parts;
    double d = 0.0;
    for (int c = 0; c < n_parts; ++c) d += src[c];
    g = p.var_factor[var] * d;
  } else if (mode == HQ_GRAD_TWOPOINT) {
    const int j = p.var_tp[var];
    const double* e = tp + (b * p.n_tp + j) * 2;
    g = (e[0] - e[1]) * p.grad_scale;     // qnn.py:51 order: (e+ - e-) * scale
  }
  jac[i] = g;
}

// grad_x[b,i] = g[b]*jac[b,i]; grad_theta[j] = Σ_b g[b]*jac[b,d+j] (sample order)
__global__ void k_vjp_x(const double* __restrict__ jac, const double* __restrict__ up, int64_t B,
                        int32_t nv, int32_t d, double* gx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * d) return;
  const int64_t b = i / d;
  const int k = (int)(i - b * d);
  gx[i] = jac[b * nv + k] * up[b];
}

__global__ void k_vjp_theta(const double* __restrict__ jac, const double* __restrict__ up,
                            int64_t B, int32_t nv, int32_t d, int32_t P, double* gt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P) return;
  double s = 0.0;
  for (int64_t b = 0; b < B; ++b) s += jac[b * nv + d + j] * up[b];
  gt[j] = s;
}

}  // namespace hq

// ===========================================================================
// Host-side launchers (called from hq_api.cpp)
// ===========================================================================

namespace hq {

static size_t onchip_smem(const hq_plan_s* pl, bool c64) {
  const size_t amp = c64 ? 8 : 16;
  const size_t prep = ((size_t)pl->dev.n_preps ? (size_t)pl->prep_total + 1 : 0) & ~(size_t)1;
  const int n_ops = (int)pl->dops.size();
  return (size_t)pl->n_slots * 16 + prep * 8 + 64 * 8 + 2 * ((size_t)1 << pl->n_qubits) * amp +
         (onchip_ops_in_smem(n_ops) ? (size_t)n_ops * sizeof(DOp) : 0);
}

size_t onchip_smem_bytes(const hq_plan_s* pl) { return onchip_smem(pl, pl->precision == HQ_C64); }

static int onchip_threads(int n) {
  int t = 1 << (n - 1);
  if (t < 32) t = 32;
  if (t > 256) t = 256;
  return t;
}

int onchip_parts(const hq_plan_s* pl) { return onchip_threads(pl->n_qubits) / 32; }

template <typename R>
static cudaError_t run_onchip(const hq_plan_s* pl, const KArgs& a, cudaStream_t st) {
  if (pl->jit.small && !a.init && !a.state) {
    ProfScope ps(pl, st, HQ_K_ONCHIP, (double)a.B * (pl->n_inputs + 1) * 8.0);
    cudaError_t e = jit_launch_small(pl, a, st);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  const size_t smem = onchip_smem(pl, sizeof(R) == 4);
  const int T = onchip_threads(pl->n_qubits);
  cudaError_t e = cudaFuncSetAttribute(k_onchip<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = a.V;
  if (grid > (1ll << 30)) grid = 1ll << 30;
  if (grid == 0) return cudaSuccess;
  {
    ProfScope ps(pl, st, HQ_K_ONCHIP, (double)a.B * (pl->n_inputs + 1) * 8.0);
    k_onchip<R><<<(unsigned)grid, T, smem, st>>>(a, pl->d_ops, (int)pl->dops.size());
  }
  return cudaGetLastError();
}

cudaError_t launch_forward(const hq_plan_s* pl, const LaunchIn& in, cudaStream_t st) {
  KArgs a;
  a.p = pl->dev;
  a.x = in.x;
  a.ldx = in.ldx;
  a.theta = in.theta;
  a.B = in.B;
  a.V = in.V;
  a.out = in.out;
  a.tp = in.tp;
  a.dpart = in.dpart;
  a.n_parts = in.n_parts;
  a.want_adj = in.want_adj;
  a.state = in.state;
  a.init = in.init;
  a.init_rows = in.init_rows;
  a.prep_off = pl->d_prep_off;
  a.prep_total = pl->prep_total;
  a.lamN = static_cast<double*>(in.sws.lamN);
  a.locpart = static_cast<double*>(in.sws.locpart);
  cudaError_t e;
  const bool c64 = pl->precision == HQ_C64;
  if (pl->onchip) e = c64 ? run_onchip<float>(pl, a, st) : run_onchip<double>(pl, a, st);
  else e = run_stream(pl, a, in.sws, st);
  if (e != cudaSuccess) return e;
  if (in.jac) {
    const int64_t tot = in.B * pl->dev.n_vars;
    if (tot > 0) {
      ProfScope ps(pl, st, HQ_K_OTHER, (double)tot * 8.0);
      k_jac<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->dev, in.B, in.dpart, in.n_parts, in.tp,
                                                         in.jac);
    }
    e = cudaGetLastError();
  }
  return e;
}

cudaError_t launch_segment(const hq_plan_s* pl, const double* x, int64_t ldx, const double* theta, int64_t B,
                           void* psi, void* lam, double* dpart, int32_t n_chunks, double* jac, cudaStream_t st) {
  KArgs a{};
  a.p = pl->dev;
  a.x = x;
  a.ldx = ldx;
  a.theta = theta;
  a.B = B;
  a.V = B;
  a.dpart = dpart;
  a.n_parts = n_chunks;
  a.want_adj = lam != nullptr;
  a.prep_off = pl->d_prep_off;
  cudaError_t e = run_segment(pl, a, psi, lam, n_chunks, lam != nullptr, st);
  if (e != cudaSuccess || !lam || !jac) return e;
  const int64_t tot = B * pl->dev.n_vars;
  if (tot > 0) {
    ProfScope ps(pl, st, HQ_K_OTHER, (double)tot * 8.0);
    k_jac<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->dev, B, dpart, n_chunks, nullptr, jac);
  }
  return cudaGetLastError();
}

cudaError_t launch_vjp(const hq_plan_s* pl, const double* jac, const double* up, int64_t B,
                       double* gx, double* gt, cudaStream_t st) {
  const int d = pl->n_inputs, P = pl->n_params, nv = d + P;
  if (gx && B * d > 0) {
    count_launch(HQ_K_OTHER);
    k_vjp_x<<<(unsigned)((B * d + 255) / 256), 256, 0, st>>>(jac, up, B, nv, d, gx);
  }
  if (gt && P > 0) {
    count_launch(HQ_K_OTHER);
    k_vjp_theta<<<(P + 127) / 128, 128, 0, st>>>(jac, up, B, nv, d, P, gt);
  }
  return cudaGetLastError();
}

}  // namespace hq
