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

#include "hq_internal.h"
#include "hq_tile.cuh"

namespace hq {

struct KArgs {
  DevPlan p;
  const double* x;
  int64_t ldx;
  const double* theta;
  int64_t B;        // real rows
  int64_t V;        // real + shifted rows
  double* out;      // [B]
  double* tp;       // [B * 2 * n_tp]
  double* dpart;    // [B, n_adj, n_parts]
  int32_t n_parts;
  int32_t want_adj;
  double* state;    // optional [V?, 2^n, 2] complex128 output
  const double* init;
  int64_t init_rows;
  const int32_t* prep_off;  // [n_preps] offsets of each prep's values in sval
  int32_t prep_total;
};

__device__ __forceinline__ const double* row_of(const KArgs& a, int64_t b) {
  return a.x + b * a.ldx;
}

// Readout weight of global index idx: Σ_i 2^i·bit(idx, measured[i]) (qnn.py:108,116).
__device__ __forceinline__ double weight_of(const DevPlan& p, uint64_t idx) {
  double w = 0.0;
  for (int i = 0; i < p.n_measured; ++i)
    if ((idx >> p.measured[i]) & 1ull) w += (double)(1ull << i);
  return w;
}

// Evaluate (cos, sin) of half of every listed slot plus the prep values.
__device__ __forceinline__ void load_slots(const KArgs& a, const VSample& vs, const int32_t* slots,
                                           int n_slots, double2* trig, double* sval, bool preps,
                                           int tid, int T) {
  const double* xr = row_of(a, vs.b);
  for (int i = tid; i < n_slots; i += T) {
    const int s = slots ? slots[i] : i;
    const double v = eval_slot(a.p, s, xr, a.theta, vs.shvar, vs.shval);
    double sn, cs;
    sincos(0.5 * v, &sn, &cs);
    trig[i] = make_double2(cs, sn);
  }
  if (preps) {
    for (int pp = 0; pp < a.p.n_preps; ++pp) {
      const int s0 = a.p.prep_slot0[pp], len = a.p.prep_len[pp], off = a.prep_off[pp];
      for (int j = tid; j < len; j += T) sval[off + j] = eval_slot(a.p, s0 + j, xr, a.theta, vs.shvar, vs.shval);
    }
  }
}

// Per-prep 1/‖v‖ (serial per prep: fixed summation order).
__device__ __forceinline__ void prep_norms(const KArgs& a, const double* sval, double* inv, int tid) {
  if (tid < a.p.n_preps) {
    const int len = a.p.prep_len[tid], off = a.prep_off[tid];
    double s = 0.0;
    for (int j = 0; j < len; ++j) s += sval[off + j] * sval[off + j];
    inv[tid] = 1.0 / sqrt(s);
  }
}

// Initial amplitude at global index idx: product of the prep vectors on their
// qubits (value bit i -> prep qubit i, zero padded), |0> elsewhere.
__device__ __forceinline__ double2 init_amp(const KArgs& a, const double* sval, const double* inv,
                                            uint64_t idx) {
  const DevPlan& p = a.p;
  double re = 1.0;
  uint64_t rest = idx;
  for (int pp = 0; pp < p.n_preps; ++pp) {
    uint32_t j = 0;
    const int q0 = p.prep_ptr[pp], q1 = p.prep_ptr[pp + 1];
    for (int k = q0; k < q1; ++k) {
      const int qb = p.prep_qubits[k];
      j |= (uint32_t)((idx >> qb) & 1ull) << (k - q0);
      rest &= ~(1ull << qb);
    }
    re *= (j < (uint32_t)p.prep_len[pp]) ? sval[a.prep_off[pp] + j] * inv[pp] : 0.0;
  }
  return make_double2(rest == 0 ? re : 0.0, 0.0);
}

template <typename R>
__device__ __forceinline__ double block_sum(double v, double* red, int tid, int T) {
  v = warp_sum<R>(v);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (tid == 0)
    for (int w = 0; w < (T >> 5); ++w) s += red[w];
  return s;  // valid on thread 0
}

// ---------------------------------------------------------------------------
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
// Streaming passes.  Grid = nv * n_chunks CTAs; CTA (v, chunk) owns tiles
// [chunk*tpc, (chunk+1)*tpc) of sample v0+v.
struct PassArgs {
  PassDev ps;
  int64_t v0;          // first virtual sample of this launch
  int64_t nv;
  int32_t n_chunks;
  int32_t tpc;         // tiles per CTA
  void* psi;           // [nv, 2^n] (sample v at offset (v - v0) * 2^n)
  void* lam;
  double* rpart;       // [nv, n_chunks] readout partials (last pass)
};

__device__ __forceinline__ uint64_t tile_base(const PassDev& ps, int n, uint64_t tile) {
  uint64_t base = 0;
  for (int i = 0; i < n - ps.q; ++i) base |= ((tile >> i) & 1ull) << ps.nonlocal[i];
  return base;
}

// global offset of tile element j: two 6-bit lookup tables
__device__ __forceinline__ uint64_t tile_off(const uint64_t* lut, uint32_t j) {
  return lut[j & 63u] | lut[64 + ((j >> 6) & 63u)] | lut[128 + (j >> 12)];
}

__device__ __forceinline__ void build_lut(const PassDev& ps, uint64_t* lut, int tid, int T) {
  for (int i = tid; i < 192; i += T) {
    const int chunk = i >> 6;
    const uint32_t bits = (uint32_t)(i & 63);
    uint64_t off = 0;
    for (int k = 0; k < 6; ++k) {
      const int tb = chunk * 6 + k;
      if (tb < ps.q && ((bits >> k) & 1u)) off |= 1ull << ps.local[tb];
    }
    lut[i] = off;
  }
}

template <typename R>
__global__ void __launch_bounds__(256) k_pass_fwd(KArgs a, PassArgs pa) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevPlan& p = a.p;
  const PassDev& ps = pa.ps;
  const int n = p.n_qubits, q = ps.q;
  const int T = blockDim.x, tid = threadIdx.x;
  const uint32_t TN = 1u << q;
  const int64_t vl = blockIdx.x / pa.n_chunks;
  const int chunk = blockIdx.x % pa.n_chunks;
  const int64_t v = pa.v0 + vl;
  const VSample vs = decode_vsample(p, v, a.B);

  uint64_t* lut = reinterpret_cast<uint64_t*>(smem);            // 192
  double2* trig = reinterpret_cast<double2*>(lut + 192);        // ps.n_slots
  double* sval = reinterpret_cast<double*>(trig + ps.n_slots);  // prep values (first pass)
  const int nsv = ps.first ? ((a.prep_total + 1) & ~1) : 0;
  double* red = sval + nsv;                                      // 32
  double* inv = red + 32;                                        // 32
  double* wt = inv + 32;                                         // 32: readout weight per tile bit
  C* tile = reinterpret_cast<C*>(wt + 32);

  build_lut(ps, lut, tid, T);
  load_slots(a, vs, ps.slots, ps.n_slots, trig, sval, ps.first && p.n_preps > 0, tid, T);
  if (ps.last && tid < q) {
    double w = 0.0;
    for (int i = 0; i < p.n_measured; ++i)
      if (p.measured[i] == ps.local[tid]) w = (double)(1ull << i);
    wt[tid] = w;
  }
  __syncthreads();
  if (ps.first && p.n_preps > 0) prep_norms(a, sval, inv, tid);
  __syncthreads();

  C* gpsi = reinterpret_cast<C*>(pa.psi) + (size_t)vl * ((size_t)1 << n);
  C* glam = pa.lam ? reinterpret_cast<C*>(pa.lam) + (size_t)vl * ((size_t)1 << n) : nullptr;
  double e = 0.0;
  for (int tt = 0; tt < pa.tpc; ++tt) {
    const uint64_t t = (uint64_t)chunk * pa.tpc + tt;
    const uint64_t base = tile_base(ps, n, t);
    if (ps.first) {
      if (a.init) {
        const double* src = a.init + (a.init_rows > 1 ? v : 0) * ((int64_t)1 << n) * 2;
        for (uint32_t j = tid; j < TN; j += T) {
          const uint64_t g = base | tile_off(lut, j);
          tile[j] = cmake<C, R>((R)src[2 * g], (R)src[2 * g + 1]);
        }
      } else if (p.n_preps > 0) {
        for (uint32_t j = tid; j < TN; j += T) {
          const double2 z = init_amp(a, sval, inv, base | tile_off(lut, j));
          tile[j] = cmake<C, R>((R)z.x, (R)z.y);
        }
      } else {
        for (uint32_t j = tid; j < TN; j += T)
          tile[j] = cmake<C, R>((R)((base | tile_off(lut, j)) == 0), (R)0);
      }
    } else {
      for (uint32_t j = tid; j < TN; j += T) tile[j] = gpsi[base | tile_off(lut, j)];
    }
    __syncthreads();
    for (int k = 0; k < ps.n_ops; ++k) {
      const DOp op = ps.ops[k];
      tile_apply<R, false>(tile, q, op, trig, base, tid, T);
      __syncthreads();
    }
    if (ps.last) {
      double wb = 0.0;
      for (int i = 0; i < p.n_measured; ++i)
        if ((base >> p.measured[i]) & 1ull) wb += (double)(1ull << i);
      for (uint32_t j = tid; j < TN; j += T) {
        double w = wb;
        for (int b = 0; b < q; ++b) if ((j >> b) & 1u) w += wt[b];
        const C z = tile[j];
        e += w * (double)(z.x * z.x + z.y * z.y);
        if (glam) glam[base | tile_off(lut, j)] = cmake<C, R>((R)w * z.x, (R)w * z.y);
      }
    }
    for (uint32_t j = tid; j < TN; j += T) gpsi[base | tile_off(lut, j)] = tile[j];
    if (a.state && ps.last) {
      double* dst = a.state + v * ((int64_t)1 << n) * 2;
      for (uint32_t j = tid; j < TN; j += T) {
        const uint64_t g = base | tile_off(lut, j);
        dst[2 * g] = (double)tile[j].x;
        dst[2 * g + 1] = (double)tile[j].y;
      }
    }
    __syncthreads();
  }
  if (ps.last) {
    e = block_sum<R>(e, red, tid, T);
    if (tid == 0) pa.rpart[vl * pa.n_chunks + chunk] = e;
  }
}

template <typename R>
__global__ void __launch_bounds__(256) k_pass_bwd(KArgs a, PassArgs pa) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevPlan& p = a.p;
  const PassDev& ps = pa.ps;
  const int n = p.n_qubits, q = ps.q;
  const int T = blockDim.x, tid = threadIdx.x, nw = T >> 5;
  const uint32_t TN = 1u << q;
  const int64_t vl = blockIdx.x / pa.n_chunks;
  const int chunk = blockIdx.x % pa.n_chunks;
  const int64_t v = pa.v0 + vl;
  const VSample vs = decode_vsample(p, v, a.B);

  uint64_t* lut = reinterpret_cast<uint64_t*>(smem);
  double2* trig = reinterpret_cast<double2*>(lut + 192);
  double* acc = reinterpret_cast<double*>(trig + ps.n_slots);   // [n_dl][nw]
  C* tpsi = reinterpret_cast<C*>(acc + ((ps.n_dl * nw + 1) & ~1));
  C* tlam = tpsi + TN;

  build_lut(ps, lut, tid, T);
  load_slots(a, vs, ps.slots, ps.n_slots, trig, nullptr, false, tid, T);
  for (int i = tid; i < ps.n_dl * nw; i += T) acc[i] = 0.0;
  __syncthreads();

  C* gpsi = reinterpret_cast<C*>(pa.psi) + (size_t)vl * ((size_t)1 << n);
  C* glam = reinterpret_cast<C*>(pa.lam) + (size_t)vl * ((size_t)1 << n);
  for (int tt = 0; tt < pa.tpc; ++tt) {
    const uint64_t t = (uint64_t)chunk * pa.tpc + tt;
    const uint64_t base = tile_base(ps, n, t);
    for (uint32_t j = tid; j < TN; j += T) {
      const uint64_t g = base | tile_off(lut, j);
      tpsi[j] = gpsi[g];
      tlam[j] = glam[g];
    }
    __syncthreads();
    int dl = ps.n_dl;
    for (int k = ps.n_ops - 1; k >= 0; --k) {
      const DOp op = ps.ops[k];
      const double d = tile_adjoint_step<R>(tpsi, tlam, q, op, trig, base, tid, T);
      if (op.dslot >= 0) {
        --dl;
        const double ws = warp_sum<R>(d);
        if ((tid & 31) == 0) acc[dl * nw + (tid >> 5)] += ws;
      }
      __syncthreads();
    }
    if (!ps.first) {
      for (uint32_t j = tid; j < TN; j += T) {
        const uint64_t g = base | tile_off(lut, j);
        gpsi[g] = tpsi[j];
        glam[g] = tlam[j];
      }
    }
    __syncthreads();
  }
  // fixed-order fold over warps
  for (int i = tid; i < ps.n_dl; i += T) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += acc[i * nw + w];
    a.dpart[((int64_t)v * p.n_adj + ps.dlist[i]) * a.n_parts + chunk] = s;
  }
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
#include "hq_launch.h"

namespace hq {

// Bracket one launch with events when the plan is being profiled.
struct ProfScope {
  const hq_plan_s* pl;
  cudaStream_t st;
  ProfRec r;
  ProfScope(const hq_plan_s* p, cudaStream_t s, int cls, double bytes) : pl(p), st(s) {
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

static size_t onchip_smem(const hq_plan_s* pl, bool c64) {
  const size_t amp = c64 ? 8 : 16;
  const size_t prep = ((size_t)pl->dev.n_preps ? (size_t)pl->prep_total + 1 : 0) & ~(size_t)1;
  return (size_t)pl->n_slots * 16 + prep * 8 + 64 * 8 + 2 * ((size_t)1 << pl->n_qubits) * amp;
}

static size_t pass_smem(const hq_plan_s* pl, const Pass& ps, bool c64, bool bwd, int T) {
  const size_t amp = c64 ? 8 : 16;
  size_t b = 192 * 8 + ps.slots.size() * 16;
  if (bwd) {
    b += (((size_t)ps.n_dslots_pass * (T / 32) + 1) & ~(size_t)1) * 8;
    b += 2 * ((size_t)1 << pl->tile_bits) * amp;
  } else {
    if (&ps == &pl->passes.front()) b += (((size_t)pl->prep_total + 1) & ~(size_t)1) * 8;
    b += 96 * 8 + ((size_t)1 << pl->tile_bits) * amp;
  }
  return b;
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

static PassDev pass_dev(const hq_plan_s* pl, int i) {
  const Pass& ps = pl->passes[i];
  PassDev d;
  d.q = pl->tile_bits;
  d.n_ops = ps.n_dops;
  d.ops = pl->d_ops + ps.first_dop;
  d.n_slots = (int)ps.slots.size();
  d.slots = pl->d_pass_slots + ps.first_slotlist;
  d.n_dl = ps.n_dslots_pass;
  d.dlist = pl->d_pass_dlist + ps.first_dlist;
  d.local = pl->d_pass_local + (size_t)i * pl->n_qubits;
  d.nonlocal = d.local + pl->tile_bits;
  d.first = i == 0;
  d.last = i == (int)pl->passes.size() - 1;
  return d;
}

template <typename R>
static cudaError_t run_stream(const hq_plan_s* pl, KArgs a, const StreamWs& ws, cudaStream_t st) {
  const int T = 256;
  const int n = pl->n_qubits;
  const int64_t n_tiles = 1ll << (n - pl->tile_bits);
  const int n_chunks = ws.n_chunks;
  const int tpc = (int)(n_tiles / n_chunks);
  const int np = (int)pl->passes.size();
  size_t sf = 0, sb = 0;
  for (int i = 0; i < np; ++i) {
    sf = std::max(sf, pass_smem(pl, pl->passes[i], sizeof(R) == 4, false, T));
    sb = std::max(sb, pass_smem(pl, pl->passes[i], sizeof(R) == 4, true, T));
  }
  cudaError_t e0 = cudaFuncSetAttribute(k_pass_fwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
  if (e0 == cudaSuccess)
    e0 = cudaFuncSetAttribute(k_pass_bwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  if (e0 != cudaSuccess) return e0;
  // real rows [0, B) then shifted rows [B, V): a launch never mixes them, so
  // only real-row launches run the adjoint sweep
  const int64_t ranges[2][2] = {{0, a.B}, {a.B, a.V}};
  for (int r = 0; r < 2; ++r) {
    for (int64_t v0 = ranges[r][0]; v0 < ranges[r][1]; v0 += ws.chunk_samples) {
      const int64_t nv = (ranges[r][1] - v0) < ws.chunk_samples ? (ranges[r][1] - v0) : ws.chunk_samples;
      const bool adj = r == 0 && a.want_adj && pl->n_adj > 0;
      PassArgs pa;
      pa.v0 = v0;
      pa.nv = nv;
      pa.n_chunks = n_chunks;
      pa.tpc = tpc;
      pa.psi = ws.psi;
      pa.lam = adj ? ws.lam : nullptr;
      pa.rpart = ws.rpart;
      const double vec = (double)nv * (double)sizeof(typename Cx<R>::T) * (double)(1ll << n);
      for (int i = 0; i < np; ++i) {
        pa.ps = pass_dev(pl, i);
        const size_t sm = pass_smem(pl, pl->passes[i], sizeof(R) == 4, false, T);
        const double moved = vec * ((i == 0 ? 0 : 1) + 1 + ((i == np - 1 && adj) ? 1 : 0));
        ProfScope ps(pl, st, HQ_K_PASS_FWD, moved);
        k_pass_fwd<R><<<(unsigned)(nv * n_chunks), T, sm, st>>>(a, pa);
      }
      {
        ProfScope ps(pl, st, HQ_K_OTHER, (double)nv * n_chunks * 8.0);
        k_readout_fold<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(ws.rpart, v0, nv, n_chunks, a.B,
                                                                    a.out, a.tp);
      }
      if (adj) {
        for (int i = np - 1; i >= 0; --i) {
          pa.ps = pass_dev(pl, i);
          const size_t sm = pass_smem(pl, pl->passes[i], sizeof(R) == 4, true, T);
          ProfScope ps(pl, st, HQ_K_PASS_BWD, vec * (2 + (i == 0 ? 0 : 2)));
          k_pass_bwd<R><<<(unsigned)(nv * n_chunks), T, sm, st>>>(a, pa);
        }
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
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
  cudaError_t e;
  const bool c64 = pl->precision == HQ_C64;
  if (pl->onchip) e = c64 ? run_onchip<float>(pl, a, st) : run_onchip<double>(pl, a, st);
  else e = c64 ? run_stream<float>(pl, a, in.sws, st) : run_stream<double>(pl, a, in.sws, st);
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

cudaError_t launch_vjp(const hq_plan_s* pl, const double* jac, const double* up, int64_t B,
                       double* gx, double* gt, cudaStream_t st) {
  const int d = pl->n_inputs, P = pl->n_params, nv = d + P;
  if (gx && B * d > 0) k_vjp_x<<<(unsigned)((B * d + 255) / 256), 256, 0, st>>>(jac, up, B, nv, d, gx);
  if (gt && P > 0) k_vjp_theta<<<(P + 127) / 128, 128, 0, st>>>(jac, up, B, nv, d, P, gt);
  return cudaGetLastError();
}

}  // namespace hq
