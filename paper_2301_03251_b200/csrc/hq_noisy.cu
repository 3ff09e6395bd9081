// NOISY machine type: per-shot Kraus trajectories (reference noise.py:93-153,
// qnn.py:107-111), complex128, one warp per trajectory.
//
// Trajectory (virtual sample v, shot s): |0...0>, then for every tape op the
// exact gate (qsim.py:150-176) followed by its channel sites (op order, then
// the op's targets, then the model's channels: noise.py:130-138).  Every site
// with a non-zero parameter consumes the next uniform of Philox4x64-10
// key = (seed, s) (numpy buffering: draw k = word k%4 of block k/4 with
// counter k/4 + 1); the final outcome consumes one more draw:
// searchsorted(cumsum(marginal), u, side="right") clamped (qsim.py:227-229).
// E = Σ outcome / shots with an exact integer sum (qnn.py:27-32).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "hq_common.cuh"
#include "hq_internal.h"

namespace hq {

__global__ void k_jac(DevPlan p, int64_t B, const double* __restrict__ dpart, int32_t n_parts,
                      const double* __restrict__ tp, double* jac);

struct NoisyArgs {
  KArgs a;
  const hq_op* ops;
  int32_t n_ops;
  const hq_noise_site* sites;
  int32_t n_sites;
  int64_t shots;
  uint64_t seed;
  int32_t n, m;
  int32_t measured[16];
  int32_t warps;          // trajectories per CTA
  size_t warp_bytes;      // shared bytes per trajectory
  unsigned long long* sum;     // [V]
  unsigned long long* counts;  // [B, 2^m] or null
};

__device__ __forceinline__ double philox_draw(uint64_t seed, uint64_t shot, uint64_t k) {
  uint64_t c0 = (k >> 2) + 1, c1 = 0, c2 = 0, c3 = 0, k0 = seed, k1 = shot;
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  const uint64_t w = (k & 3) == 0 ? c0 : (k & 3) == 1 ? c1 : (k & 3) == 2 ? c2 : c3;
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }


// Execution teams: one warp per trajectory with the state in shared memory
// (n ≤ 13), or one 256-thread CTA per trajectory with the state in global
// memory (larger circuits, up to the reference's 24 qubits and beyond).
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct WarpTeam {
  int tid;
  static constexpr int T = 32;
  __device__ void sync() const { __syncwarp(); }
  __device__ double sum(double v) const { return warp_sum_d(v); }
};

struct BlockTeam {
  int tid;
  double* red;  // [T / 32] shared
  static constexpr int T = 256;
  __device__ void sync() const { __syncthreads(); }
  __device__ double sum(double v) const {  // fixed order, result on every thread
    v = warp_sum_d(v);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < T / 32; ++w) s += red[w];
    __syncthreads();
    return s;
  }
};

// A cluster of kClusterCtas CTAs on one trajectory (large n, few
// trajectories): the state in global memory, barrier.cluster between gates
// (release/acquire at cluster scope covers the global-memory state), sums
// through distributed shared memory in a fixed order.
constexpr int kClusterCtas = 8;
struct ClusterTeam {
  int tid;      // cluster rank * 256 + threadIdx.x
  double* red;  // [8] shared, per CTA
  static constexpr int T = 256 * kClusterCtas;
  __device__ void sync() const { cooperative_groups::this_cluster().sync(); }
  __device__ double sum(double v) const {
    auto cl = cooperative_groups::this_cluster();
    v = warp_sum_d(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    cl.sync();
    double s = 0.0;
    for (int r = 0; r < kClusterCtas; ++r) {
      const double* rr = cl.map_shared_rank(red, r);
      for (int w = 0; w < 8; ++w) s += rr[w];
    }
    cl.sync();
    return s;
  }
};

// 2x2 gate on qubit q (qsim.py:25-45 matrices)
template <class Team>
__device__ void t_gate1(double2* psi, int n, int q, double2 m00, double2 m01, double2 m10, double2 m11,
                        const Team& tm) {
  const uint32_t half = 1u << (n - 1);
  for (uint32_t i = tm.tid; i < half; i += Team::T) {
    const uint32_t i0 = ins0(i, q), i1 = i0 | (1u << q);
    const double2 a0 = psi[i0], a1 = psi[i1];
    psi[i0] = cadd(cmul(m00, a0), cmul(m01, a1));
    psi[i1] = cadd(cmul(m10, a0), cmul(m11, a1));
  }
}

template <class Team>
__device__ void t_apply(double2* psi, int n, int kind, int q0, int q1, double ang, const Team& tm) {
  const double2 z = make_double2(0.0, 0.0), one = make_double2(1.0, 0.0);
  switch (kind) {
    case HQ_GATE_H: {
      const double h = 0.70710678118654752440;
      t_gate1(psi, n, q0, make_double2(h, 0), make_double2(h, 0), make_double2(h, 0), make_double2(-h, 0), tm);
      break;
    }
    case HQ_GATE_X: t_gate1(psi, n, q0, z, one, one, z, tm); break;
    case HQ_GATE_Y: t_gate1(psi, n, q0, z, make_double2(0, -1), make_double2(0, 1), z, tm); break;
    case HQ_GATE_Z: t_gate1(psi, n, q0, one, z, z, make_double2(-1, 0), tm); break;
    case HQ_GATE_RX: {
      const double c = cos(ang / 2.0), s = sin(ang / 2.0);
      t_gate1(psi, n, q0, make_double2(c, 0), make_double2(0, -s), make_double2(0, -s), make_double2(c, 0), tm);
      break;
    }
    case HQ_GATE_RY: {
      const double c = cos(ang / 2.0), s = sin(ang / 2.0);
      t_gate1(psi, n, q0, make_double2(c, 0), make_double2(-s, 0), make_double2(s, 0), make_double2(c, 0), tm);
      break;
    }
    case HQ_GATE_RZ: {
      double s, c;
      sincos(0.5 * ang, &s, &c);
      t_gate1(psi, n, q0, make_double2(c, -s), z, z, make_double2(c, s), tm);
      break;
    }
    default: {  // two-qubit kinds: loop over the quarter space
      const int lo = q0 < q1 ? q0 : q1, hi = q0 < q1 ? q1 : q0;
      const uint32_t quarter = 1u << (n - 2);
      const uint32_t b0 = 1u << q0, b1 = 1u << q1;
      double2 ph = make_double2(-1.0, 0.0);
      if (kind == HQ_GATE_CR) { double s, c; sincos(ang, &s, &c); ph = make_double2(c, s); }
      for (uint32_t i = tm.tid; i < quarter; i += Team::T) {
        const uint32_t base = ins0(ins0(i, lo), hi);
        if (kind == HQ_GATE_CNOT) {
          const double2 t = psi[base | b0];
          psi[base | b0] = psi[base | b0 | b1];
          psi[base | b0 | b1] = t;
        } else if (kind == HQ_GATE_SWAP) {
          const double2 t = psi[base | b0];
          psi[base | b0] = psi[base | b1];
          psi[base | b1] = t;
        } else {  // CZ / CR: phase on |11>
          psi[base | b0 | b1] = cmul(ph, psi[base | b0 | b1]);
        }
      }
      break;
    }
  }
  tm.sync();
}

// One trajectory (virtual sample v, shot) on `psi` (2^n amplitudes) with
// marginal scratch `marg` (2^m doubles).
template <class Team>
__device__ void run_trajectory(const NoisyArgs& na, double2* psi, double* marg, int64_t v, uint64_t shot,
                               const Team& tm) {
  const KArgs& a = na.a;
  const DevPlan& p = a.p;
  const VSample vs = decode_vsample(p, v, a.B);
  const double* xr = a.x + vs.b * a.ldx;
  const int n = na.n;
  const uint32_t N = 1u << n;
  for (uint32_t i = tm.tid; i < N; i += Team::T) psi[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
  tm.sync();
  uint64_t k = 0;  // draws consumed
  int sp = 0;
  for (int oi = 0; oi < na.n_ops; ++oi) {
    const hq_op op = na.ops[oi];
    const double ang = op.slot >= 0 ? eval_slot(p, op.slot, xr, a.theta, vs.shvar, vs.shval) : 0.0;
    t_apply(psi, n, op.kind, op.q0, op.q1, ang, tm);
    for (; sp < na.n_sites && na.sites[sp].op == oi; ++sp) {
      const hq_noise_site st = na.sites[sp];
      const double pr = st.param;
      if (pr == 0.0) continue;  // draws nothing (noise.py:99)
      const double u = philox_draw(na.seed, shot, k++);
      const int q = st.qubit;
      if (st.channel == HQ_CH_BIT_FLIP) {
        if (u < pr) t_apply(psi, n, HQ_GATE_X, q, -1, 0.0, tm);
      } else if (st.channel == HQ_CH_PHASE_FLIP) {
        if (u < pr) t_apply(psi, n, HQ_GATE_Z, q, -1, 0.0, tm);
      } else if (st.channel == HQ_CH_DEPOLARIZING) {
        if (u < 0.75 * pr) {
          // Python float floor division u // (0.25 p) (CPython float_floor_div)
          const double d = 0.25 * pr;
          const double mod = fmod(u, d);
          const double div = (u - mod) / d;
          double fl = floor(div);
          if (div - fl > 0.5) fl += 1.0;
          const int which = (int)fl;
          t_apply(psi, n, which == 0 ? HQ_GATE_X : which == 1 ? HQ_GATE_Y : HQ_GATE_Z, q, -1, 0.0, tm);
        }
      } else {  // amplitude damping (noise.py:112-127)
        double ex = 0.0;
        for (uint32_t i = tm.tid; i < (N >> 1); i += Team::T) {
          const double2 a1 = psi[ins0(i, q) | (1u << q)];
          ex += a1.x * a1.x + a1.y * a1.y;
        }
        const double p_jump = pr * tm.sum(ex);
        double norm;
        if (u < p_jump) {
          const double sq = sqrt(pr);
          for (uint32_t i = tm.tid; i < (N >> 1); i += Team::T) {
            const uint32_t i0 = ins0(i, q), i1 = i0 | (1u << q);
            psi[i0] = make_double2(sq * psi[i1].x, sq * psi[i1].y);
            psi[i1] = make_double2(0.0, 0.0);
          }
          norm = sqrt(p_jump);
        } else {
          const double sq = sqrt(1.0 - pr);
          for (uint32_t i = tm.tid; i < (N >> 1); i += Team::T) {
            const uint32_t i1 = ins0(i, q) | (1u << q);
            psi[i1] = make_double2(sq * psi[i1].x, sq * psi[i1].y);
          }
          norm = sqrt(1.0 - p_jump);
        }
        tm.sync();
        if (norm > 0.0) {
          for (uint32_t i = tm.tid; i < N; i += Team::T) psi[i] = make_double2(psi[i].x / norm, psi[i].y / norm);
        }
        tm.sync();
      }
    }
  }
  // marginal over the measured qubits (outcome bit t = measured[t])
  const int m = na.m;
  const uint32_t nout = 1u << m;
  if (nout <= 16) {
    // every thread: strided partials of all outcomes; then one fixed-order
    // team reduction per outcome
    double part[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) part[j] = 0.0;
    for (uint32_t i = tm.tid; i < N; i += Team::T) {
      uint32_t o = 0;
      for (int t = 0; t < m; ++t) o |= ((i >> na.measured[t]) & 1u) << t;
      const double2 z = psi[i];
      const double pz = z.x * z.x + z.y * z.y;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j == (int)o) part[j] += pz;
    }
    for (uint32_t j = 0; j < nout; ++j) {
      const double s = tm.sum(part[j]);
      if (tm.tid == 0) marg[j] = s;
    }
  } else {
    // thread owns outcomes j ≡ tid (mod T), each summed in increasing index order
    const uint32_t nrest = 1u << (n - m);
    uint32_t mmask = 0;
    for (int t = 0; t < m; ++t) mmask |= 1u << na.measured[t];
    for (uint32_t j = tm.tid; j < nout; j += Team::T) {
      uint32_t ib = 0;
      for (int t = 0; t < m; ++t) ib |= ((j >> t) & 1u) << na.measured[t];
      double s = 0.0;
      for (uint32_t r = 0; r < nrest; ++r) {
        uint32_t ir = 0, rr = r;
        for (int q = 0; q < n && rr; ++q)
          if (!(mmask >> q & 1u)) { ir |= (rr & 1u) << q; rr >>= 1; }
        const double2 z = psi[ib | ir];
        s += z.x * z.x + z.y * z.y;
      }
      marg[j] = s;
    }
  }
  tm.sync();
  if (tm.tid == 0) {
    const double u = philox_draw(na.seed, shot, k);
    double cum = 0.0;
    uint32_t idx = nout - 1;
    for (uint32_t j = 0; j < nout; ++j) {
      cum += marg[j];
      if (cum > u) { idx = j; break; }
    }
    atomicAdd(na.sum + v, (unsigned long long)idx);
    if (na.counts && v < a.B) atomicAdd(na.counts + (size_t)v * nout + idx, 1ull);
  }
}

__global__ void k_noisy(NoisyArgs na) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t traj = (int64_t)blockIdx.x * na.warps + w;
  if (traj >= na.a.V * na.shots) return;
  const int64_t v = traj / na.shots;
  const uint64_t shot = (uint64_t)(traj - v * na.shots);
  double2* psi = reinterpret_cast<double2*>(smem + (size_t)w * na.warp_bytes);
  double* marg = reinterpret_cast<double*>(psi + ((size_t)1 << na.n));
  run_trajectory(na, psi, marg, v, shot, WarpTeam{lane});
}

// one cluster per trajectory of [traj0, traj0 + gridDim.x / kClusterCtas)
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(256)
    k_noisy_cluster(NoisyArgs na, int64_t traj0, double2* states, double* margs) {
  __shared__ double red[8];
  const int64_t c = blockIdx.x / kClusterCtas;
  const int64_t traj = traj0 + c;
  if (traj >= na.a.V * na.shots) return;   // whole cluster: c is uniform in it
  const int64_t v = traj / na.shots;
  const uint64_t shot = (uint64_t)(traj - v * na.shots);
  double2* psi = states + (size_t)c * ((size_t)1 << na.n);
  double* marg = margs + (size_t)c * ((size_t)1 << na.m);
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  run_trajectory(na, psi, marg, v, shot, ClusterTeam{rank * 256 + (int)threadIdx.x, red});
}

// one CTA per trajectory of [traj0, traj0 + gridDim.x); state in global
// memory (states != nullptr) or in dynamic shared memory
__global__ void __launch_bounds__(256) k_noisy_block(NoisyArgs na, int64_t traj0, double2* states, double* margs) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[8];
  const int64_t traj = traj0 + blockIdx.x;
  if (traj >= na.a.V * na.shots) return;
  const int64_t v = traj / na.shots;
  const uint64_t shot = (uint64_t)(traj - v * na.shots);
  double2* psi;
  double* marg;
  if (states) {
    psi = states + (size_t)blockIdx.x * ((size_t)1 << na.n);
    marg = margs + (size_t)blockIdx.x * ((size_t)1 << na.m);
  } else {
    psi = reinterpret_cast<double2*>(smem);
    marg = reinterpret_cast<double*>(psi + ((size_t)1 << na.n));
  }
  run_trajectory(na, psi, marg, v, shot, BlockTeam{(int)threadIdx.x, red});
}

__global__ void k_noisy_finish(const unsigned long long* sum, int64_t V, int64_t B, int64_t shots, double* out,
                               double* tp) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const double e = (double)sum[v] / (double)shots;
  if (v < B) out[v] = e;
  else tp[v - B] = e;
}

}  // namespace hq

namespace {
size_t al(size_t x) { return (x + 255) & ~size_t(255); }
}

constexpr int kNoisySmemQubits = 13;   // above: one CTA per trajectory, state in global memory

// trajectories resident at once in the global-memory variant: ≤ 1024 CTAs
// (≈7 per SM) and ≤ 4 GiB of states
static int64_t noisy_chunk(const hq_plan_s* pl) {
  const size_t per = ((size_t)16 << pl->n_qubits) + ((size_t)8 << pl->dev.n_measured);
  const int64_t c = (int64_t)(((size_t)4 << 30) / per);
  return std::max<int64_t>(1, std::min<int64_t>(c, 1024));
}

extern "C" size_t hq_noisy_workspace_bytes(hq_plan pl, int64_t batch, int32_t flags, int32_t n_sites) {
  if (!pl || batch < 0) return 0;
  const int64_t V = batch + ((flags & HQ_WANT_JAC) ? batch * 2 * pl->n_tp : 0);
  size_t b = al((size_t)V * 8) + al((size_t)(V - batch) * 8 + 8) + al((size_t)std::max(n_sites, 1) * sizeof(hq_noise_site)) +
             256;
  if (pl->n_qubits > kNoisySmemQubits) {
    const int64_t c = noisy_chunk(pl);
    b += al((size_t)c << (pl->n_qubits + 4)) + al((size_t)c << (pl->dev.n_measured + 3));
  }
  return b;
}

extern "C" hq_status hq_noisy(hq_plan pl, const double* x, int64_t ldx, const double* theta, int64_t batch,
                              int32_t flags, const hq_noise_site* sites, int32_t n_sites, int64_t shots,
                              uint64_t seed, double* out, double* jac, uint64_t* counts, void* ws,
                              size_t ws_bytes, void* stream) {
  if (!pl) return hq::fail_status(HQ_E_CONFIG, "null plan");
  if (batch < 0) return hq::fail_status(HQ_E_DIMENSION, "negative batch");
  if (batch == 0) return HQ_OK;
  if (shots < 1) return hq::fail_status(HQ_E_CONFIG, "shots must be >= 1");
  if (pl->has_preps) return hq::fail_status(HQ_E_CIRCUIT, "noisy trajectories need gate-level state preparation");
  const int n = pl->n_qubits;
  if (n > 26) return hq::fail_status(HQ_E_CONFIG, "noisy trajectories support up to 26 qubits");
  if (pl->n_inputs > 0 && (!x || ldx < pl->n_inputs)) return hq::fail_status(HQ_E_DIMENSION, "input rows too narrow");
  if (pl->n_params > 0 && !theta) return hq::fail_status(HQ_E_DIMENSION, "missing parameters");
  const bool want_jac = (flags & HQ_WANT_JAC) != 0;
  if (want_jac && pl->n_adj > 0)
    return hq::fail_status(HQ_E_CONFIG, "noisy gradients use the two-point rule for every variable");
  if (ws_bytes < hq_noisy_workspace_bytes(pl, batch, flags, n_sites))
    return hq::fail_status(HQ_E_CONFIG, "workspace too small");
  std::vector<hq_noise_site> keep;
  for (int i = 0; i < n_sites; ++i) {
    const hq_noise_site& s = sites[i];
    if (s.op < 0 || s.op >= pl->n_tape || s.qubit < 0 || s.qubit >= n || s.channel < 0 || s.channel > 3 ||
        !(s.param >= 0.0 && s.param <= 1.0))
      return hq::fail_status(HQ_E_CONFIG, "invalid noise site");
    if (i && s.op < sites[i - 1].op) return hq::fail_status(HQ_E_CONFIG, "noise sites must be in op order");
    if (s.param > 0.0) keep.push_back(s);
  }
  const int64_t V = batch + (want_jac ? batch * 2 * pl->n_tp : 0);
  char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  auto* sum = reinterpret_cast<unsigned long long*>(w);
  double* tp = reinterpret_cast<double*>(w + al((size_t)V * 8));
  auto* dsites = reinterpret_cast<hq_noise_site*>(w + al((size_t)V * 8) + al((size_t)(V - batch) * 8 + 8));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  hq::NoisyArgs na{};
  hq::KArgs& a = na.a;
  a.p = pl->dev;
  a.x = x;
  a.ldx = ldx;
  a.theta = theta;
  a.B = batch;
  a.V = V;
  na.ops = pl->d_tape;
  na.n_ops = pl->n_tape;
  na.sites = dsites;
  na.n_sites = (int32_t)keep.size();
  na.shots = shots;
  na.seed = seed;
  na.n = n;
  na.m = pl->dev.n_measured;
  if (na.m > 16) return hq::fail_status(HQ_E_CONFIG, "too many measured qubits");
  for (int t = 0; t < na.m; ++t) na.measured[t] = pl->host_measured[t];
  cudaError_t e;
  na.sum = sum;
  na.counts = reinterpret_cast<unsigned long long*>(counts);
  if (!keep.empty()) cudaMemcpyAsync(dsites, keep.data(), keep.size() * sizeof(hq_noise_site), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(sum, 0, (size_t)V * 8, st);
  if (counts) cudaMemsetAsync(counts, 0, ((size_t)batch << na.m) * 8, st);
  const int64_t traj = V * shots;
  if (n > kNoisySmemQubits) {
    const int64_t c = noisy_chunk(pl);
    char* sbase = reinterpret_cast<char*>(dsites) + al((size_t)std::max(n_sites, 1) * sizeof(hq_noise_site));
    auto* states = reinterpret_cast<double2*>(sbase);
    auto* margs = reinterpret_cast<double*>(sbase + al((size_t)c << (n + 4)));
    if (traj * hq::kClusterCtas <= 2 * 148 * 8 && !std::getenv("HQ_NOISY_NO_CLUSTER")) {
      // few trajectories: a cluster of CTAs per trajectory spreads them over the SMs
      for (int64_t t0 = 0; t0 < traj; t0 += c)
        hq::k_noisy_cluster<<<(unsigned)(std::min<int64_t>(c, traj - t0) * hq::kClusterCtas), 256, 0, st>>>(
            na, t0, states, margs);
    } else {
      for (int64_t t0 = 0; t0 < traj; t0 += c)
        hq::k_noisy_block<<<(unsigned)std::min<int64_t>(c, traj - t0), 256, 0, st>>>(na, t0, states, margs);
    }
  } else if (const size_t tb = ((size_t)16 << n) + ((size_t)8 << na.m);
             traj <= 148 * (int64_t)std::min<size_t>(8, (size_t)(200 * 1024) / tb)) {
    // one wave of CTAs holds every trajectory: a whole CTA per trajectory
    // (8× the lanes on each state) beats a warp per trajectory
    e = cudaFuncSetAttribute(hq::k_noisy_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb);
    if (e != cudaSuccess) return hq::fail_status(HQ_E_CUDA, cudaGetErrorString(e));
    hq::k_noisy_block<<<(unsigned)traj, 256, tb, st>>>(na, 0, nullptr, nullptr);
  } else {
    na.warp_bytes = ((size_t)16 << n) + ((size_t)8 << na.m);
    // few trajectories: spread them over the SMs (fewer warps per CTA)
    const int64_t spread = std::max<int64_t>(1, (traj + 147) / 148);
    na.warps = (int32_t)std::max<int64_t>(
        1, std::min<int64_t>(std::min<int64_t>(8, spread), (int64_t)((size_t)(96 * 1024) / na.warp_bytes)));
    const size_t smem = (size_t)na.warps * na.warp_bytes;
    e = cudaFuncSetAttribute(hq::k_noisy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return hq::fail_status(HQ_E_CUDA, cudaGetErrorString(e));
    hq::k_noisy<<<(unsigned)((traj + na.warps - 1) / na.warps), 32 * na.warps, smem, st>>>(na);
  }

  hq::k_noisy_finish<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(sum, V, batch, shots, out, tp);
  if (want_jac && jac && pl->n_inputs + pl->n_params > 0) {
    const int64_t tot = batch * (pl->n_inputs + pl->n_params);
    hq::k_jac<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->dev, batch, nullptr, 1, tp, jac);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return hq::fail_status(HQ_E_CUDA, cudaGetErrorString(e));
  return HQ_OK;
}
