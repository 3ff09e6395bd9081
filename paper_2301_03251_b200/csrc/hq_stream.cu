// HBM-streaming path: one kernel launch per pass and direction.
//
//   k_wfwd  tile: global -> smem (coalesced, swizzled) -> registers; register
//           windows apply the pass's gates (smem re-distribution between
//           windows); registers -> smem -> global.  The first pass builds the
//           initial state in place (|0>, state loads or a caller state); the
//           last pass folds the readout E = Σ w|ψ|² and writes λ = wψ.
//   k_wbwd  same traffic pattern over ψ and λ, walking the windows and their
//           gates in reverse: per gate the derivative dot (accumulated per
//           thread in shared memory) and the un-apply on both vectors.
//
// Byte model per sample and pass (b = bytes/amplitude, N = 2^n): fwd reads and
// writes ψ (2Nb; first pass writes only; last pass also writes λ), bwd reads
// and writes ψ and λ (4Nb; pass 0 only reads) — SURVEY.md §8(d).
#include <algorithm>

#include "hq_common.cuh"
#include "hq_window.cuh"
#include "hq_jit.h"

namespace hq {

// register bits per thread: 16 complex64 or 8 complex128 amplitudes (both 32
// registers per vector; the adjoint keeps ψ and λ resident)
template <typename R> struct RBits { static constexpr int v = sizeof(R) == 4 ? 4 : 3; };

struct WPass {
  int32_t q, tbits, n_win, n_wops, n_slots, n_dl, first, last;
  const WinDev* wins;
  const WOp* wops;
  const int32_t* slots;
  const int32_t* dlist;
  const int32_t* local;
  const int32_t* nonlocal;
};

struct SArgs {
  WPass ps;
  int64_t v0, nv;
  int32_t n_chunks, tpc;
  void* psi;
  void* lam;
  double* rpart;
};

__device__ __forceinline__ uint64_t wtile_base(const WPass& ps, int n, uint64_t tile) {
  uint64_t base = 0;
  for (int i = 0; i < n - ps.q; ++i) base |= ((tile >> i) & 1ull) << ps.nonlocal[i];
  return base;
}

__device__ __forceinline__ uint64_t wtile_off(const uint64_t* lut, uint32_t j) {
  return lut[j & 63u] | lut[64 + ((j >> 6) & 63u)] | lut[128 + ((j >> 12) & 63u)];
}

__device__ __forceinline__ void wbuild_lut(const WPass& ps, uint64_t* lut, int tid, int T) {
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

// Staging: thread tid moves tile elements j = tid + i*T (i < 2^RB).  Their
// global offsets split as off(tid) | off(i*T) (disjoint tile bits), so one
// 16-entry table (hi) plus a per-thread constant give every address; the loop
// is fully unrolled so each thread keeps 2^RB loads in flight.
template <int RB>
__device__ __forceinline__ void stage_offsets(const uint64_t* lut, int tid, int T, uint64_t* hi,
                                              uint64_t& ot) {
  ot = wtile_off(lut, (uint32_t)tid);
  if (tid < (1 << RB)) hi[tid] = wtile_off(lut, (uint32_t)(tid * T));
}

template <typename C, int RB>
__device__ __forceinline__ void stage_in(C* tile, const C* __restrict__ g, uint64_t gbase,
                                         const uint64_t* hi, int tid, int T, C (&v)[1 << RB]) {
#pragma unroll
  for (int i = 0; i < (1 << RB); ++i) v[i] = g[gbase | hi[i]];
#pragma unroll
  for (int i = 0; i < (1 << RB); ++i) tile[swz((uint32_t)(tid + i * T))] = v[i];
}

template <typename C, int RB>
__device__ __forceinline__ void stage_out(const C* tile, C* __restrict__ g, uint64_t gbase,
                                          const uint64_t* hi, int tid, int T) {
#pragma unroll
  for (int i = 0; i < (1 << RB); ++i) g[gbase | hi[i]] = tile[swz((uint32_t)(tid + i * T))];
}

__device__ __forceinline__ void copy_plan(const WPass& ps, WinDev* wins, WOp* wops, int tid, int T) {
  const uint4* ws = reinterpret_cast<const uint4*>(ps.wins);
  uint4* wd = reinterpret_cast<uint4*>(wins);
  for (int i = tid; i < ps.n_win * 2; i += T) wd[i] = ws[i];
  const uint2* os = reinterpret_cast<const uint2*>(ps.wops);
  uint2* od = reinterpret_cast<uint2*>(wops);
  for (int i = tid; i < ps.n_wops; i += T) od[i] = os[i];
}

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

struct WLayout {
  size_t tile, lut, trig, wins, wops, extra, total;
};

// shared-memory carve-up (same on host and device)
__host__ __device__ inline WLayout wlayout(int q, int amp_bytes, int n_vec, int n_slots, int n_win,
                                           int n_wops, size_t extra_bytes) {
  WLayout L;
  size_t o = 0;
  L.tile = o; o = align16(o + (size_t)n_vec * ((size_t)amp_bytes << q));
  L.lut = o; o = align16(o + (192 + 16) * 8);
  L.trig = o; o = align16(o + (size_t)n_slots * 16);
  L.wins = o; o = align16(o + (size_t)n_win * sizeof(WinDev));
  L.wops = o; o = align16(o + (size_t)n_wops * sizeof(WOp));
  L.extra = o; o = align16(o + extra_bytes);
  L.total = o;
  return L;
}

template <typename R, bool EXACT_RZ>
__global__ void __launch_bounds__(256, 2) k_wfwd(KArgs a, SArgs sa) {
  using C = typename Cx<R>::T;
  constexpr int kRB = RBits<R>::v;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevPlan& p = a.p;
  const WPass& ps = sa.ps;
  const int n = p.n_qubits, q = ps.q;
  const int T = blockDim.x, tid = threadIdx.x;
  const uint32_t TN = 1u << q;
  const int64_t vl = blockIdx.x / sa.n_chunks;
  const int chunk = blockIdx.x % sa.n_chunks;
  const int64_t v = sa.v0 + vl;
  const VSample vs = decode_vsample(p, v, a.B);
  const int nsv = ps.first ? ((a.prep_total + 1) & ~1) : 0;
  const WLayout L = wlayout(q, sizeof(C), 1, ps.n_slots, ps.n_win, ps.n_wops, (size_t)(nsv + 96) * 8);
  C* tile = reinterpret_cast<C*>(smem + L.tile);
  uint64_t* lut = reinterpret_cast<uint64_t*>(smem + L.lut);
  double2* trig = reinterpret_cast<double2*>(smem + L.trig);
  WinDev* wins = reinterpret_cast<WinDev*>(smem + L.wins);
  WOp* wops = reinterpret_cast<WOp*>(smem + L.wops);
  double* sval = reinterpret_cast<double*>(smem + L.extra);
  double* red = sval + nsv;
  double* inv = red + 32;
  double* wt = inv + 32;

  uint64_t* hi = lut + 192;
  wbuild_lut(ps, lut, tid, T);
  copy_plan(ps, wins, wops, tid, T);
  load_slots(a, vs, ps.slots, ps.n_slots, trig, sval, ps.first && p.n_preps > 0, tid, T);
  __syncthreads();
  uint64_t ot;
  stage_offsets<kRB>(lut, tid, T, hi, ot);
  if (ps.last && tid < q) {
    double w = 0.0;
    for (int i = 0; i < p.n_measured; ++i)
      if (p.measured[i] == ps.local[tid]) w = (double)(1ull << i);
    wt[tid] = w;
  }
  __syncthreads();
  if (ps.first && p.n_preps > 0) prep_norms(a, sval, inv, tid);
  __syncthreads();

  C* gpsi = reinterpret_cast<C*>(sa.psi) + (size_t)vl * ((size_t)1 << n);
  C* glam = sa.lam ? reinterpret_cast<C*>(sa.lam) + (size_t)vl * ((size_t)1 << n) : nullptr;
  double e = 0.0;
  C r[1 << kRB];
  for (int tt = 0; tt < sa.tpc; ++tt) {
    const uint64_t t = (uint64_t)chunk * sa.tpc + tt;
    const uint64_t base = wtile_base(ps, n, t);
    if (ps.first) {
      if (a.init) {
        const double* src = a.init + (a.init_rows > 1 ? v : 0) * ((int64_t)1 << n) * 2;
        for (uint32_t j = tid; j < TN; j += T) {
          const uint64_t g = base | wtile_off(lut, j);
          tile[swz(j)] = cmake<C, R>((R)src[2 * g], (R)src[2 * g + 1]);
        }
      } else if (p.n_preps > 0) {
        for (uint32_t j = tid; j < TN; j += T) {
          const double2 z = init_amp(a, sval, inv, base | wtile_off(lut, j));
          tile[swz(j)] = cmake<C, R>((R)z.x, (R)z.y);
        }
      } else {
        for (uint32_t j = tid; j < TN; j += T)
          tile[swz(j)] = cmake<C, R>((R)((base | wtile_off(lut, j)) == 0), (R)0);
      }
    } else {
      stage_in<C, kRB>(tile, gpsi, base | ot, hi, tid, T, r);
    }
    __syncthreads();
    smem_to_regs<C, kRB>(r, tile, wins[0], tid, ps.tbits);
    for (int w = 0; w < ps.n_win; ++w) {
      if (w > 0) {
        __syncthreads();
        regs_to_smem<C, kRB>(r, tile, wins[w - 1], tid, ps.tbits);
        __syncthreads();
        smem_to_regs<C, kRB>(r, tile, wins[w], tid, ps.tbits);
      }
      const int o1 = wins[w].op1;
      for (int k = wins[w].op0; k < o1; ++k)
        wop_apply<R, kRB, false, EXACT_RZ>(r, wops[k], trig, tid, base);
    }
    __syncthreads();
    regs_to_smem<C, kRB>(r, tile, wins[ps.n_win - 1], tid, ps.tbits);
    __syncthreads();
    if (ps.last) {
      double wb = 0.0;
      for (int i = 0; i < p.n_measured; ++i)
        if ((base >> p.measured[i]) & 1ull) wb += (double)(1ull << i);
      double wthr = wb;   // weight of this thread's fixed tile bits
      for (int bb = 0; bb < q - kRB; ++bb)
        if ((tid >> bb) & 1) wthr += wt[bb];
#pragma unroll
      for (int i = 0; i < (1 << kRB); ++i) {
        const uint32_t j = tid + i * T;
        double w = wthr;
        for (int bb = q - kRB; bb < q; ++bb)
          if ((j >> bb) & 1u) w += wt[bb];
        const C z = tile[swz(j)];
        const uint64_t g = base | ot | hi[i];
        e += w * (double)(z.x * z.x + z.y * z.y);
        gpsi[g] = z;
        if (glam) glam[g] = cmake<C, R>((R)w * z.x, (R)w * z.y);
        if (a.state) {
          double* dst = a.state + v * ((int64_t)1 << n) * 2;
          dst[2 * g] = (double)z.x;
          dst[2 * g + 1] = (double)z.y;
        }
      }
    } else {
      stage_out<C, kRB>(tile, gpsi, base | ot, hi, tid, T);
    }
    __syncthreads();
  }
  if (ps.last) {
    e = block_sum<R>(e, red, tid, T);
    if (tid == 0) sa.rpart[vl * sa.n_chunks + chunk] = e;
  }
}

template <typename R>
__global__ void __launch_bounds__(256, 2) k_wbwd(KArgs a, SArgs sa) {
  using C = typename Cx<R>::T;
  constexpr int kRB = RBits<R>::v;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevPlan& p = a.p;
  const WPass& ps = sa.ps;
  const int n = p.n_qubits, q = ps.q;
  const int T = blockDim.x, tid = threadIdx.x;
  const uint32_t TN = 1u << q;
  const int64_t vl = blockIdx.x / sa.n_chunks;
  const int chunk = blockIdx.x % sa.n_chunks;
  const int64_t v = sa.v0 + vl;
  const VSample vs = decode_vsample(p, v, a.B);
  const int nw = T >> 5;
  const WLayout L = wlayout(q, sizeof(C), 2, ps.n_slots, ps.n_win, ps.n_wops,
                            (size_t)ps.n_dl * nw * sizeof(double));
  C* tp = reinterpret_cast<C*>(smem + L.tile);
  C* tl = tp + TN;
  uint64_t* lut = reinterpret_cast<uint64_t*>(smem + L.lut);
  double2* trig = reinterpret_cast<double2*>(smem + L.trig);
  WinDev* wins = reinterpret_cast<WinDev*>(smem + L.wins);
  WOp* wops = reinterpret_cast<WOp*>(smem + L.wops);
  double* dacc = reinterpret_cast<double*>(smem + L.extra);   // [n_dl][warps]

  uint64_t* hi = lut + 192;
  wbuild_lut(ps, lut, tid, T);
  copy_plan(ps, wins, wops, tid, T);
  load_slots(a, vs, ps.slots, ps.n_slots, trig, nullptr, false, tid, T);
  for (int i = tid; i < ps.n_dl * nw; i += T) dacc[i] = 0.0;
  __syncthreads();
  uint64_t ot;
  stage_offsets<kRB>(lut, tid, T, hi, ot);
  __syncthreads();

  C* gpsi = reinterpret_cast<C*>(sa.psi) + (size_t)vl * ((size_t)1 << n);
  C* glam = reinterpret_cast<C*>(sa.lam) + (size_t)vl * ((size_t)1 << n);
  C rp[1 << kRB], rl[1 << kRB];
  const int last = ps.n_win - 1;
  for (int tt = 0; tt < sa.tpc; ++tt) {
    const uint64_t t = (uint64_t)chunk * sa.tpc + tt;
    const uint64_t base = wtile_base(ps, n, t);
    stage_in<C, kRB>(tp, gpsi, base | ot, hi, tid, T, rp);
    stage_in<C, kRB>(tl, glam, base | ot, hi, tid, T, rl);
    __syncthreads();
    smem_to_regs<C, kRB>(rp, tp, wins[last], tid, ps.tbits);
    smem_to_regs<C, kRB>(rl, tl, wins[last], tid, ps.tbits);
    for (int w = last; w >= 0; --w) {
      if (w < last) {
        __syncthreads();
        regs_to_smem<C, kRB>(rp, tp, wins[w + 1], tid, ps.tbits);
        regs_to_smem<C, kRB>(rl, tl, wins[w + 1], tid, ps.tbits);
        __syncthreads();
        smem_to_regs<C, kRB>(rp, tp, wins[w], tid, ps.tbits);
        smem_to_regs<C, kRB>(rl, tl, wins[w], tid, ps.tbits);
      }
      const int o0 = wins[w].op0;
      for (int k = wins[w].op1 - 1; k >= o0; --k) {
        const WOp op = wops[k];
        const R d = wop_adjoint<R, kRB, true>(rp, rl, op, trig, tid, base);
        if (op.dl >= 0) {
          const double ws = warp_sum<R>((double)d);
          if ((tid & 31) == 0) dacc[op.dl * nw + (tid >> 5)] += ws;
        }
      }
    }
    if (!ps.first) {
      __syncthreads();
      regs_to_smem<C, kRB>(rp, tp, wins[0], tid, ps.tbits);
      regs_to_smem<C, kRB>(rl, tl, wins[0], tid, ps.tbits);
      __syncthreads();
      stage_out<C, kRB>(tp, gpsi, base | ot, hi, tid, T);
      stage_out<C, kRB>(tl, glam, base | ot, hi, tid, T);
    }
    __syncthreads();
  }
  // fixed-order fold over threads
  for (int i = tid; i < ps.n_dl; i += T) {
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s += dacc[i * nw + k];
    a.dpart[((int64_t)v * p.n_adj + ps.dlist[i]) * a.n_parts + chunk] = s;
  }
}

// ---------------------------------------------------------------------------
// Gradients of folded gates (leading single-qubit gates of qubits outside the
// first pass's tile, applied analytically in the initial product state).
// With u_p the initial factor of qubit p and lamN[t] = λ at the circuit start
// contracted over the first pass's tile (written by its backward kernel), the
// reduced adjoint of folded qubit q is r_q[c] = Σ_{t: bit_q(t)=c} lamN[t]·
// conj(Π_{p≠q} u_p[bit_p(t)]); for q's j-th folded gate G_j (state after it
// a = G_j..G_1|0>, y = G_{j+1}^†..G_K^† r_q) the pairwise products are
// X[b'][b] = a_b·conj(y_b'), and the derivative dot is the passes' formula
// on X (RY: Re X10 − Re X01; RX: Im X01 + Im X10; RZ: −2 Im X11).
// One CTA per (sample, non-tile qubit); writes part 0 of each folded
// derivative slot of that qubit.
__global__ void __launch_bounds__(256) k_fold_grad(KArgs a, int64_t v0, int32_t n_chunks) {
  const DevPlan& p = a.p;
  const int tid = threadIdx.x, T = blockDim.x;
  const int nq = p.n_fold_nonlocal + p.n_fold_local;
  const int64_t vl = blockIdx.x / nq, v = v0 + vl;
  const int kq = (int)(blockIdx.x - vl * nq);
  const VSample vs = decode_vsample(p, v, a.B);
  const double* xr = a.x + vs.b * a.ldx;
  const bool local = kq >= p.n_fold_nonlocal;
  const int q = local ? p.fold_local[kq - p.n_fold_nonlocal] : p.fold_nonlocal[kq];
  bool any = false;
  for (int j = p.fold_ptr[q]; j < p.fold_ptr[q + 1]; ++j) any |= p.fold_dslot[j] >= 0;
  if (!any) return;
  __shared__ double u[64][4];
  __shared__ double red[8][4];
  __shared__ double r[4];
  for (int qq = tid; qq < p.n_qubits; qq += T) fold_state(p, vs, xr, a.theta, qq, u[qq]);
  __syncthreads();
  if (local) {
    // tile qubit: Σ over this sample's CTAs of the per-CTA reduced adjoints
    if (tid == 0) {
      const int j = kq - p.n_fold_nonlocal, nlq = p.n_fold_local;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int ch = 0; ch < n_chunks; ++ch)
        for (int c = 0; c < 2; ++c) {
          const double* src = a.locpart + 2 * (((int64_t)vl * n_chunks + ch) * 2 * nlq + 2 * j + c);
          acc[2 * c] += src[0];
          acc[2 * c + 1] += src[1];
        }
      for (int c = 0; c < 4; ++c) r[c] = acc[c];
    }
  } else {
    const int k = kq, m = p.n_fold_nonlocal;
    const double* lam = a.lamN + 2 * vl * (1ll << m);
    // weight(t) = Π_{i≠k} u_i[bit_i(t)] = W_hi(t >> Lb) · W_lo(t mod 2^Lb)
    const int Lb = m < 9 ? m : 9;
    __shared__ double2 wlo[512];
    for (int lo = tid; lo < (1 << Lb); lo += T) {
      double wr = 1.0, wi = 0.0;
      for (int i = 0; i < Lb; ++i) {
        if (i == k) continue;
        const double* f = u[p.fold_nonlocal[i]] + 2 * ((lo >> i) & 1);
        const double nr = wr * f[0] - wi * f[1];
        wi = wr * f[1] + wi * f[0];
        wr = nr;
      }
      wlo[lo] = make_double2(wr, wi);
    }
    __syncthreads();
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t hi = 0; hi < (1ll << (m - Lb)); ++hi) {
      double hr = 1.0, hm = 0.0;
      for (int i = Lb; i < m; ++i) {
        if (i == k) continue;
        const double* f = u[p.fold_nonlocal[i]] + 2 * ((hi >> (i - Lb)) & 1);
        const double nr = hr * f[0] - hm * f[1];
        hm = hr * f[1] + hm * f[0];
        hr = nr;
      }
      if (hr == 0.0 && hm == 0.0) continue;
      for (int lo = tid; lo < (1 << Lb); lo += T) {
        const int64_t t = (hi << Lb) | lo;
        const double2 w = wlo[lo];
        const double wr = hr * w.x - hm * w.y, wi = hr * w.y + hm * w.x;
        const double lr = lam[2 * t], li = lam[2 * t + 1];
        const int c = (int)((t >> k) & 1);
        acc[2 * c] += lr * wr + li * wi;
        acc[2 * c + 1] += li * wr - lr * wi;
      }
    }
    for (int c = 0; c < 4; ++c) {
      double x = acc[c];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if ((tid & 31) == 0) red[tid >> 5][c] = x;
    }
    __syncthreads();
    if (tid == 0)
      for (int c = 0; c < 4; ++c) {
        double x = 0.0;
        for (int w = 0; w < (T >> 5); ++w) x += red[w][c];
        r[c] = x;
      }
  }
  __syncthreads();
  if (tid == 0) {
    // states after each folded gate, then the adjoint walk back
    const int j0 = p.fold_ptr[q], K = p.fold_ptr[q + 1] - j0;
    double st[33][4];
    st[0][0] = 1.0; st[0][1] = 0.0; st[0][2] = 0.0; st[0][3] = 0.0;
    double ang[32];
    for (int j = 0; j < K; ++j) {
      const int s = p.fold_slot[j0 + j];
      ang[j] = s >= 0 ? eval_slot(p, s, xr, a.theta, vs.shvar, vs.shval) : 0.0;
      for (int c = 0; c < 4; ++c) st[j + 1][c] = st[j][c];
      apply_1q(p.fold_kind[j0 + j], ang[j], false, st[j + 1]);
    }
    double y[4] = {r[0], r[1], r[2], r[3]};
    for (int j = K - 1; j >= 0; --j) {
      const int ds = p.fold_dslot[j0 + j];
      if (ds >= 0) {
        // X[b'][b] = a_b conj(y_b'), a = st[j + 1]
        auto X = [&](int bp, int b, double* re, double* im) {
          const double ar = st[j + 1][2 * b], ai = st[j + 1][2 * b + 1];
          const double yr = y[2 * bp], yi = -y[2 * bp + 1];
          *re = ar * yr - ai * yi;
          *im = ar * yi + ai * yr;
        };
        double r10, i10, r01, i01, r11, i11;
        X(1, 0, &r10, &i10);
        X(0, 1, &r01, &i01);
        X(1, 1, &r11, &i11);
        const int kind = p.fold_kind[j0 + j];
        const double dot = kind == HQ_GATE_RY ? r10 - r01 : kind == HQ_GATE_RX ? i01 + i10 : -2.0 * i11;
        double* dst = a.dpart + ((int64_t)v * p.n_adj + ds) * a.n_parts;
        dst[0] = dot;
        for (int pp = 1; pp < a.n_parts; ++pp) dst[pp] = 0.0;
      }
      apply_1q(p.fold_kind[j0 + j], ang[j], true, y);
    }
  }
}

static int rb_of(const hq_plan_s* pl) { return pl->reg_bits; }

static WPass wpass(const hq_plan_s* pl, int i) {
  const Pass& P = pl->passes[i];
  WPass w;
  w.q = pl->tile_bits;
  w.tbits = pl->tile_bits - rb_of(pl);
  w.n_win = (int32_t)P.wins.size();
  w.n_wops = (int32_t)P.wops.size();
  w.n_slots = (int32_t)P.slots.size();
  w.n_dl = P.n_dslots_pass;
  w.first = i == 0;
  w.last = i == (int)pl->passes.size() - 1;
  w.wins = pl->d_wins + P.first_win;
  w.wops = pl->d_wops + P.first_wop;
  w.slots = pl->d_pass_slots + P.first_slotlist;
  w.dlist = pl->d_pass_dlist + P.first_dlist;
  w.local = pl->d_pass_local + (size_t)i * pl->n_qubits;
  w.nonlocal = w.local + pl->tile_bits;
  return w;
}

static JPass jpass(const hq_plan_s* pl, int i, const SArgs& sa) {
  const Pass& P = pl->passes[i];
  JPass j;
  j.v0 = sa.v0;
  j.nv = sa.nv;
  j.n_chunks = sa.n_chunks;
  j.tpc = sa.tpc;
  j.first = i == 0;
  j.last = i == (int)pl->passes.size() - 1;
  j.n_slots = (int32_t)P.slots.size();
  j.n_dl = P.n_dslots_pass;
  j.psi = sa.psi;
  j.psi_out = sa.psi;
  j.lam = sa.lam;
  j.rpart = sa.rpart;
  j.slots = pl->d_pass_slots + P.first_slotlist;
  j.dlist = pl->d_pass_dlist + P.first_dlist;
  j.local = pl->d_pass_local + (size_t)i * pl->n_qubits;
  j.nonlocal = j.local + pl->tile_bits;
  return j;
}

static size_t wsmem(const hq_plan_s* pl, int i, bool bwd) {
  const Pass& P = pl->passes[i];
  const int amp = pl->precision == HQ_C64 ? 8 : 16;
  const int T = 1 << (pl->tile_bits - rb_of(pl));
  size_t extra;
  if (bwd) extra = (size_t)P.n_dslots_pass * (T / 32) * 8;
  else extra = (size_t)((i == 0 ? ((pl->prep_total + 1) & ~1) : 0) + 96) * 8;
  return wlayout(pl->tile_bits, amp, bwd ? 2 : 1, (int)P.slots.size(), (int)P.wins.size(),
                 (int)P.wops.size(), extra).total;
}

size_t stream_smem_bytes(const hq_plan_s* pl, int pass, bool bwd) { return wsmem(pl, pass, bwd); }

template <typename R>
static cudaError_t run_stream_t(const hq_plan_s* pl, const KArgs& a, const StreamWs& ws, cudaStream_t st) {
  const int n = pl->n_qubits;
  const int T = 1 << (pl->tile_bits - RBits<R>::v);
  const int64_t n_tiles = 1ll << (n - pl->tile_bits);
  const int n_chunks = ws.n_chunks;
  const int tpc = (int)(n_tiles / n_chunks);
  const int np = (int)pl->passes.size();
  size_t sf = 0, sb = 0;
  for (int i = 0; i < np; ++i) {
    sf = std::max(sf, wsmem(pl, i, false));
    sb = std::max(sb, wsmem(pl, i, true));
  }
  const bool exact = a.state != nullptr;
  cudaError_t e0 = pl->jit.ok ? cudaSuccess : exact
      ? cudaFuncSetAttribute(k_wfwd<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf)
      : cudaFuncSetAttribute(k_wfwd<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
  if (e0 == cudaSuccess && !pl->jit.ok)
    e0 = cudaFuncSetAttribute(k_wbwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  if (e0 != cudaSuccess) return e0;
  const double amp = (double)sizeof(typename Cx<R>::T) * (double)(1ll << n);
  // real rows [0, B) then shifted rows [B, V): only real-row launches run the adjoint
  const int64_t ranges[2][2] = {{0, a.B}, {a.B, a.V}};
  for (int r = 0; r < 2; ++r) {
    for (int64_t v0 = ranges[r][0]; v0 < ranges[r][1]; v0 += ws.chunk_samples) {
      const int64_t nv = std::min<int64_t>(ranges[r][1] - v0, ws.chunk_samples);
      const bool adj = r == 0 && a.want_adj && pl->n_adj > 0;
      SArgs sa;
      sa.v0 = v0;
      sa.nv = nv;
      sa.n_chunks = n_chunks;
      sa.tpc = tpc;
      sa.psi = ws.psi;
      sa.lam = adj ? ws.lam : nullptr;
      sa.rpart = ws.rpart;
      const double vec = (double)nv * amp;
      // specialised kernels + adjoint: the last forward pass and its backward
      // run fused (λ = wψ in registers, no ψ/λ round trip through HBM)
      const bool fuse = pl->jit.ok && adj && pl->jit.fused != nullptr;
      // checkpoint k (ψ after forward pass k-1) of this launch's samples
      const bool ck = adj && ws.ckpt > 0;
      auto ckpt_ptr = [&](int k) -> void* {
        return static_cast<char*>(ws.psi) + (size_t)(k - 1) * (size_t)ws.chunk_samples *
                                                 sizeof(typename Cx<R>::T) * ((size_t)1 << n);
      };
      for (int i = 0; i < np; ++i) {
        sa.ps = wpass(pl, i);
        const size_t sm = wsmem(pl, i, false);
        if (fuse && i == np - 1) {
          JPass jp = jpass(pl, i, sa);
          if (ck) { jp.psi = ckpt_ptr(i); jp.psi_out = nullptr; }
          ProfScope prof(pl, st, HQ_K_PASS_BWD, vec * ((i == 0 ? 0 : 1) + (i == 0 ? 0 : (ck ? 1 : 2))));
          cudaError_t e = jit_launch_pass(pl, i, 2, a, jp, (unsigned)(nv * n_chunks), st);
          if (e != cudaSuccess) return e;
          continue;
        }
        ProfScope prof(pl, st, HQ_K_PASS_FWD, vec * ((i == 0 ? 0 : 1) + 1 + ((i == np - 1 && adj) ? 1 : 0)));
        if (pl->jit.ok) {
          JPass jp = jpass(pl, i, sa);
          if (ck) { jp.psi = i == 0 ? nullptr : ckpt_ptr(i); jp.psi_out = ckpt_ptr(i + 1); }
          cudaError_t e = jit_launch_pass(pl, i, 0, a, jp, (unsigned)(nv * n_chunks), st);
          if (e != cudaSuccess) return e;
        } else if (exact) {
          k_wfwd<R, true><<<(unsigned)(nv * n_chunks), T, sm, st>>>(a, sa);
        } else {
          k_wfwd<R, false><<<(unsigned)(nv * n_chunks), T, sm, st>>>(a, sa);
        }
      }
      {
        ProfScope prof(pl, st, HQ_K_OTHER, (double)nv * n_chunks * 8.0);
        k_readout_fold<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(ws.rpart, v0, nv, n_chunks, a.B,
                                                                    a.out, a.tp);
      }
      if (adj) {
        for (int i = fuse ? np - 2 : np - 1; i >= 0; --i) {
          sa.ps = wpass(pl, i);
          const size_t sm = wsmem(pl, i, true);
          ProfScope prof(pl, st, HQ_K_PASS_BWD, vec * (2 + (i == 0 ? 0 : (ck ? 1 : 2))));
          if (pl->jit.ok) {
            JPass jp = jpass(pl, i, sa);
            if (ck) { jp.psi = ckpt_ptr(i + 1); jp.psi_out = nullptr; }
            cudaError_t e = jit_launch_pass(pl, i, 1, a, jp, (unsigned)(nv * n_chunks), st);
            if (e != cudaSuccess) return e;
          } else {
            k_wbwd<R><<<(unsigned)(nv * n_chunks), T, sm, st>>>(a, sa);
          }
        }
        if (pl->fold_grad) {
          ProfScope prof(pl, st, HQ_K_OTHER, (double)nv * 16.0 * (double)n_tiles);
          const int nq = pl->dev.n_fold_nonlocal + pl->dev.n_fold_local;
          k_fold_grad<<<(unsigned)(nv * nq), 256, 0, st>>>(a, v0, n_chunks);
        }
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

cudaError_t run_stream(const hq_plan_s* pl, const KArgs& a, const StreamWs& ws, cudaStream_t st) {
  return pl->precision == HQ_C64 ? run_stream_t<float>(pl, a, ws, st) : run_stream_t<double>(pl, a, ws, st);
}

// Segment plans (amplitude-sharded execution): every pass in place on the
// caller's state rows psi [B, 2^n] (and λ rows for the backward direction).
// Forward: passes 0..np-1; backward: passes np-1..0 un-applying ψ, applying
// G† to λ and writing per-CTA derivative partials into a.dpart.
cudaError_t run_segment(const hq_plan_s* pl, const KArgs& a, void* psi, void* lam, int32_t n_chunks, bool backward,
                        cudaStream_t st) {
  const int n = pl->n_qubits;
  const int64_t n_tiles = 1ll << (n - pl->tile_bits);
  const int tpc = (int)(n_tiles / n_chunks);
  const int np = (int)pl->passes.size();
  const double vec = (double)a.B * (double)(pl->precision == HQ_C64 ? 8 : 16) * (double)(1ll << n);
  SArgs sa;
  sa.v0 = 0;
  sa.nv = a.B;
  sa.n_chunks = n_chunks;
  sa.tpc = tpc;
  sa.psi = psi;
  sa.lam = backward ? lam : nullptr;
  sa.rpart = nullptr;
  for (int k = 0; k < np; ++k) {
    const int i = backward ? np - 1 - k : k;
    sa.ps = wpass(pl, i);
    JPass jp = jpass(pl, i, sa);   // psi_out = psi: in place
    ProfScope prof(pl, st, backward ? HQ_K_PASS_BWD : HQ_K_PASS_FWD, vec * (backward ? 4.0 : 2.0));
    cudaError_t e = jit_launch_pass(pl, i, backward ? 1 : 0, a, jp, (unsigned)(a.B * n_chunks), st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace hq
