// Register-window executor for the HBM streaming passes.
//
// A tile of 2^q amplitudes is spread over T = 2^(q-RB) threads, each holding
// 2^RB amplitudes in registers.  Within a *window* the register bits map to RB
// chosen tile qubits (those whose pairs the window's gates exchange); the other
// tile qubits are thread-index bits, whose value every thread knows, so
// diagonal gates and controls on them need no data movement.  Between windows
// the tile is re-distributed through shared memory (one store + one load).
//
// Operand codes of a WOp qubit:  0..RB-1  register bit
//                                16 + s   thread-index bit s (tile qubit S_w[s])
//                                64 + g   global qubit g outside the tile (bit of the tile base)
//
// Shared-memory element j lives at swz(j) = j ^ ((j>>4 ^ j>>8) & 15): the bank
// of an 8-byte element is linear in the tile bits, so the planner can pick lane
// bits that hit all 16 bank pairs.
#pragma once

#include "hq_tile.cuh"

namespace hq {


template <int RB>
__device__ __forceinline__ uint32_t win_tbase(const WinDev& w, int tid, int tbits) {
  uint32_t t = 0;
#pragma unroll 10
  for (int s = 0; s < tbits; ++s)
    if ((tid >> s) & 1) t ^= w.ps[s];
  return t;
}

// swizzled smem index of register k (compile-time k) under window w
template <int RB, int K>
__device__ __forceinline__ uint32_t reg_phys(uint32_t tb, const uint16_t* pr) {
  uint32_t p = tb;
#pragma unroll
  for (int i = 0; i < RB; ++i)
    if (K & (1 << i)) p ^= pr[i];
  return p;
}

template <typename C, int RB>
struct RegIO {
  template <int K>
  __device__ __forceinline__ static void store(C (&a)[1 << RB], C* s, uint32_t tb, const uint16_t* pr) {
    s[reg_phys<RB, K>(tb, pr)] = a[K];
    if constexpr (K + 1 < (1 << RB)) store<K + 1>(a, s, tb, pr);
  }
  template <int K>
  __device__ __forceinline__ static void load(C (&a)[1 << RB], const C* s, uint32_t tb, const uint16_t* pr) {
    a[K] = s[reg_phys<RB, K>(tb, pr)];
    if constexpr (K + 1 < (1 << RB)) load<K + 1>(a, s, tb, pr);
  }
};

template <typename C, int RB>
__device__ __forceinline__ void regs_to_smem(C (&a)[1 << RB], C* s, const WinDev& w, int tid, int tbits) {
  uint16_t pr[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) pr[i] = w.pr[i];
  RegIO<C, RB>::template store<0>(a, s, win_tbase<RB>(w, tid, tbits), pr);
}

template <typename C, int RB>
__device__ __forceinline__ void smem_to_regs(C (&a)[1 << RB], const C* s, const WinDev& w, int tid, int tbits) {
  uint16_t pr[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) pr[i] = w.pr[i];
  RegIO<C, RB>::template load<0>(a, s, win_tbase<RB>(w, tid, tbits), pr);
}

// ---------------------------------------------------------------------------
// operand decoding
struct Operand {
  int reg;      // register bit or -1
  int fixed;    // -1 if register; else the operand's constant bit value for this thread/tile
};

__device__ __forceinline__ Operand decode(int code, int tid, uint64_t base) {
  Operand o;
  if (code < 16) { o.reg = code; o.fixed = -1; }
  else if (code < 64) { o.reg = -1; o.fixed = (tid >> (code - 16)) & 1; }
  else { o.reg = -1; o.fixed = (int)((base >> (code - 64)) & 1ull); }
  return o;
}

// ---------------------------------------------------------------------------
// register-bit templated gate bodies.  N = 2^RB amplitudes per thread.
template <typename C, typename R, int K, int N>
__device__ __forceinline__ void real2_k(C (&a)[N], R m00, R m01, R m10, R m11) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i & (1 << K)) continue;
    const C a0 = a[i], a1 = a[i | (1 << K)];
    a[i].x = m00 * a0.x + m01 * a1.x;
    a[i].y = m00 * a0.y + m01 * a1.y;
    a[i | (1 << K)].x = m10 * a0.x + m11 * a1.x;
    a[i | (1 << K)].y = m10 * a0.y + m11 * a1.y;
  }
}

// RX(c, s): a0' = c a0 - i s a1, a1' = -i s a0 + c a1
template <typename C, typename R, int K, int N>
__device__ __forceinline__ void rx_k(C (&a)[N], R c, R s) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i & (1 << K)) continue;
    const C a0 = a[i], a1 = a[i | (1 << K)];
    a[i].x = c * a0.x + s * a1.y;
    a[i].y = c * a0.y - s * a1.x;
    a[i | (1 << K)].x = s * a0.y + c * a1.x;
    a[i | (1 << K)].y = c * a1.y - s * a0.x;
  }
}

// Y: a0' = -i a1, a1' = i a0
template <typename C, int K, int N>
__device__ __forceinline__ void y_k(C (&a)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i & (1 << K)) continue;
    const C a0 = a[i], a1 = a[i | (1 << K)];
    a[i].x = a1.y;
    a[i].y = -a1.x;
    a[i | (1 << K)].x = -a0.y;
    a[i | (1 << K)].y = a0.x;
  }
}

// controlled X on target K: pairs whose (runtime) control mask is satisfied
template <typename C, int K, int N>
__device__ __forceinline__ void cx_k(C (&a)[N], int cmask, bool live) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i & (1 << K)) continue;
    const bool go = live && ((i & cmask) == cmask);
    const C a0 = a[i], a1 = a[i | (1 << K)];
    a[i] = go ? a1 : a0;
    a[i | (1 << K)] = go ? a0 : a1;
  }
}

template <typename C, typename R>
__device__ __forceinline__ C cmulr(C z, R c, R s) {
  C r;
  r.x = z.x * c - z.y * s;
  r.y = z.x * s + z.y * c;
  return r;
}

// multiply amplitudes whose register bits contain `mask` (runtime) by (c + i s)
template <typename C, typename R, int N>
__device__ __forceinline__ void phase_mask(C (&a)[N], int mask, bool live, R c, R s) {
  if (!live) return;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if ((i & mask) == mask) a[i] = cmulr(a[i], c, s);
}

#define HQ_DISPATCH_K(k, RB, CALL)                  \
  switch (k) {                                      \
    case 0: { constexpr int KK = 0; CALL; break; }  \
    case 1: { constexpr int KK = 1; CALL; break; }  \
    case 2: { if constexpr (RB > 2) { constexpr int KK = 2; CALL; } break; } \
    case 3: { if constexpr (RB > 3) { constexpr int KK = 3; CALL; } break; } \
    case 4: { if constexpr (RB > 4) { constexpr int KK = 4; CALL; } break; } \
    default: break;                                 \
  }

// Apply one op (forward, or inverse when INV) to the registers.  EXACT_RZ keeps
// RZ = diag(e^{-iφ/2}, e^{iφ/2}); otherwise the global phase is dropped and RZ
// multiplies only the |1> half by e^{iφ} (|ψ|² and <λ|G|ψ> are unchanged).
template <typename R, int RB, bool INV, bool EXACT_RZ>
__device__ __forceinline__ void wop_apply(typename Cx<R>::T (&a)[1 << RB], const WOp& op,
                                          const double2* trig, int tid, uint64_t base) {
  using C = typename Cx<R>::T;
  constexpr int N = 1 << RB;
  const Operand A = decode(op.a, tid, base);
  switch (op.kind) {
    case HQ_GATE_H: {
      const R h = (R)0.70710678118654752440;
      HQ_DISPATCH_K(A.reg, RB, (real2_k<C, R, KK, N>(a, h, h, h, -h)));
      break;
    }
    case HQ_GATE_X:
      HQ_DISPATCH_K(A.reg, RB, (cx_k<C, KK, N>(a, 0, true)));
      break;
    case HQ_GATE_Y:
      HQ_DISPATCH_K(A.reg, RB, (y_k<C, KK, N>(a)));
      break;
    case HQ_GATE_RY: {
      const double2 cs = trig[op.slot];
      const R c = (R)cs.x, s = INV ? (R)-cs.y : (R)cs.y;
      HQ_DISPATCH_K(A.reg, RB, (real2_k<C, R, KK, N>(a, c, -s, s, c)));
      break;
    }
    case HQ_GATE_RX: {
      const double2 cs = trig[op.slot];
      const R c = (R)cs.x, s = INV ? (R)-cs.y : (R)cs.y;
      HQ_DISPATCH_K(A.reg, RB, (rx_k<C, R, KK, N>(a, c, s)));
      break;
    }
    case HQ_GATE_Z: case HQ_GATE_RZ: {
      R c1, s1, c0 = (R)1, s0 = (R)0;
      if (op.kind == HQ_GATE_Z) {
        c1 = (R)-1; s1 = (R)0;
      } else {
        const double2 cs = trig[op.slot];
        if (EXACT_RZ) {
          c0 = (R)cs.x; s0 = INV ? (R)cs.y : (R)-cs.y;
          c1 = (R)cs.x; s1 = INV ? (R)-cs.y : (R)cs.y;
        } else {
          const double co = cs.x * cs.x - cs.y * cs.y, si = 2.0 * cs.x * cs.y;  // e^{iφ}
          c1 = (R)co; s1 = INV ? (R)-si : (R)si;
        }
      }
      if (A.reg >= 0) {
        const int m = 1 << A.reg;
        if (EXACT_RZ && op.kind == HQ_GATE_RZ) {
#pragma unroll
          for (int i = 0; i < N; ++i) a[i] = (i & m) ? cmulr(a[i], c1, s1) : cmulr(a[i], c0, s0);
        } else {
          phase_mask<C, R, N>(a, m, true, c1, s1);
        }
      } else {
        const R c = A.fixed ? c1 : c0, s = A.fixed ? s1 : s0;
        if (EXACT_RZ || A.fixed || op.kind != HQ_GATE_RZ) phase_mask<C, R, N>(a, 0, true, c, s);
      }
      break;
    }
    case HQ_GATE_CNOT: {
      const Operand B = decode(op.b, tid, base);  // target: always a register bit
      const int cm = A.reg >= 0 ? (1 << A.reg) : 0;
      const bool live = A.reg >= 0 ? true : (A.fixed != 0);
      HQ_DISPATCH_K(B.reg, RB, (cx_k<C, KK, N>(a, cm, live)));
      break;
    }
    case HQ_GATE_CZ: case HQ_GATE_CR: {
      const Operand B = decode(op.b, tid, base);
      R c = (R)-1, s = (R)0;
      if (op.kind == HQ_GATE_CR) {
        const double2 cs = trig[op.slot];
        c = (R)(cs.x * cs.x - cs.y * cs.y);
        s = (R)(2.0 * cs.x * cs.y);
        if (INV) s = -s;
      }
      const int m = (A.reg >= 0 ? (1 << A.reg) : 0) | (B.reg >= 0 ? (1 << B.reg) : 0);
      const bool live = (A.reg >= 0 || A.fixed) && (B.reg >= 0 || B.fixed);
      phase_mask<C, R, N>(a, m, live, c, s);
      break;
    }
    default:
      break;
  }
}

// Im<λ|Y|ψ> over pairs on register bit K = Re(λ1* ψ0) - Re(λ0* ψ1)
template <typename C, typename R, int K, int N>
__device__ __forceinline__ R dot_ry_k(const C (&p)[N], const C (&l)[N]) {
  R acc = (R)0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i & (1 << K)) continue;
    const int j = i | (1 << K);
    acc += l[j].x * p[i].x + l[j].y * p[i].y - l[i].x * p[j].x - l[i].y * p[j].y;
  }
  return acc;
}

// Im<λ|X|ψ> = Im(λ0* ψ1) + Im(λ1* ψ0)
template <typename C, typename R, int K, int N>
__device__ __forceinline__ R dot_rx_k(const C (&p)[N], const C (&l)[N]) {
  R acc = (R)0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i & (1 << K)) continue;
    const int j = i | (1 << K);
    acc += l[i].x * p[j].y - l[i].y * p[j].x + l[j].x * p[i].y - l[j].y * p[i].x;
  }
  return acc;
}

// Adjoint step at (ψ_k, λ_k): this thread's share of dE/dα (if dl >= 0), then
// un-apply the op on both register sets.
template <typename R, int RB, bool EXACT_RZ>
__device__ __forceinline__ R wop_adjoint(typename Cx<R>::T (&p)[1 << RB], typename Cx<R>::T (&l)[1 << RB],
                                         const WOp& op, const double2* trig, int tid, uint64_t base) {
  using C = typename Cx<R>::T;
  constexpr int N = 1 << RB;
  R acc = (R)0;
  if (op.dl >= 0) {
    const Operand A = decode(op.a, tid, base);
    switch (op.kind) {
      case HQ_GATE_RY:
        HQ_DISPATCH_K(A.reg, RB, (acc = dot_ry_k<C, R, KK, N>(p, l)));
        break;
      case HQ_GATE_RX:
        HQ_DISPATCH_K(A.reg, RB, (acc = dot_rx_k<C, R, KK, N>(p, l)));
        break;
      case HQ_GATE_RZ: case HQ_GATE_CR: {
        // dE/dφ = -2 Im<λ|P|ψ> over the amplitudes the phase touches
        // (RZ: |1> of the target, using Im<λ|ψ> = 0; CR: |11>)
        int m = 0;
        bool live = true;
        if (A.reg >= 0) m |= 1 << A.reg; else live = live && A.fixed;
        if (op.kind == HQ_GATE_CR) {
          const Operand B = decode(op.b, tid, base);
          if (B.reg >= 0) m |= 1 << B.reg; else live = live && B.fixed;
        }
        if (live) {
#pragma unroll
          for (int i = 0; i < N; ++i)
            if ((i & m) == m) acc += l[i].x * p[i].y - l[i].y * p[i].x;
        }
        acc *= (R)-2;
        break;
      }
      default:
        break;
    }
  }
  wop_apply<R, RB, true, EXACT_RZ>(p, op, trig, tid, base);
  wop_apply<R, RB, true, EXACT_RZ>(l, op, trig, tid, base);
  return acc;
}

}  // namespace hq
