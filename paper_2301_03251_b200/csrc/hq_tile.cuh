// Device building blocks: complex helpers, slot evaluation, and the gate /
// adjoint-step executors over a shared-memory tile of 2^q amplitudes.
//
// Gate conventions restate pkg/src/hyqnet/qsim.py:33-45,150-176: qubit k is
// bit k of the index; RX=[[c,-is],[-is,c]], RY=[[c,-s],[s,c]],
// RZ=diag(e^{-iθ/2},e^{iθ/2}) with c=cos θ/2, s=sin θ/2; CNOT(control,target);
// CZ negates |11>; CR(θ) multiplies |11> by e^{iθ}; SWAP exchanges |01>,|10>.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hq_internal.h"
#include "hq_dev.cuh"

namespace hq {

template <typename R> struct CT;
template <> struct CT<float> { using T = float2; };
template <> struct CT<double> { using T = double2; };

template <typename R>
struct Cx {
  using T = typename CT<R>::T;
};

template <typename C, typename R>
__device__ __forceinline__ C cmake(R re, R im) { C c; c.x = re; c.y = im; return c; }

// a*b
template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r;
}
// a*b + c*d
template <typename C>
__device__ __forceinline__ C cmul2(C a, C b, C c, C d) {
  C r;
  r.x = a.x * b.x - a.y * b.y + c.x * d.x - c.y * d.y;
  r.y = a.x * b.y + a.y * b.x + c.x * d.y + c.y * d.x;
  return r;
}

template <typename C>
struct M2 { C m00, m01, m10, m11; };

// 2x2 matrix of a non-controlled kind; INV gives the conjugate transpose.
template <typename R, bool INV>
__device__ __forceinline__ M2<typename Cx<R>::T> gate_matrix(int kind, double2 cs) {
  using C = typename Cx<R>::T;
  const R c = (R)cs.x;
  const R s = INV ? (R)(-cs.y) : (R)cs.y;
  const R z = (R)0, o = (R)1;
  M2<C> m;
  switch (kind) {
    case HQ_GATE_H: {
      const R h = (R)0.70710678118654752440;
      m.m00 = cmake<C, R>(h, z); m.m01 = cmake<C, R>(h, z);
      m.m10 = cmake<C, R>(h, z); m.m11 = cmake<C, R>(-h, z);
      break;
    }
    case HQ_GATE_X:
      m.m00 = cmake<C, R>(z, z); m.m01 = cmake<C, R>(o, z);
      m.m10 = cmake<C, R>(o, z); m.m11 = cmake<C, R>(z, z);
      break;
    case HQ_GATE_Y:
      m.m00 = cmake<C, R>(z, z); m.m01 = cmake<C, R>(z, -o);
      m.m10 = cmake<C, R>(z, o); m.m11 = cmake<C, R>(z, z);
      break;
    case HQ_GATE_RX:
      m.m00 = cmake<C, R>(c, z); m.m01 = cmake<C, R>(z, -s);
      m.m10 = cmake<C, R>(z, -s); m.m11 = cmake<C, R>(c, z);
      break;
    default:  // HQ_GATE_RY
      m.m00 = cmake<C, R>(c, z); m.m01 = cmake<C, R>(-s, z);
      m.m10 = cmake<C, R>(s, z); m.m11 = cmake<C, R>(c, z);
      break;
  }
  return m;
}

__device__ __forceinline__ uint32_t ins0(uint32_t p, int t) {
  return ((p >> t) << (t + 1)) | (p & ((1u << t) - 1u));
}
__device__ __forceinline__ uint32_t ins00(uint32_t p, int lo, int hi) {
  return ins0(ins0(p, lo), hi);
}

// ---------------------------------------------------------------------------
// Forward (INV=false) or inverse (INV=true) application of one op to a tile.
// `base` holds the global index bits of the non-resident qubits.
template <typename R, bool INV>
__device__ __forceinline__ void tile_apply(typename Cx<R>::T* s, int q, const DOp& op,
                                           const double2* trig, uint64_t base, int tid, int T) {
  using C = typename Cx<R>::T;
  const uint32_t half = 1u << (q - 1);
  const int kind = op.kind;
  switch (kind) {
    case HQ_GATE_H: case HQ_GATE_X: case HQ_GATE_Y: case HQ_GATE_RX: case HQ_GATE_RY: {
      const double2 cs = op.slot >= 0 ? trig[op.slot] : make_double2(1.0, 0.0);
      const M2<C> m = gate_matrix<R, INV>(kind, cs);
      const int t = op.a;
      for (uint32_t p = tid; p < half; p += T) {
        const uint32_t i0 = ins0(p, t), i1 = i0 | (1u << t);
        const C a0 = s[i0], a1 = s[i1];
        s[i0] = cmul2(m.m00, a0, m.m01, a1);
        s[i1] = cmul2(m.m10, a0, m.m11, a1);
      }
      break;
    }
    case HQ_GATE_Z: case HQ_GATE_RZ: {
      C d0, d1;
      if (kind == HQ_GATE_Z) {
        d0 = cmake<C, R>((R)1, (R)0); d1 = cmake<C, R>((R)-1, (R)0);
      } else {
        const double2 cs = trig[op.slot];
        const R c = (R)cs.x, sn = INV ? (R)(-cs.y) : (R)cs.y;
        d0 = cmake<C, R>(c, -sn); d1 = cmake<C, R>(c, sn);
      }
      if (op.a >= 0) {
        const int t = op.a;
        for (uint32_t p = tid; p < half; p += T) {
          const uint32_t i0 = ins0(p, t), i1 = i0 | (1u << t);
          s[i0] = cmul(s[i0], d0);
          s[i1] = cmul(s[i1], d1);
        }
      } else {
        const C d = ((base >> (~op.a)) & 1ull) ? d1 : d0;
        for (uint32_t i = tid; i < 2 * half; i += T) s[i] = cmul(s[i], d);
      }
      break;
    }
    case HQ_GATE_CNOT: {
      const int t = op.b;
      if (op.a >= 0) {
        const int c = op.a;
        const int lo = c < t ? c : t, hi = c < t ? t : c;
        for (uint32_t p = tid; p < (half >> 1); p += T) {
          const uint32_t i0 = ins00(p, lo, hi) | (1u << c), i1 = i0 | (1u << t);
          const C a0 = s[i0];
          s[i0] = s[i1];
          s[i1] = a0;
        }
      } else if ((base >> (~op.a)) & 1ull) {
        for (uint32_t p = tid; p < half; p += T) {
          const uint32_t i0 = ins0(p, t), i1 = i0 | (1u << t);
          const C a0 = s[i0];
          s[i0] = s[i1];
          s[i1] = a0;
        }
      }
      break;
    }
    case HQ_GATE_CZ: case HQ_GATE_CR: {
      C ph;
      if (kind == HQ_GATE_CZ) {
        ph = cmake<C, R>((R)-1, (R)0);
      } else {
        const double2 cs = trig[op.slot];
        const double co = cs.x * cs.x - cs.y * cs.y, si = 2.0 * cs.x * cs.y;
        ph = cmake<C, R>((R)co, INV ? (R)(-si) : (R)si);
      }
      int la = op.a, lb = op.b;
      if (la < 0) { if (!((base >> (~la)) & 1ull)) break; la = -1; }
      if (lb < 0) { if (!((base >> (~lb)) & 1ull)) break; lb = -1; }
      if (la >= 0 && lb >= 0) {
        const int lo = la < lb ? la : lb, hi = la < lb ? lb : la;
        for (uint32_t p = tid; p < (half >> 1); p += T) {
          const uint32_t i = ins00(p, lo, hi) | (1u << la) | (1u << lb);
          s[i] = cmul(s[i], ph);
        }
      } else if (la >= 0 || lb >= 0) {
        const int x = la >= 0 ? la : lb;
        for (uint32_t p = tid; p < half; p += T) {
          const uint32_t i = ins0(p, x) | (1u << x);
          s[i] = cmul(s[i], ph);
        }
      } else {
        for (uint32_t i = tid; i < 2 * half; i += T) s[i] = cmul(s[i], ph);
      }
      break;
    }
    case HQ_GATE_SWAP: {
      const int a = op.a, b = op.b;
      const int lo = a < b ? a : b, hi = a < b ? b : a;
      for (uint32_t p = tid; p < (half >> 1); p += T) {
        const uint32_t i = ins00(p, lo, hi), ia = i | (1u << a), ib = i | (1u << b);
        const C t0 = s[ia];
        s[ia] = s[ib];
        s[ib] = t0;
      }
      break;
    }
    default:
      break;
  }
}

// Im(conj(a) b), Re(conj(a) b)
template <typename C>
__device__ __forceinline__ auto cimdot(C a, C b) { return a.x * b.y - a.y * b.x; }
template <typename C>
__device__ __forceinline__ auto credot(C a, C b) { return a.x * b.x + a.y * b.y; }

// Adjoint step for one op at (psi_k, lam_k): returns this thread's share of
// dE/dα_k (when want_dot) and then un-applies the op on both vectors.
//   RX/RY/RZ: dE/dα = Im<λ|G|ψ> (G = X, Y, Z);  CR: dE/dα = -2 Im<λ|P11|ψ>.
template <typename R>
__device__ __forceinline__ double tile_adjoint_step(typename Cx<R>::T* psi, typename Cx<R>::T* lam,
                                                    int q, const DOp& op, const double2* trig,
                                                    uint64_t base, int tid, int T) {
  using C = typename Cx<R>::T;
  R acc = (R)0;
  const bool want = op.dslot >= 0;
  const uint32_t half = 1u << (q - 1);
  if (want) {
    switch (op.kind) {
      case HQ_GATE_RX: case HQ_GATE_RY: {
        const int t = op.a;
        for (uint32_t p = tid; p < half; p += T) {
          const uint32_t i0 = ins0(p, t), i1 = i0 | (1u << t);
          const C p0 = psi[i0], p1 = psi[i1], l0 = lam[i0], l1 = lam[i1];
          if (op.kind == HQ_GATE_RX) acc += cimdot(l0, p1) + cimdot(l1, p0);
          else acc += credot(l1, p0) - credot(l0, p1);
        }
        break;
      }
      case HQ_GATE_RZ: {
        if (op.a >= 0) {
          const int t = op.a;
          for (uint32_t p = tid; p < half; p += T) {
            const uint32_t i0 = ins0(p, t), i1 = i0 | (1u << t);
            acc += cimdot(lam[i0], psi[i0]) - cimdot(lam[i1], psi[i1]);
          }
        } else {
          for (uint32_t i = tid; i < 2 * half; i += T) acc += cimdot(lam[i], psi[i]);
          if ((base >> (~op.a)) & 1ull) acc = -acc;
        }
        break;
      }
      case HQ_GATE_CR: {
        int la = op.a, lb = op.b;
        bool live = true;
        if (la < 0) { live = live && ((base >> (~la)) & 1ull); la = -1; }
        if (lb < 0) { live = live && ((base >> (~lb)) & 1ull); lb = -1; }
        if (!live) break;
        if (la >= 0 && lb >= 0) {
          const int lo = la < lb ? la : lb, hi = la < lb ? lb : la;
          for (uint32_t p = tid; p < (half >> 1); p += T) {
            const uint32_t i = ins00(p, lo, hi) | (1u << la) | (1u << lb);
            acc += cimdot(lam[i], psi[i]);
          }
        } else if (la >= 0 || lb >= 0) {
          const int x = la >= 0 ? la : lb;
          for (uint32_t p = tid; p < half; p += T) {
            const uint32_t i = ins0(p, x) | (1u << x);
            acc += cimdot(lam[i], psi[i]);
          }
        } else {
          for (uint32_t i = tid; i < 2 * half; i += T) acc += cimdot(lam[i], psi[i]);
        }
        acc *= (R)-2;
        break;
      }
      default:
        break;
    }
  }
  // each thread re-touches exactly the elements it just read, so no barrier
  tile_apply<R, true>(psi, q, op, trig, base, tid, T);
  tile_apply<R, true>(lam, q, op, trig, base, tid, T);
  return (double)acc;
}

}  // namespace hq
