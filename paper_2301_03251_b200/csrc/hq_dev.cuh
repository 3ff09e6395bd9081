// Device helpers shared by the static kernels and the NVRTC-generated ones
// (embedded verbatim into every JIT program: CUDA builtins only, no includes).
#pragma once

namespace hq {

// Value of a tape variable for virtual sample (xrow, shifted var).
__device__ __forceinline__ double var_value(const DevPlan& p, int var, const double* xrow,
                                            const double* theta, int shvar, double shval) {
  double v = var < p.n_inputs ? xrow[var] : theta[var - p.n_inputs];
  if (var == shvar) v += shval;
  return v;
}

__device__ __forceinline__ double eval_slot(const DevPlan& p, int s, const double* xrow,
                                            const double* theta, int shvar, double shval) {
  double v = p.slot_const[s];
  const int k1 = p.slot_ptr[s + 1];
  for (int k = p.slot_ptr[s]; k < k1; ++k)
    v += p.slot_coef[k] * var_value(p, p.slot_var[k], xrow, theta, shvar, shval);
  return v;
}

// Virtual sample v: v < B are the real rows; the rest are the shifted rows of
// the batched two-point rule (qnn.py:44-51): row b, variable tp_var[j],
// +shift (k even) / -shift (k odd).
struct VSample {
  int64_t b;
  int shvar;
  double shval;
  int64_t u;  // index into the two-point result buffer, -1 for real rows
};

__device__ __forceinline__ VSample decode_vsample(const DevPlan& p, int64_t v, int64_t B) {
  VSample r;
  if (v < B) { r.b = v; r.shvar = -1; r.shval = 0.0; r.u = -1; return r; }
  const int64_t u = v - B;
  const int64_t per = 2 * (int64_t)p.n_tp;
  r.b = u / per;
  const int k = (int)(u - r.b * per);
  r.shvar = p.tp_var[k >> 1];
  r.shval = (k & 1) ? -p.shift : p.shift;
  r.u = u;
  return r;
}

template <typename R>
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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


__device__ __forceinline__ uint32_t swz(uint32_t j) { return j ^ (((j >> 4) ^ (j >> 8)) & 15u); }

}  // namespace hq

// ---------------------------------------------------------------------------
// streaming-tile helpers (shared by the static window kernels and JIT passes)
namespace hq {

// lut[c*64 + b] = global offset of tile bits {6c..6c+5} = b
__device__ __forceinline__ void lut_build(const int32_t* local, int q, uint64_t* lut, int tid, int T) {
  for (int i = tid; i < 192; i += T) {
    const int chunk = i >> 6;
    const uint32_t bits = (uint32_t)(i & 63);
    uint64_t off = 0;
    for (int k = 0; k < 6; ++k) {
      const int tb = chunk * 6 + k;
      if (tb < q && ((bits >> k) & 1u)) off |= 1ull << local[tb];
    }
    lut[i] = off;
  }
}

__device__ __forceinline__ uint64_t lut_off(const uint64_t* lut, uint32_t j) {
  return lut[j & 63u] | lut[64 + ((j >> 6) & 63u)] | lut[128 + ((j >> 12) & 63u)];
}

__device__ __forceinline__ uint64_t tile_base_of(const int32_t* nonlocal, int nb, uint64_t tile) {
  uint64_t base = 0;
  for (int i = 0; i < nb; ++i) base |= ((tile >> i) & 1ull) << nonlocal[i];
  return base;
}

// Per listed slot, 8 values: (c, s) of half the angle, (cos, sin) of the full
// angle, and the 3-shear form of the half-angle rotation
//   [[c,-s],[s,c]] = sg * shear(t) * shear_y(u) * shear(t),
// folded to |phi| <= pi/2 (sg = -1 absorbs the rest) so |t| <= 1.
template <typename R>
__device__ __forceinline__ void load_trig8(const KArgs& a, const VSample& vs, const int32_t* slots,
                                           int n_slots, R* trig, int tid, int T) {
  const double* xr = a.x + vs.b * a.ldx;
  for (int i = tid; i < n_slots; i += T) {
    const double v = eval_slot(a.p, slots[i], xr, a.theta, vs.shvar, vs.shval);
    double sn, cs;
    sincos(0.5 * v, &sn, &cs);
    const double sg = cs < 0.0 ? -1.0 : 1.0;
    const double c2 = sg * cs, s2 = sg * sn;
    trig[8 * i + 0] = (R)cs;
    trig[8 * i + 1] = (R)sn;
    trig[8 * i + 2] = (R)(cs * cs - sn * sn);
    trig[8 * i + 3] = (R)(2.0 * cs * sn);
    trig[8 * i + 4] = (R)(-s2 / (1.0 + c2));
    trig[8 * i + 5] = (R)s2;
    trig[8 * i + 6] = (R)sg;
    trig[8 * i + 7] = (R)0;
  }
}

// Exact 2x2 single-qubit gate (qsim.py:25-45 conventions) on z = (a0, a1)
// stored as {re0, im0, re1, im1}; inv applies the adjoint.
__device__ inline void apply_1q(int kind, double ang, bool inv, double* z) {
  const double r0 = z[0], i0 = z[1], r1 = z[2], i1 = z[3];
  const double th = inv ? -ang : ang;
  switch (kind) {
    case HQ_GATE_H: {
      const double h = 0.70710678118654752440;
      z[0] = h * (r0 + r1); z[1] = h * (i0 + i1); z[2] = h * (r0 - r1); z[3] = h * (i0 - i1);
      break;
    }
    case HQ_GATE_X: z[0] = r1; z[1] = i1; z[2] = r0; z[3] = i0; break;
    case HQ_GATE_Y:   // [[0, -i], [i, 0]] (self-adjoint)
      z[0] = i1; z[1] = -r1; z[2] = -i0; z[3] = r0;
      break;
    case HQ_GATE_Z: z[2] = -r1; z[3] = -i1; break;
    case HQ_GATE_RX: {  // [[c, -is], [-is, c]]
      double s, c;
      sincos(0.5 * th, &s, &c);
      z[0] = c * r0 + s * i1; z[1] = c * i0 - s * r1;
      z[2] = c * r1 + s * i0; z[3] = c * i1 - s * r0;
      break;
    }
    case HQ_GATE_RY: {  // [[c, -s], [s, c]]
      double s, c;
      sincos(0.5 * th, &s, &c);
      z[0] = c * r0 - s * r1; z[1] = c * i0 - s * i1;
      z[2] = s * r0 + c * r1; z[3] = s * i0 + c * i1;
      break;
    }
    case HQ_GATE_RZ: {  // diag(e^{-iθ/2}, e^{iθ/2})
      double s, c;
      sincos(0.5 * th, &s, &c);
      z[0] = c * r0 + s * i0; z[1] = c * i0 - s * r0;
      z[2] = c * r1 - s * i1; z[3] = c * i1 + s * r1;
      break;
    }
    default: break;
  }
}

// Factor of qubit q in the initial product state: its folded gates on |0>.
__device__ inline void fold_state(const DevPlan& p, const VSample& vs, const double* xr, const double* theta,
                                  int q, double* z) {
  z[0] = 1.0; z[1] = 0.0; z[2] = 0.0; z[3] = 0.0;
  for (int k = p.fold_ptr[q]; k < p.fold_ptr[q + 1]; ++k) {
    const int s = p.fold_slot[k];
    apply_1q(p.fold_kind[k], s >= 0 ? eval_slot(p, s, xr, theta, vs.shvar, vs.shval) : 0.0, false, z);
  }
}

__device__ __forceinline__ void load_prep_values(const KArgs& a, const VSample& vs, double* sval,
                                                 int tid, int T) {
  const double* xr = a.x + vs.b * a.ldx;
  for (int pp = 0; pp < a.p.n_preps; ++pp) {
    const int s0 = a.p.prep_slot0[pp], len = a.p.prep_len[pp], off = a.prep_off[pp];
    for (int j = tid; j < len; j += T) sval[off + j] = eval_slot(a.p, s0 + j, xr, a.theta, vs.shvar, vs.shval);
  }
}

}  // namespace hq
