// Plain-old-data layouts shared by the host, the static kernels and the
// NVRTC-generated kernels (this text is embedded verbatim into every JIT
// program, so it may only use int8_t..uint64_t / double / pointers, which the
// includer defines).
#pragma once

namespace hq {

// Device-resident, immutable plan constants (all pointers are device memory).
struct DevPlan {
  int32_t n_qubits;
  int32_t n_slots;
  int32_t n_inputs, n_params, n_vars;
  int32_t n_measured;
  int32_t n_preps;
  int32_t n_tp;     // two-point variables
  int32_t n_adj;    // derivative slots (distinct angle slots the adjoint sweep differentiates)
  double shift, grad_scale;
  const double* slot_const;
  const int32_t* slot_ptr;
  const int32_t* slot_var;
  const double* slot_coef;
  const int32_t* measured;
  const int32_t* prep_ptr;
  const int32_t* prep_qubits;
  const int32_t* prep_slot0;
  const int32_t* prep_len;
  const int32_t* tp_var;       // [n_tp] variable ids
  const int32_t* var_mode;     // [n_vars] HQ_GRAD_*
  const int32_t* var_dsl;      // [n_vars] ADJOINT: derivative slot
  const int32_t* var_tp;       // [n_vars] TWOPOINT: index into tp_var
  const double* var_factor;    // [n_vars] ADJOINT: 2*grad_scale*sin(coef*shift)
  int32_t n_rz;                // RZ gates (their dropped half-angle phases, for exact amplitudes)
  const int32_t* rz_slots;
  int32_t n_rot;               // RX/RY gates (their dropped global signs, specialised kernels)
  const int32_t* rot_slots;
  // folded leading single-qubit gates per qubit (initial product state)
  int32_t n_fold;
  const int32_t* fold_ptr;     // [n_qubits + 1]
  const int32_t* fold_kind;
  const int32_t* fold_slot;
  const int32_t* fold_dslot;
  const int32_t* fold_nonlocal; // first pass's non-local qubits (tile-id bit i -> qubit)
  int32_t n_fold_nonlocal;
  const int32_t* fold_local;    // first-tile qubits with differentiated folded gates
  int32_t n_fold_local;
  int32_t perm;                 // trailing X/CNOT gates folded into the readout
  const uint64_t* perm_mask;    // [n_qubits]
  const int32_t* perm_const;    // [n_qubits]
};

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
  double* lamN;             // fold_grad: λ at the first pass's start contracted over its tile, [V, 2^(n-q)] complex
  double* locpart;          // [V, n_chunks, n_fold_local, 2] complex: tile-qubit reduced adjoints per CTA
};


// Launch arguments of one generated streaming pass (hq_jit.cpp).
struct JPass {
  int64_t v0, nv;        // virtual samples of this launch
  int32_t n_chunks, tpc; // CTAs per sample, tiles per CTA
  int32_t first, last;   // pass index is 0 / the last one
  int32_t n_slots, n_dl;
  void* psi;               // ψ read by this pass (sample vl at + vl·2^n)
  void* psi_out;           // ψ written by this pass, or null (backward passes with checkpoints)
  void* lam;
  double* rpart;
  const int32_t* slots;    // pass-local slot list
  const int32_t* dlist;    // pass-local derivative index -> derivative slot
  const int32_t* local;    // [q] global qubit of tile bit i
  const int32_t* nonlocal; // [n-q] global qubit of tile-id bit i
};

}  // namespace hq
