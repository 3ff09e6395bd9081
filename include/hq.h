/*
 * hq.h — C ABI of the B200 batched variational-circuit simulator.
 *
 * This is the drop-in boundary for the reference's hot path (VQNet 2.0 /
 * `hyqnet`, pure Python + NumPy).  Each entry point replaces one piece of it:
 *
 *   hq_plan_create   replaces the per-evaluation circuit rebuild + validation:
 *                    QuantumLayer._build (pkg/src/hyqnet/qnn.py:95-105),
 *                    GateOp.__post_init__ / Circuit.add (qsim.py:54-71,109-113).
 *                    The tape is traced once per batch (tracer.py), not per
 *                    evaluation.
 *   hq_forward       replaces the serial batch loop of QuantumLayer.forward
 *                    (qnn.py:123-133): simulate (qsim.py:179-191) + apply_gate
 *                    (qsim.py:150-176) + probabilities (qsim.py:194-211) + the
 *                    EXACT_PROB readout E = Σ_j j·P(j) (qnn.py:107-116).  With
 *                    HQ_WANT_JAC it also produces, per sample, the row the
 *                    reference's df_x / df_p closures compute with
 *                    parameter_shift_grad (qnn.py:35-52,136-153) at upstream 1.
 *   hq_vjp           replaces the upstream scaling + sequential batch sum of
 *                    df_x / df_p (qnn.py:137-152).
 *   hq_state         replaces simulate() returning the amplitudes
 *                    (qsim.py:179-191), for StateVector-level parity tests.
 *   hq_sample        replaces measure_shots (qsim.py:236-248) / SHOT_SAMPLING.
 *   hq_noisy         replaces simulate_noisy (noise.py:141-153) / the NOISY
 *                    machine type (qnn.py:109-111, NoiseQuantumLayer
 *                    qnn.py:157-166) with its shift-rule gradients.
 *
 * Conventions (all pinned by the reference tests): qubit k is
 * bit k of the amplitude index; rotations are half-angle; CR(θ) multiplies
 * |11⟩ by e^{iθ}; the readout weights are w(idx) = Σ_i 2^i·bit(idx, measured[i]).
 *
 * All pointers passed to hq_forward / hq_vjp / hq_state are DEVICE pointers
 * (caller-owned, e.g. torch tensors); `stream` is a cudaStream_t.  Plans are
 * immutable after creation and may be used concurrently on distinct streams
 * with distinct workspaces.  Errors: a non-zero hq_status plus a thread-local
 * message from hq_last_error(); the Python layer maps HQ_E_CIRCUIT ->
 * CircuitError, HQ_E_CONFIG -> ConfigError, HQ_E_DIMENSION -> DimensionError,
 * HQ_E_ENCODING -> EncodingError (errors.py:8-26), anything else -> NativeError.
 */
#ifndef HQ_H
#define HQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HQ_ABI_VERSION 2

typedef struct hq_plan_s* hq_plan;

typedef enum {
  HQ_OK = 0,
  HQ_E_CIRCUIT = 1,
  HQ_E_CONFIG = 2,
  HQ_E_DIMENSION = 3,
  HQ_E_CUDA = 4,
  HQ_E_OOM = 5,
  HQ_E_ENCODING = 6
} hq_status;

/* amplitude precision: complex64 (fast mode, 1e-5) or complex128 (reference, 1e-10) */
enum { HQ_C64 = 0, HQ_C128 = 1 };

/* gate kinds: qsim.py:19-22 plus the native state load */
enum {
  HQ_GATE_H = 0, HQ_GATE_X = 1, HQ_GATE_Y = 2, HQ_GATE_Z = 3,
  HQ_GATE_RX = 4, HQ_GATE_RY = 5, HQ_GATE_RZ = 6,
  HQ_GATE_CNOT = 7, HQ_GATE_CZ = 8, HQ_GATE_CR = 9, HQ_GATE_SWAP = 10,
  HQ_GATE_STATEPREP = 11
};

/* gradient mode per variable (inputs first, then params) */
enum { HQ_GRAD_ZERO = 0, HQ_GRAD_ADJOINT = 1, HQ_GRAD_TWOPOINT = 2 };

/* hq_forward flags */
enum { HQ_WANT_JAC = 1 };

/* One tape entry.  q0 is the control of CNOT/CZ/CR (GateOp targets order).
 * slot indexes the affine slot table for RX/RY/RZ/CR, else -1.
 * STATEPREP: q0 = index into the prep table, q1 = slot = -1. */
typedef struct {
  int32_t kind, q0, q1, slot;
} hq_op;

typedef struct {
  int32_t n_qubits;
  int32_t precision;                 /* HQ_C64 | HQ_C128 */
  int32_t n_ops;
  const hq_op* ops;
  /* affine slots: value[s] = slot_const[s] + Σ_{k in [slot_ptr[s], slot_ptr[s+1])}
   *               slot_coef[k] * var[slot_var[k]],  var = [inputs | params] */
  int32_t n_slots;
  const double* slot_const;
  const int32_t* slot_ptr;           /* n_slots + 1 */
  const int32_t* slot_var;
  const double* slot_coef;
  int32_t n_inputs, n_params;
  int32_t n_measured;                /* 0 => all qubits (qnn.py:108) */
  const int32_t* measured;
  /* state loads (amplitude_embedding): prep p covers qubits
   * prep_qubits[prep_ptr[p] .. prep_ptr[p+1]) (value bit i -> qubit i of that
   * list) with values = slots [prep_slot0[p], prep_slot0[p] + prep_len[p]) */
  int32_t n_preps;
  const int32_t* prep_ptr;
  const int32_t* prep_qubits;
  const int32_t* prep_slot0;
  const int32_t* prep_len;
  /* gradient spec, length n_inputs + n_params (NULL => no gradient) */
  const int32_t* grad_mode;
  const int32_t* grad_slot;          /* ADJOINT: the single slot the variable enters */
  const double* grad_factor;         /* ADJOINT: 2*grad_scale*sin(coef*shift) */
  double shift;                      /* qnn.py:64, default pi/2 */
  double grad_scale;                 /* qnn.py:64, default 0.5 */
} hq_plan_desc;

int hq_abi_version(void);
const char* hq_last_error(void);

hq_status hq_plan_create(const hq_plan_desc* desc, hq_plan* out);
void hq_plan_destroy(hq_plan plan);

/* human-readable execution plan (kernel choice, passes) — valid until the plan dies */
const char* hq_plan_describe(hq_plan plan);

/* bytes of device workspace hq_forward / hq_state need for `batch` samples */
size_t hq_workspace_bytes(hq_plan plan, int64_t batch, int32_t flags);

/* out[b] = E(x[b], theta); with HQ_WANT_JAC, jac[b, v] (row stride
 * n_inputs + n_params) = the reference's per-sample shift-rule gradient at
 * upstream 1 for every variable with a non-ZERO mode, 0 otherwise.
 * x: [batch, ldx] f64, theta: [n_params] f64, out: [batch] f64. */
hq_status hq_forward(hq_plan plan, const double* x, int64_t ldx, const double* theta,
                     int64_t batch, int32_t flags, double* out, double* jac,
                     void* workspace, size_t workspace_bytes, void* stream);

/* grad_x[b, i] = upstream[b] * jac[b, i];
 * grad_theta[j] = Σ_b upstream[b] * jac[b, n_inputs + j], summed in sample
 * order (qnn.py:147-152).  Either output may be NULL. */
hq_status hq_vjp(hq_plan plan, const double* jac, const double* upstream, int64_t batch,
                 double* grad_x, double* grad_theta, void* stream);

/* final amplitudes, interleaved complex128 [batch, 2^n, 2]; `init` (optional,
 * same layout, batch rows or 1 row broadcast) replaces |0...0>. */
hq_status hq_state(hq_plan plan, const double* x, int64_t ldx, const double* theta,
                   int64_t batch, const double* init, int64_t init_rows, double* state,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ---- SHOT_SAMPLING (qsim.py:222-248, qnn.py:27-32) ------------------------ */

/* Per row of `state` ([rows, 2^n, 2] complex128, device): marginal over
 * `measured` (host array, outcome bit i = measured[i]), np.cumsum order,
 * `shots` draws u_s = Philox4x64-10(key=[seed, s]).random(), outcome =
 * searchsorted(cum, u, side="right") clamped.  Outputs (device, optional):
 * counts [rows, 2^m] uint64, expectation [rows] = Σ outcome / shots. */
size_t hq_sample_workspace_bytes(int64_t rows, int32_t n_qubits, int32_t n_measured);
hq_status hq_sample(const double* state, int64_t rows, int32_t n_qubits, const int32_t* measured,
                    int32_t n_measured, int64_t shots, uint64_t seed, uint64_t* counts,
                    double* expectation, void* workspace, size_t workspace_bytes, void* stream);

/* marginal Born probabilities of each row of `state` ([rows, 2^n, 2]
 * complex128, device) over `measured` (host list, outcome bit i =
 * measured[i]): probs [rows, 2^m] (device), fixed-order sums.
 * Replaces probabilities (qsim.py:194-211) for device-resident states. */
size_t hq_marginal_workspace_bytes(int64_t rows, int32_t n_qubits, int32_t n_measured);
hq_status hq_marginal(const double* state, int64_t rows, int32_t n_qubits, const int32_t* measured,
                      int32_t n_measured, double* probs, void* workspace, size_t workspace_bytes, void* stream);

/* u_s for s in [shot0, shot0 + count): the per-shot uniform stream of shot_rng (qsim.py:222-224) */
hq_status hq_shot_uniforms(uint64_t seed, int64_t shot0, int64_t count, double* out, void* stream);

/* ---- NOISY machine type: per-shot Kraus trajectories (noise.py) ---------- */

enum { HQ_CH_BIT_FLIP = 0, HQ_CH_PHASE_FLIP = 1, HQ_CH_DEPOLARIZING = 2, HQ_CH_AMP_DAMPING = 3 };

/* One channel application: after tape op `op`, on `qubit` (one of the op's
 * targets), in the order the reference visits them (noise.py:130-138: op order,
 * then the op's targets, then the model's channel list).  Sites with param 0
 * draw nothing (noise.py:99) and may be omitted. */
typedef struct {
  int32_t op, qubit, channel;
  double param;
} hq_noise_site;

size_t hq_noisy_workspace_bytes(hq_plan plan, int64_t batch, int32_t flags, int32_t n_sites);

/* simulate_noisy for every (virtual) sample (noise.py:141-153): `shots`
 * trajectories from |0...0>, shot s drawing from Philox4x64-10(key=[seed, s])
 * (one draw per non-zero channel application, one final outcome draw).
 * out[b] = Σ outcome / shots (qnn.py:27-32); HQ_WANT_JAC: jac rows by the
 * two-point rule on the same streams (every differentiated variable must be
 * HQ_GRAD_TWOPOINT); counts (optional) [batch, 2^m] uint64.  Complex128
 * state; circuits up to 26 qubits without state loads (n > 13: the state lives
 * in the workspace, see hq_noisy_workspace_bytes).
 * Replaces: qnn.py:109-111 (NOISY _execute) and its shift-rule closures. */
hq_status hq_noisy(hq_plan plan, const double* x, int64_t ldx, const double* theta, int64_t batch,
                   int32_t flags, const hq_noise_site* sites, int32_t n_sites, int64_t shots, uint64_t seed,
                   double* out, double* jac, uint64_t* counts, void* workspace, size_t workspace_bytes,
                   void* stream);

/* ---- amplitude-sharded execution ----------------
 *
 * A circuit too large for one GPU is split by amplitude: index bits >= L are
 * the rank.  The host scheduler (shard.py) cuts the tape into local segments
 * separated by global<->local qubit exchanges (NCCL all-to-all of contiguous
 * chunks).  Each segment runs as a SEGMENT plan over the L local qubits:
 * every pass in place on the caller's shard, no readout, no folding, no
 * global-phase bookkeeping (phases common to all ranks are global phases).
 * Replaces, for n > 24 (beyond the reference, qsim.py:17): simulate
 * (qsim.py:179-191) and the df_p closure (qnn.py:145-153) of one circuit. */

/* like hq_plan_create; grad_mode may only use HQ_GRAD_ZERO / HQ_GRAD_ADJOINT */
hq_status hq_plan_create_segment(const hq_plan_desc* desc, hq_plan* out);
size_t hq_seg_workspace_bytes(hq_plan plan, int64_t batch);
/* psi: [batch, 2^n] amplitudes in the plan's precision (interleaved complex),
 * updated in place: psi <- U_segment psi */
hq_status hq_seg_forward(hq_plan plan, const double* x, int64_t ldx, const double* theta, int64_t batch,
                         void* psi, void* workspace, size_t workspace_bytes, void* stream);
/* adjoint sweep over the segment: psi <- U^-1 psi, lam <- U^† lam, and
 * jac[b, v] (row stride n_inputs + n_params) = factor_v · 2 Re<lam|dG_v|psi>
 * at each differentiated gate (0 for variables the segment does not touch);
 * summed over segments and ranks this is the df_p row (qnn.py:145-153). */
hq_status hq_seg_backward(hq_plan plan, const double* x, int64_t ldx, const double* theta, int64_t batch,
                          void* psi, void* lam, double* jac, void* workspace, size_t workspace_bytes,
                          void* stream);
/* this rank's EXACT_PROB partial  e_out[0] = Σ_j w(j)|psi_j|^2  over one shard
 * of 2^n_local amplitudes, w(j) = w0 + Σ_i wk[i]·bit(j, pos[i]) (pos/wk: host
 * arrays; local measured qubits, 2^i weights; w0: the measured rank bits);
 * fixed-order reduction; lam (optional) <- w·psi.  e_out is device memory. */
size_t hq_shard_readout_workspace_bytes(void);
hq_status hq_shard_readout(const void* psi, int32_t precision, int32_t n_local, const int32_t* pos,
                           const double* wk, int32_t k, double w0, double* e_out, void* lam, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ---- multi-GPU communicator (one process per GPU; NCCL loaded at run time) --
 * The library's own NCCL communicator for the two collectives of SURVEY.md
 * §8(e): the [P] gradient all-reduce of the sample-sharded layer and the
 * global<->local qubit all-to-all of the amplitude-sharded executor. */
typedef struct hq_comm_s* hq_comm;
size_t hq_comm_id_bytes(void);                           /* ncclUniqueId size (128) */
hq_status hq_comm_unique_id(void* id_out);               /* on one rank; share it with the others */
hq_status hq_comm_init(const void* id, int32_t rank, int32_t world, hq_comm* out);
void hq_comm_destroy(hq_comm comm);
/* in-place sum over ranks (device buffer) */
hq_status hq_comm_allreduce_f64(hq_comm comm, double* buf, int64_t count, void* stream);
/* chunk j of send -> rank j; chunk from rank j -> chunk j of recv (contiguous,
 * bytes_per_rank each; send != recv) */
hq_status hq_comm_alltoall(hq_comm comm, const void* send, void* recv, int64_t bytes_per_rank, void* stream);
/* one data-parallel step: hq_forward(HQ_WANT_JAC) + hq_vjp + all-reduce of
 * grad_theta (replaces qnn.py:131,147-152 across ranks); comm may be NULL
 * (single rank).  grad_x optional. */
hq_status hq_backward_dp(hq_plan plan, const double* x, int64_t ldx, const double* theta, int64_t batch,
                         const double* upstream, double* out, double* jac, double* grad_x, double* grad_theta,
                         hq_comm comm, void* workspace, size_t workspace_bytes, void* stream);

/* ---- introspection / measurement ---------------------------------------- */

typedef struct {
  int32_t path;              /* 0 = on-chip (state in shared memory), 1 = HBM streaming */
  int32_t n_passes;          /* streaming: HBM passes per direction */
  int32_t tile_bits;         /* amplitudes per tile = 2^tile_bits */
  int32_t n_adjoint_slots;   /* derivatives produced by the adjoint sweep */
  int32_t n_twopoint_vars;   /* variables evaluated by the batched two-point rule */
  int64_t launches;          /* kernel launches one hq_forward(batch, flags) makes */
  int64_t chunk_samples;     /* streaming: samples resident per launch */
  double state_bytes;        /* bytes of one sample's state vector */
} hq_plan_stats;

hq_status hq_stats(hq_plan plan, int64_t batch, int32_t flags, hq_plan_stats* out);

/* Kernel classes of the live profile. */
enum { HQ_K_ONCHIP = 0, HQ_K_PASS_FWD = 1, HQ_K_PASS_BWD = 2, HQ_K_OTHER = 3, HQ_K_CLASSES = 4 };

typedef struct {
  double ms[HQ_K_CLASSES];       /* summed device time per class (CUDA events) */
  int64_t launches[HQ_K_CLASSES];
  double bytes[HQ_K_CLASSES];    /* state bytes each class reads + writes (traffic model) */
} hq_profile_result;

/* While enabled, every launch of this plan is bracketed by CUDA events on its
 * stream.  hq_profile_read synchronises those events, sums them and resets.
 * Not thread-safe while enabled. */
hq_status hq_profile_enable(hq_plan plan, int32_t enable);
hq_status hq_profile_read(hq_plan plan, hq_profile_result* out);

/* Process-wide count of kernel launches per class (HQ_K_*) since the library
 * was loaded, over every plan (always on; host-side counters only). */
void hq_launch_counts(int64_t out[HQ_K_CLASSES]);

#ifdef __cplusplus
}
#endif
#endif /* HQ_H */
