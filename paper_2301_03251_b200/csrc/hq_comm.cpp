// Multi-GPU entry points of the C ABI: an NCCL communicator
// owned by the library and the two collectives the data-parallel and
// amplitude-sharded paths need, plus the fused data-parallel step.
//
// NCCL is loaded at run time (dlopen, like NVRTC): the instance torch already
// loaded is reused when present (RTLD_NOLOAD), else libnccl.so.2 from the
// system.  One process per GPU; the ncclUniqueId travels between ranks through
// whatever the host uses (torch.distributed broadcast in dist.py).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "hq_internal.h"
#include "hq_launch.h"

namespace {

// the subset of nccl.h this file uses (ABI-stable since NCCL 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclUint8 = 1, kNcclFloat64 = 8 };
enum { kNcclSum = 0 };

struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl load_nccl() {
  Nccl n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) { n.why = "libnccl.so.2 not found"; return n; }
  n.get_unique_id = (decltype(n.get_unique_id))dlsym(h, "ncclGetUniqueId");
  n.comm_init_rank = (decltype(n.comm_init_rank))dlsym(h, "ncclCommInitRank");
  n.comm_destroy = (decltype(n.comm_destroy))dlsym(h, "ncclCommDestroy");
  n.all_reduce = (decltype(n.all_reduce))dlsym(h, "ncclAllReduce");
  n.send = (decltype(n.send))dlsym(h, "ncclSend");
  n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
  n.group_start = (decltype(n.group_start))dlsym(h, "ncclGroupStart");
  n.group_end = (decltype(n.group_end))dlsym(h, "ncclGroupEnd");
  n.error_string = (decltype(n.error_string))dlsym(h, "ncclGetErrorString");
  n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce && n.send && n.recv &&
         n.group_start && n.group_end && n.error_string;
  if (!n.ok) n.why = "libnccl lacks the expected symbols";
  return n;
}

Nccl& nccl() {
  static Nccl n = load_nccl();
  return n;
}

hq_status nccl_fail(ncclResult_t r, const char* what) {
  return hq::fail_status(HQ_E_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct hq_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

extern "C" size_t hq_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" hq_status hq_comm_unique_id(void* id_out) {
  if (!id_out) return hq::fail_status(HQ_E_CONFIG, "hq_comm_unique_id: null output");
  Nccl& n = nccl();
  if (!n.ok) return hq::fail_status(HQ_E_CONFIG, "NCCL unavailable: " + n.why);
  ncclUniqueId id;
  const ncclResult_t r = n.get_unique_id(&id);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof id);
  return HQ_OK;
}

extern "C" hq_status hq_comm_init(const void* id, int32_t rank, int32_t world, hq_comm* out) {
  if (!id || !out) return hq::fail_status(HQ_E_CONFIG, "hq_comm_init: null id / output");
  if (world < 1 || rank < 0 || rank >= world) return hq::fail_status(HQ_E_CONFIG, "hq_comm_init: bad rank / world");
  Nccl& n = nccl();
  if (!n.ok) return hq::fail_status(HQ_E_CONFIG, "NCCL unavailable: " + n.why);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  auto c = new hq_comm_s();
  c->rank = rank;
  c->world = world;
  const ncclResult_t r = n.comm_init_rank(&c->comm, world, uid, rank);
  if (r != 0) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return HQ_OK;
}

extern "C" void hq_comm_destroy(hq_comm c) {
  if (!c) return;
  if (c->comm) nccl().comm_destroy(c->comm);
  delete c;
}

extern "C" hq_status hq_comm_allreduce_f64(hq_comm c, double* buf, int64_t count, void* stream) {
  if (!c) return hq::fail_status(HQ_E_CONFIG, "null communicator");
  if (count <= 0) return HQ_OK;
  if (!buf) return hq::fail_status(HQ_E_CONFIG, "hq_comm_allreduce_f64: null buffer");
  const ncclResult_t r = nccl().all_reduce(buf, buf, (size_t)count, kNcclFloat64, kNcclSum, c->comm,
                                           static_cast<cudaStream_t>(stream));
  return r == 0 ? HQ_OK : nccl_fail(r, "ncclAllReduce");
}

// Contiguous equal chunks: chunk j of `send` goes to rank j and the chunk from
// rank j lands at chunk j of `recv` (the global<->local qubit exchange of
// shard.py: all rank bits <-> the top local bits).  Grouped send/recv pairs.
extern "C" hq_status hq_comm_alltoall(hq_comm c, const void* send, void* recv, int64_t bytes_per_rank,
                                      void* stream) {
  if (!c) return hq::fail_status(HQ_E_CONFIG, "null communicator");
  if (bytes_per_rank <= 0) return HQ_OK;
  if (!send || !recv || send == recv) return hq::fail_status(HQ_E_CONFIG, "hq_comm_alltoall: distinct buffers needed");
  Nccl& n = nccl();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(send);
  char* d = static_cast<char*>(recv);
  ncclResult_t r = n.group_start();
  if (r != 0) return nccl_fail(r, "ncclGroupStart");
  for (int p = 0; p < c->world; ++p) {
    r = n.send(s + (size_t)p * bytes_per_rank, (size_t)bytes_per_rank, kNcclUint8, p, c->comm, st);
    if (r == 0) r = n.recv(d + (size_t)p * bytes_per_rank, (size_t)bytes_per_rank, kNcclUint8, p, c->comm, st);
    if (r != 0) {
      n.group_end();
      return nccl_fail(r, "ncclSend/ncclRecv");
    }
  }
  r = n.group_end();
  return r == 0 ? HQ_OK : nccl_fail(r, "ncclGroupEnd");
}

// One data-parallel step of the sample-sharded layer:
// this rank's forward + jacobian rows (hq_forward(HQ_WANT_JAC)), the upstream
// vector-jacobian product (hq_vjp: grad_x rows, grad_theta summed in sample
// order) and ONE all-reduce of grad_theta over the communicator.  Replaces the
// serial batch loop and the sequential gradient sum of qnn.py:131,147-152.
extern "C" hq_status hq_backward_dp(hq_plan plan, const double* x, int64_t ldx, const double* theta, int64_t batch,
                                    const double* upstream, double* out, double* jac, double* grad_x,
                                    double* grad_theta, hq_comm c, void* ws, size_t ws_bytes, void* stream) {
  if (!grad_theta && plan && plan->n_params > 0)
    return hq::fail_status(HQ_E_CONFIG, "hq_backward_dp: null grad_theta");
  hq_status s = hq_forward(plan, x, ldx, theta, batch, HQ_WANT_JAC, out, jac, ws, ws_bytes, stream);
  if (s != HQ_OK) return s;
  if (batch > 0) {
    s = hq_vjp(plan, jac, upstream, batch, grad_x, grad_theta, stream);
    if (s != HQ_OK) return s;
  } else if (grad_theta && plan->n_params > 0) {
    cudaMemsetAsync(grad_theta, 0, (size_t)plan->n_params * 8, static_cast<cudaStream_t>(stream));
  }
  if (c && c->world > 1 && plan->n_params > 0) return hq_comm_allreduce_f64(c, grad_theta, plan->n_params, stream);
  return HQ_OK;
}
