// SHOT_SAMPLING on the device.
//
// Restates measure_shots (pkg/src/hyqnet/qsim.py:222-248) for a batch of final
// states: marginal Born probabilities over the measured qubits (outcome bit i
// = measured[i], qsim.py:194-211), their cumulative sum (sequential, as
// np.cumsum), and per shot s one uniform from Philox4x64-10 keyed
// [seed, s] (np.random.Philox(key=[seed, s]).random(): counter word 0 bumped to
// 1 before the first block, u = (word0 >> 11) * 2^-53) mapped by
// searchsorted(cum, u, side="right") clamped to the last outcome.
// Counts are integer atomics, so results are deterministic.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "hq_internal.h"

namespace hq {

__device__ __forceinline__ double philox_uniform(uint64_t seed, uint64_t shot) {
  uint64_t c0 = 1, c1 = 0, c2 = 0, c3 = 0, k0 = seed, k1 = shot;
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return (double)(c0 >> 11) * (1.0 / 9007199254740992.0);
}

struct SampleArgs {
  const double* state;   // [rows, 2^n, 2]
  int64_t rows;
  int32_t n, m;
  int32_t measured[34];
  int32_t unmeasured[34];
  int32_t chunk_bits;    // unmeasured index space split into 2^chunk_bits chunks
  double* part;          // [rows, 2^m, chunks]
  double* cum;           // [rows, 2^m]
  int64_t shots;
  uint64_t seed;
  unsigned long long* counts;  // [rows, 2^m] or null
  long long* sum;              // [rows] Σ outcome
};

// partial marginals: thread (row, outcome j, chunk c) sums its chunk in index order
__global__ void k_marginal_part(SampleArgs a) {
  const int64_t nout = 1ll << a.m;
  const int64_t nch = 1ll << a.chunk_bits;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.rows * nout * nch) return;
  const int64_t row = i / (nout * nch);
  const int64_t rem = i - row * nout * nch;
  const int64_t j = rem / nch, c = rem - j * nch;
  const int nu = a.n - a.m;
  const int per = nu - a.chunk_bits;
  uint64_t basej = 0;
  for (int k = 0; k < a.m; ++k) basej |= (uint64_t)((j >> k) & 1) << a.measured[k];
  const double* st = a.state + row * ((int64_t)2 << a.n);
  double s = 0.0;
  for (int64_t u = 0; u < (1ll << per); ++u) {
    const uint64_t w = ((uint64_t)c << per) | (uint64_t)u;   // unmeasured bits, chunk-major
    uint64_t idx = basej;
    for (int k = 0; k < nu; ++k) idx |= ((w >> k) & 1ull) << a.unmeasured[k];
    const double re = st[2 * idx], im = st[2 * idx + 1];
    s += re * re + im * im;
  }
  a.part[(row * nout + j) * nch + c] = s;
}

// per row: fold chunks in order, then sequential cumulative sum
__global__ void k_cumsum(SampleArgs a) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= a.rows) return;
  const int64_t nout = 1ll << a.m, nch = 1ll << a.chunk_bits;
  double acc = 0.0;
  for (int64_t j = 0; j < nout; ++j) {
    double p = 0.0;
    for (int64_t c = 0; c < nch; ++c) p += a.part[(row * nout + j) * nch + c];
    acc += p;
    a.cum[row * nout + j] = acc;
  }
}

__global__ void k_shots(SampleArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.rows * a.shots) return;
  const int64_t row = i / a.shots, s = i - row * a.shots;
  const int64_t nout = 1ll << a.m;
  const double u = philox_uniform(a.seed, (uint64_t)s);
  const double* cum = a.cum + row * nout;
  int64_t lo = 0, hi = nout;  // first index with cum[idx] > u
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cum[mid] > u) hi = mid; else lo = mid + 1;
  }
  const int64_t idx = lo < nout ? lo : nout - 1;
  if (a.counts) atomicAdd(a.counts + row * nout + idx, 1ull);
  atomicAdd(reinterpret_cast<unsigned long long*>(a.sum + row), (unsigned long long)idx);
}

// E = Σ outcome values / shots (qnn.py:27-32: exact integer sum, one division)
__global__ void k_expect(const long long* sum, int64_t rows, int64_t shots, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) out[i] = (double)sum[i] / (double)shots;
}

__global__ void k_uniforms(uint64_t seed, int64_t shot0, int64_t count, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = philox_uniform(seed, (uint64_t)(shot0 + i));
}

}  // namespace hq

namespace {
int chunk_bits_for(int64_t rows, int n, int m) {
  int cb = 0;
  while ((rows << (m + cb)) < 65536 && cb < n - m) ++cb;
  return cb;
}
}  // namespace

extern "C" size_t hq_sample_workspace_bytes(int64_t rows, int32_t n_qubits, int32_t n_measured) {
  if (rows <= 0 || n_measured < 1 || n_measured > n_qubits) return 256;
  const int cb = chunk_bits_for(rows, n_qubits, n_measured);
  const size_t nout = (size_t)1 << n_measured;
  return (size_t)rows * nout * (((size_t)1 << cb) + 1) * 8 + (size_t)rows * 8 + 1024;
}

extern "C" hq_status hq_sample(const double* state, int64_t rows, int32_t n_qubits, const int32_t* measured,
                               int32_t n_measured, int64_t shots, uint64_t seed, uint64_t* counts,
                               double* expectation, void* ws, size_t ws_bytes, void* stream) {
  if (rows <= 0) return HQ_OK;
  if (n_qubits < 1 || n_qubits > 34 || n_measured < 1 || n_measured > n_qubits || !measured)
    return hq::fail_status(HQ_E_CIRCUIT, "hq_sample: need 1 <= n_measured <= n_qubits <= 34 and a measured list");
  if (shots < 1) return hq::fail_status(HQ_E_CONFIG, "hq_sample: shots must be >= 1");
  if (ws_bytes < hq_sample_workspace_bytes(rows, n_qubits, n_measured))
    return hq::fail_status(HQ_E_CONFIG, "hq_sample: workspace too small");
  hq::SampleArgs a{};
  a.state = state;
  a.rows = rows;
  a.n = n_qubits;
  a.m = n_measured;
  uint64_t mask = 0;
  for (int k = 0; k < n_measured; ++k) {
    if (measured[k] < 0 || measured[k] >= n_qubits || (mask >> measured[k] & 1))
      return hq::fail_status(HQ_E_CIRCUIT, "hq_sample: measured qubit out of range or repeated");
    mask |= 1ull << measured[k];
    a.measured[k] = measured[k];
  }
  int u = 0;
  for (int q = 0; q < n_qubits; ++q)
    if (!(mask >> q & 1)) a.unmeasured[u++] = q;
  a.chunk_bits = chunk_bits_for(rows, n_qubits, n_measured);
  const size_t nout = (size_t)1 << n_measured;
  char* w = static_cast<char*>(ws);
  a.part = reinterpret_cast<double*>(w);
  a.cum = a.part + (size_t)rows * nout * ((size_t)1 << a.chunk_bits);
  long long* sum = reinterpret_cast<long long*>(a.cum + (size_t)rows * nout);
  a.sum = sum;
  a.shots = shots;
  a.seed = seed;
  a.counts = reinterpret_cast<unsigned long long*>(counts);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(sum, 0, (size_t)rows * 8, st);
  if (counts) cudaMemsetAsync(counts, 0, (size_t)rows * nout * 8, st);
  const int64_t t1 = (int64_t)rows * nout << a.chunk_bits;
  hq::k_marginal_part<<<(unsigned)((t1 + 255) / 256), 256, 0, st>>>(a);
  hq::k_cumsum<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(a);
  const int64_t t3 = rows * shots;
  hq::k_shots<<<(unsigned)((t3 + 255) / 256), 256, 0, st>>>(a);
  if (expectation) hq::k_expect<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(sum, rows, shots, expectation);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HQ_OK : hq::fail_status(HQ_E_CUDA, std::string("hq_sample launch: ") + cudaGetErrorString(e));
}

extern "C" hq_status hq_shot_uniforms(uint64_t seed, int64_t shot0, int64_t count, double* out, void* stream) {
  if (count <= 0) return HQ_OK;
  if (!out) return hq::fail_status(HQ_E_CONFIG, "hq_shot_uniforms: null output");
  hq::k_uniforms<<<(unsigned)((count + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, shot0, count,
                                                                                                  out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HQ_OK
                          : hq::fail_status(HQ_E_CUDA, std::string("hq_shot_uniforms launch: ") + cudaGetErrorString(e));
}

// ---- marginal Born probabilities on the device (qsim.py:194-211) ----------
namespace hq {
__global__ void k_marginal_fold(const double* part, int64_t rows, int32_t m, int32_t chunk_bits, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nout = 1ll << m, nch = 1ll << chunk_bits;
  if (i >= rows * nout) return;
  double p = 0.0;
  for (int64_t c = 0; c < nch; ++c) p += part[i * nch + c];   // fixed chunk order
  out[i] = p;
}
}  // namespace hq

extern "C" size_t hq_marginal_workspace_bytes(int64_t rows, int32_t n_qubits, int32_t n_measured) {
  if (rows <= 0 || n_measured < 1 || n_measured > n_qubits) return 256;
  const int cb = chunk_bits_for(rows, n_qubits, n_measured);
  return (size_t)rows * ((size_t)1 << n_measured) * ((size_t)1 << cb) * 8 + 256;
}

extern "C" hq_status hq_marginal(const double* state, int64_t rows, int32_t n_qubits, const int32_t* measured,
                                 int32_t n_measured, double* probs, void* ws, size_t ws_bytes, void* stream) {
  if (rows <= 0) return HQ_OK;
  if (!state || !probs) return hq::fail_status(HQ_E_CONFIG, "hq_marginal: null state / output");
  if (n_qubits < 1 || n_qubits > 34 || n_measured < 1 || n_measured > n_qubits || !measured)
    return hq::fail_status(HQ_E_CIRCUIT, "hq_marginal: need 1 <= n_measured <= n_qubits <= 34 and a measured list");
  if (!ws || ws_bytes < hq_marginal_workspace_bytes(rows, n_qubits, n_measured))
    return hq::fail_status(HQ_E_CONFIG, "hq_marginal: workspace too small");
  hq::SampleArgs a{};
  a.state = state;
  a.rows = rows;
  a.n = n_qubits;
  a.m = n_measured;
  uint64_t mask = 0;
  for (int k = 0; k < n_measured; ++k) {
    if (measured[k] < 0 || measured[k] >= n_qubits || (mask >> measured[k] & 1))
      return hq::fail_status(HQ_E_CIRCUIT, "hq_marginal: measured qubit out of range or repeated");
    mask |= 1ull << measured[k];
    a.measured[k] = measured[k];
  }
  int u = 0;
  for (int q = 0; q < n_qubits; ++q)
    if (!(mask >> q & 1)) a.unmeasured[u++] = q;
  a.chunk_bits = chunk_bits_for(rows, n_qubits, n_measured);
  a.part = static_cast<double*>(ws);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t t1 = (int64_t)rows << (n_measured + a.chunk_bits);
  hq::count_launch(HQ_K_OTHER);
  hq::k_marginal_part<<<(unsigned)((t1 + 255) / 256), 256, 0, st>>>(a);
  const int64_t t2 = (int64_t)rows << n_measured;
  hq::count_launch(HQ_K_OTHER);
  hq::k_marginal_fold<<<(unsigned)((t2 + 255) / 256), 256, 0, st>>>(a.part, rows, n_measured, a.chunk_bits, probs);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HQ_OK : hq::fail_status(HQ_E_CUDA, std::string("hq_marginal launch: ") + cudaGetErrorString(e));
}
