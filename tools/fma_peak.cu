// FP32 / packed-FP32x2 / FP64 FMA throughput on this GPU (SURVEY.md §8(d):
// "measure the FP32/FP64 peaks with an FMA microbenchmark before quoting
// compute fractions").  Independent FMA chains per thread, grid = 4 x SMs x
// 1024 threads, CUDA-event timed after a warm-up.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fma_peak.cu -o /tmp/fma_peak && /tmp/fma_peak
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[kChains];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  const unsigned long long A = *reinterpret_cast<unsigned long long*>(&av);
  const unsigned long long B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float2 v = make_float2(threadIdx.x * 1e-7f + c, c * 0.5f);
    x[c] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float2 v = *reinterpret_cast<float2*>(&x[c]);
    s += v.x + v.y;
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_dfma(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7 + c;
  for (int i = 0; i < kIters / 8; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
static double time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int grid = 4 * prop.multiProcessorCount, block = 1024;
  float* out;
  cudaMalloc(&out, 16);
  const double threads = (double)grid * block;
  const double t1 = time_ms([&] { k_ffma<<<grid, block>>>(out, 0.999f, 1e-3f); });
  const double t2 = time_ms([&] { k_ffma2<<<grid, block>>>(out, 0.999f, 1e-3f); });
  const double t3 = time_ms([&] { k_dfma<<<grid, block>>>((double*)out, 0.999, 1e-3); });
  const double f1 = threads * kIters * kChains * 2 / (t1 * 1e-3) / 1e12;
  const double f2 = threads * kIters * kChains * 4 / (t2 * 1e-3) / 1e12;
  const double f3 = threads * (kIters / 8) * kChains * 2 / (t3 * 1e-3) / 1e12;
  cudaError_t err = cudaGetLastError();
  std::printf("{\"device\": \"%s\", \"sms\": %d, \"fp32_ffma_tflops\": %.2f, \"fp32_ffma2_tflops\": %.2f, "
              "\"fp64_dfma_tflops\": %.2f, \"error\": \"%s\"}\n",
              prop.name, prop.multiProcessorCount, f1, f2, f3, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
