// FP64 pipe throughput vs resident warps for the pass kernels' math pattern:
// 16 independent shear chains per thread (3 dependent DFMA each, like RY on
// 4 amplitude pairs of psi and lambda), looped.  Launches 148 x k CTAs of 256
// threads (k CTAs per SM) and prints TFLOP/s, to see whether one tile group
// of 8 warps can keep the FP64 pipe busy on its own (ping-pong kernels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_occ tools/dfma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256, 1) k_shear(double* out, int iters, double t, double u) {
  double x[CHAINS], y[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { x[c] = threadIdx.x * 1e-3 + c; y[c] = blockIdx.x * 1e-3 - c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      x[c] = fma(t, y[c], x[c]);
      y[c] = fma(u, x[c], y[c]);
      x[c] = fma(t, y[c], x[c]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c] + y[c];
  if (s == 1.2345) out[0] = s;   // keep the work
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int per_sm = 1; per_sm <= 2; ++per_sm) {
    for (int w = 0; w < 2; ++w) {
      const int grid = 148 * per_sm;
      k_shear<16><<<grid, 256>>>(d, 16, 0.3, -0.2);
      cudaEventRecord(a);
      k_shear<16><<<grid, 256>>>(d, iters, 0.3, -0.2);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double flops = 2.0 * 3 * 16 * (double)iters * 256 * grid;
      if (w) std::printf("{\"ctas_per_sm\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", per_sm, 8 * per_sm,
                         flops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
