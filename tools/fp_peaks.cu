// FP-pipe peak microbenchmarks (measurement tooling for the roofline
// denominators; MEASURED_PEAKS.json only carries HBM and bf16 tensor peaks).
// Each thread runs 8 independent FMA chains; the grid fills every SM many
// times over. Returned values are FMA instructions per second (x2 = flop/s).
#include <cuda_runtime.h>

#include <cstdint>

template <class T>
__global__ void fma_chains(T* out, int iters, T a, T b) {
  T x0 = T(threadIdx.x), x1 = x0 + T(1), x2 = x0 + T(2), x3 = x0 + T(3);
  T x4 = x0 + T(4), x5 = x0 + T(5), x6 = x0 + T(6), x7 = x0 + T(7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == T(-12345.678)) out[threadIdx.x] = s;  // keep the work alive
}

template <class T>
static double run(int device, int iters) {
  cudaSetDevice(device);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  T* out = nullptr;
  cudaMalloc(&out, 1024 * sizeof(T));
  const int blocks = prop.multiProcessorCount * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_chains<T><<<blocks, threads>>>(out, 8, T(0.999), T(0.001));  // warm-up
  cudaEventRecord(e0);
  fma_chains<T><<<blocks, threads>>>(out, iters, T(0.999), T(0.001));
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double fmas = double(blocks) * threads * iters * 16 * 8;
  return fmas / (ms * 1e-3);
}

extern "C" double sfp_dfma_per_s(int device, int iters) { return run<double>(device, iters); }
extern "C" double sfp_ffma_per_s(int device, int iters) { return run<float>(device, iters); }
