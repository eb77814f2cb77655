#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// Pattern microbenchmark: per step 2 bits x 16 slots x (LOP3 + 2 DFMA), all in registers.
template <int V, int MODE>
__global__ void __launch_bounds__(256, 2) k(const uint32_t* __restrict__ vin, double* out, int iters, uint32_t seed) {
  uint32_t vv[V];
  double gh[V], gl[V];
  for (int i = 0; i < V; ++i) { vv[i] = vin[threadIdx.x + 32 * i] ^ (seed * (i + 1)); gh[i] = 0; gl[i] = 0; }
  double L1x = 1e-300 * (threadIdx.x + 1), L1y = 2e-300, L2x = 3e-300, L2y = 4e-300;
  uint32_t m = 1u << (threadIdx.x & 7);
  for (int it = 0; it < iters; ++it) {
    const uint32_t m1 = m, m2 = m << 8;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      double f1, f2;
      if (MODE == 0) { f1 = __hiloint2double(vv[i] & m1, 0); f2 = __hiloint2double(vv[i] & m2, 0); }
      else { f1 = __hiloint2double((vv[i] & m1) ? 0x3ff00000 : 0, 0); f2 = __hiloint2double((vv[i] & m2) ? 0x3ff00000 : 0, 0); }
      gh[i] = fma(L1x, f1, gh[i]); gl[i] = fma(L1y, f1, gl[i]);
      gh[i] = fma(L2x, f2, gh[i]); gl[i] = fma(L2y, f2, gl[i]);
    }
    m = (m << 1) | (m >> 31);
  }
  double s = 0;
  for (int i = 0; i < V; ++i) s += gh[i] + gl[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int V, int MODE>
void run(const char* name, uint32_t* vin, double* out) {
  const int iters = 2000, blocks = 148 * 2 * 4;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<V, MODE><<<blocks, 256>>>(vin, out, iters, 1);
  cudaEventRecord(a);
  k<V, MODE><<<blocks, 256>>>(vin, out, iters, 2);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double dfma = 4.0 * V * iters * (double)blocks * 256;
  printf("%s: %.3f ms, %.2f e12 DFMA/s\n", name, ms, dfma / ms / 1e9);
}
int main() {
  uint32_t* vin; double* out;
  cudaMalloc(&vin, 4096 * 4); cudaMemset(vin, 0x5a, 4096 * 4);
  cudaMalloc(&out, 148 * 2 * 4 * 256 * 8);
  run<16, 0>("lop3-factor V16", vin, out);
  run<16, 1>("sel-factor  V16", vin, out);
  run<8, 0>("lop3-factor V8", vin, out);
  return 0;
}
