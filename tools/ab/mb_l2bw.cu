#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const int4* __restrict__ p, size_t n16, int passes, int* out) {
  int acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int ps = 0; ps < passes; ++ps)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x + (size_t)ps * 977; i < n16 + (size_t)ps * 977; i += stride) {
      const int4 v = __ldcg(p + (i % n16));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345) out[0] = acc;
}
int main() {
  for (size_t mb : {16, 48, 96}) {
    size_t bytes = mb << 20; int4* p; int* o;
    cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes); cudaMalloc(&o, 4);
    const int passes = 50;
    rd<<<148 * 8, 512>>>(p, bytes / 16, 2, o);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    rd<<<148 * 8, 512>>>(p, bytes / 16, passes, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("L2 read (ld.cg, %zu MB buffer): %.1f GB/s\n", mb, (double)bytes * passes / ms / 1e6);
    cudaFree(p); cudaFree(o);
  }
}
