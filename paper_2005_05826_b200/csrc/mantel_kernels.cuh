// Mantel permutation test on device (replaces mantel,
// validate.cpp:111-159).
//
// x, y are the condensed upper triangles of two n x n distance matrices.
// r = sum (x - mx)(y - my) / sqrt(sxx syy); permutation p relabels the
// samples of the second matrix with the reference's stream (mt19937_64 +
// std::shuffle seeded from splitmix64(seed ^ splitmix64(p + 1)), generated on
// the host by the same C++ library code), and only the cross term changes:
//   dot_p = sum_{i<j} (X[i][j] - mx) * (Y[pi_i][pi_j] - my).
// Each term is formed exactly as the reference forms it (xc = x - mx rounded
// first, then xc * (yv - my)); only the summation order differs, so r and
// dot_p agree to ~1e-15 relative and the exceed counts agree except at exact
// ties. Sums are deterministic: fixed per-block partials, reduced in a fixed
// order.
//
// Layout: X, Y row-major n x n fp64 in HBM (C3: 5 GB each). The permutation
// kernel runs one CTA per (permutation, row pair {i, n-1-i}) with the
// permutations of a batch fastest-varying, so the CTAs that read X row i run
// together and share it through L2; Y rows are gathered per permutation
// (HBM-bound: ~n^2 x 8 B of Y per permutation).
#pragma once

#include <cstdint>

namespace sf {

constexpr int kMantelThreads = 256;

__device__ __forceinline__ double block_sum_256(double v, double* sh) {
  // fixed-shape tree: deterministic for a given blockDim
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (kMantelThreads >> 5); ++w) t += sh[w];
  return t;
}

// Row-paired partial sums over the condensed triangle. mode 0: sum x, sum y
// (and the first asymmetric pair of each matrix, row-major, like
// condensed_upper's check, validate.cpp:87-91); mode 1: sxx, syy about the
// means into part, and the sxy partials into pxy (reduced like the
// permutations' cross terms, so the identity relabeling reproduces r's
// numerator bit for bit, as in the reference).
__global__ void __launch_bounds__(kMantelThreads) mt_stats_kernel(
    const double* __restrict__ X, const double* __restrict__ Y, int32_t n, int32_t mode, double mx,
    double my, double* __restrict__ part, double* __restrict__ pxy,
    unsigned long long* __restrict__ first_asym) {
  __shared__ double sh[kMantelThreads / 32];
  const int rp = blockIdx.x;  // row pair index
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int side = 0; side < 2; ++side) {
    const int i = side == 0 ? rp : n - 1 - rp;
    if (side == 1 && i == rp) break;  // middle row of odd n
    if (i >= n - 1) continue;
    const double* xr = X + static_cast<int64_t>(i) * n;
    const double* yr = Y + static_cast<int64_t>(i) * n;
    for (int j = i + 1 + threadIdx.x; j < n; j += kMantelThreads) {
      const double xv = xr[j], yv = yr[j];
      if (mode == 0) {
        a0 += xv;
        a1 += yv;
        const unsigned long long at = static_cast<unsigned long long>(i) * static_cast<unsigned long long>(n) + j;
        if (fabs(xv - X[static_cast<int64_t>(j) * n + i]) > 1e-12) atomicMin(first_asym, at);
        if (fabs(yv - Y[static_cast<int64_t>(j) * n + i]) > 1e-12) atomicMin(first_asym + 1, at);
      } else {
        const double xc = xv - mx, yc = yv - my;
        a0 += xc * xc;
        a1 += yc * yc;
        a2 += xc * yc;
      }
    }
  }
  const double s0 = block_sum_256(a0, sh);
  const double s1 = block_sum_256(a1, sh);
  const double s2 = mode ? block_sum_256(a2, sh) : 0.0;
  if (threadIdx.x == 0) {
    part[2 * static_cast<int64_t>(rp)] = s0;
    part[2 * static_cast<int64_t>(rp) + 1] = s1;
    if (mode) pxy[rp] = s2;
  }
}

// Cross terms of a batch of permutations: block (p, rp) -> part[p][rp].
__global__ void __launch_bounds__(kMantelThreads) mt_perm_kernel(
    const double* __restrict__ X, const double* __restrict__ Y, int32_t n, double mx, double my,
    const int32_t* __restrict__ perms, int32_t nrp, double* __restrict__ part) {
  __shared__ double sh[kMantelThreads / 32];
  const int p = blockIdx.x;
  const int rp = blockIdx.y;
  const int32_t* pi = perms + static_cast<int64_t>(p) * n;
  double acc = 0.0;
  for (int side = 0; side < 2; ++side) {
    const int i = side == 0 ? rp : n - 1 - rp;
    if (side == 1 && i == rp) break;
    if (i >= n - 1) continue;
    const double* xr = X + static_cast<int64_t>(i) * n;
    const double* yr = Y + static_cast<int64_t>(__ldg(pi + i)) * n;
    for (int j = i + 1 + threadIdx.x; j < n; j += kMantelThreads) {
      const double xc = __ldg(xr + j) - mx;  // the reference's xc[at]
      acc += xc * (__ldg(yr + __ldg(pi + j)) - my);
    }
  }
  const double s = block_sum_256(acc, sh);
  if (threadIdx.x == 0) part[static_cast<int64_t>(p) * nrp + rp] = s;
}

// dot[p] = sum over rp of part[p][rp], one block per permutation.
__global__ void __launch_bounds__(kMantelThreads) mt_reduce_kernel(const double* __restrict__ part,
                                                                   int32_t nrp, double* __restrict__ dot) {
  __shared__ double sh[kMantelThreads / 32];
  const double* row = part + static_cast<int64_t>(blockIdx.x) * nrp;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nrp; i += kMantelThreads) acc += row[i];
  const double s = block_sum_256(acc, sh);
  if (threadIdx.x == 0) dot[blockIdx.x] = s;
}

}  // namespace sf
