// K1: postorder embedding on device.
//
// Replaces Embedder::next_batch (embed.cpp:42-82) + relative_abundance /
// presence (table.cpp:208-222). A postorder row range (a "chunk") is built
// in three steps, all bit-identical to the reference's row values:
//   1. leaf rows: scatter the feature's CSR entries, c / total[s] (weighted)
//      or presence bits (unweighted);
//   2. internal rows, one launch per tree height: row = ((0 + c1) + c2) + ...
//      over children in postorder (the reference's pending fold, embed.cpp:
//      71-79) — sum for weighted, OR for unweighted presence bits;
//   3. rows whose parent lies in a later chunk are copied to pending slots.
// Row layouts: weighted rows are fp64 (fp32 kernels round at staging, once,
// matching cast_batch, embed.hpp:71-84); unweighted rows are 32-bit words,
// bit b of word w = sample 32w+b.
#pragma once

#include <cstdint>

namespace sf {

// One warp per leaf row: entries of feature leaf_feat[i] scattered into row
// leaf_rows[i] of the chunk buffer. (table.cpp:208-214)
__global__ void embed_leaf_values(double* __restrict__ buf, int64_t stride,
                                  const int32_t* __restrict__ leaf_rows,
                                  const int32_t* __restrict__ leaf_feat, int32_t n_leaf,
                                  const int64_t* __restrict__ feat_ptr,
                                  const int32_t* __restrict__ sidx,
                                  const double* __restrict__ counts,
                                  const double* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_leaf; i += nwarps) {
    double* row = buf + static_cast<int64_t>(leaf_rows[i]) * stride;
    const int f = leaf_feat[i];
    for (int64_t e = feat_ptr[f] + lane; e < feat_ptr[f + 1]; e += 32) {
      const int s = sidx[e];
      row[s] = counts[e] / totals[s];
    }
  }
}

// Unweighted leaves: presence bits (table.cpp:216-222: c > 0 -> 1).
__global__ void embed_leaf_bits(uint32_t* __restrict__ buf, int64_t stride,
                                const int32_t* __restrict__ leaf_rows,
                                const int32_t* __restrict__ leaf_feat, int32_t n_leaf,
                                const int64_t* __restrict__ feat_ptr,
                                const int32_t* __restrict__ sidx,
                                const double* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_leaf; i += nwarps) {
    uint32_t* row = buf + static_cast<int64_t>(leaf_rows[i]) * stride;
    const int f = leaf_feat[i];
    for (int64_t e = feat_ptr[f] + lane; e < feat_ptr[f + 1]; e += 32) {
      if (counts[e] > 0.0) {
        const int s = sidx[e];
        atomicOr(row + (s >> 5), 1u << (s & 31));
      }
    }
  }
}

// Child location code: >= 0 is a row of the current chunk buffer, < 0 is
// pending slot (-1 - code).
template <class T>
__device__ __forceinline__ const T* child_row(const T* buf, int64_t stride, const T* pend,
                                              int32_t code) {
  return code >= 0 ? buf + static_cast<int64_t>(code) * stride
                   : pend + static_cast<int64_t>(-1 - code) * stride;
}

// Internal rows of one height: grid.x over columns, grid.y (strided) over rows.
__global__ void embed_level_values(double* __restrict__ buf, int64_t stride,
                                   const double* __restrict__ pend,
                                   const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ cptr,
                                   const int32_t* __restrict__ codes, int32_t n_rows,
                                   int32_t n_cols) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n_cols) return;
  for (int i = blockIdx.y; i < n_rows; i += gridDim.y) {
    double acc = 0.0;  // pending_ starts at RowVectorXd::Zero (embed.cpp:75-76)
    for (int c = cptr[i]; c < cptr[i + 1]; ++c) acc += child_row(buf, stride, pend, codes[c])[col];
    buf[static_cast<int64_t>(rows[i]) * stride + col] = acc;
  }
}

__global__ void embed_level_bits(uint32_t* __restrict__ buf, int64_t stride,
                                 const uint32_t* __restrict__ pend,
                                 const int32_t* __restrict__ rows,
                                 const int32_t* __restrict__ cptr,
                                 const int32_t* __restrict__ codes, int32_t n_rows,
                                 int32_t n_cols) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n_cols) return;
  for (int i = blockIdx.y; i < n_rows; i += gridDim.y) {
    uint32_t acc = 0u;  // cwiseMax of 0/1 rows is OR (embed.cpp:78)
    for (int c = cptr[i]; c < cptr[i + 1]; ++c) acc |= child_row(buf, stride, pend, codes[c])[col];
    buf[static_cast<int64_t>(rows[i]) * stride + col] = acc;
  }
}

// Rows of this chunk whose parent is emitted in a later chunk move to
// pending slots (the reference keeps them in its pending_ map).
template <class T>
__global__ void embed_carry(const T* __restrict__ buf, T* __restrict__ pend, int64_t stride,
                            const int32_t* __restrict__ src_rows,
                            const int32_t* __restrict__ dst_slots, int32_t n, int32_t n_cols) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n_cols) return;
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    pend[static_cast<int64_t>(dst_slots[i]) * stride + col] =
        buf[static_cast<int64_t>(src_rows[i]) * stride + col];
}

}  // namespace sf
