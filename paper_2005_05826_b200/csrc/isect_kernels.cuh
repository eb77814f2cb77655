// K2-UW (intersection form): the unweighted stripes from exact shared-length sums.
//
// update_entry<Unweighted> (kernels.hpp:55-66) summed over all rows gives, for
// a slot (k, l = (k+s+1) mod n) and presence sets S_e,
//   t = sum_{e: k in S_e or  l in S_e} L_e,
//   d = sum_{e: k in S_e xor l in S_e} L_e.
// The reference adds these in postorder in floating point. Here they are
// computed EXACTLY in fixed point (L_e -> round(L_e * 2^q), a 64-bit integer
// split into two 32-bit limbs that are summed without carries) and rounded to
// the output precision once, so the result is the correctly rounded exact sum;
// it agrees with the reference's sequential sum to within that sum's own
// rounding error (<= ~1e-14 relative at the EMP shape; the north-star gate is
// 1e-12). Because the sums are exact, the order of the rows no longer
// matters, and the union can be replaced by an intersection:
//
//   X_e  = S_e if |S_e| <= n/2 ("sparse" row), else the complement of S_e
//          ("dense" row: near-root rows are present in most samples);
//   x_k  = sum_{e: k in X_e} L_e,   p_k = sum_{sparse e: k in S_e} L_e,
//   C    = sum_{dense e} L_e,       G_kl = sum_{e: k in X_e and l in X_e} L_e,
//   t_kl = p_k + p_l + C - G_kl,    d_kl = x_k + x_l - 2 G_kl.
//
// (sparse rows: [k or l] = [k] + [l] - [k and l]; dense rows: [k or l] =
// 1 - [not k and not l]; and xor is invariant under complementing a row.)
// At the EMP shape a slot's union holds ~13,300 rows but its X-intersection
// only ~750, so the per-slot walk is ~18x shorter than the union walk of
// stripe_sparse_kernel, which stays as the bitwise-identical (exact) path.
//
// Layout (built on device from the node-packed presence bits NB[w][c], see
// sparse_kernels.cuh): NX[w][c] = NB[w][c] ^ dense_mask[w]; rows are grouped
// 1024 at a time (32 words). For group g and column c:
//   occ[g][c]   bit (31-i) set when word 32g+i of column c is nonzero;
//   base[g][c]  offset of the column's nonzero words in `packed` (group-major,
//               column-minor, so a window of consecutive columns is one
//               contiguous range);
//   limbs[row]  (hi, lo) 32-bit limbs of round(L_row * 2^q).
#pragma once

#include <cstdint>

namespace sf {

// ---- preparation --------------------------------------------------------

// One warp per row of the sample-packed presence rows: |S_e|, the dense-row
// mask (row 32w+r at bit 31-r of dmask[w]) and C = sum of dense-row limbs.
__global__ void isect_row_count_kernel(const uint32_t* __restrict__ rows, int64_t stride,
                                       int32_t E, int32_t n, const uint2* __restrict__ limbs,
                                       uint32_t* __restrict__ dmask,
                                       unsigned long long* __restrict__ cacc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < E; r += nwarps) {
    const uint32_t* row = rows + r * stride;
    int m = 0;
    for (int64_t i = lane; i < stride; i += 32) m += __popc(__ldg(row + i));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m += __shfl_xor_sync(0xffffffffu, m, off);
    if (lane == 0 && 2 * m > n) {
      atomicOr(dmask + (r >> 5), 0x80000000u >> (r & 31));
      const uint2 L = limbs[r];
      atomicAdd(cacc, static_cast<unsigned long long>(L.x));
      atomicAdd(cacc + 1, static_cast<unsigned long long>(L.y));
    }
  }
}

// One thread per (group, column): occupancy mask and nonzero-word count of
// the column's 32 X-words; for real columns (c < n) also the column sums
// x_c (all X rows) and p_c (sparse rows), limb by limb.
// colsum layout: [4][n] = x_hi, x_lo, p_hi, p_lo.
__global__ void isect_occ_kernel(const uint32_t* __restrict__ nb, int64_t n_ext, int32_t n,
                                 int32_t W, int32_t G, const uint32_t* __restrict__ dmask,
                                 const uint2* __restrict__ limbs, uint32_t* __restrict__ occ,
                                 uint32_t* __restrict__ cnt,
                                 unsigned long long* __restrict__ colsum) {
  const int64_t total = static_cast<int64_t>(G) * n_ext;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(idx / n_ext);
    const int64_t c = idx - static_cast<int64_t>(g) * n_ext;
    uint32_t o = 0u;
    int count = 0;
    unsigned long long xh = 0, xl = 0, ph = 0, pl = 0;
    for (int i = 0; i < 32; ++i) {
      const int w = 32 * g + i;
      if (w >= W) break;
      const uint32_t dm = __ldg(dmask + w);
      const uint32_t x = __ldg(nb + static_cast<int64_t>(w) * n_ext + c) ^ dm;
      if (x == 0u) continue;
      o |= 0x80000000u >> i;
      ++count;
      if (c < n) {
        uint32_t b = x;
        while (b) {
          const int r = __clz(b);
          const uint32_t m = 0x80000000u >> r;
          b ^= m;
          const uint2 L = __ldg(limbs + 32 * w + r);
          xh += L.x;
          xl += L.y;
          if (!(dm & m)) {
            ph += L.x;
            pl += L.y;
          }
        }
      }
    }
    occ[idx] = o;
    cnt[idx] = static_cast<uint32_t>(count);
    if (c < n && (xh | xl)) {
      atomicAdd(colsum + c, xh);
      atomicAdd(colsum + n + c, xl);
      if (ph | pl) {
        atomicAdd(colsum + 2 * static_cast<int64_t>(n) + c, ph);
        atomicAdd(colsum + 3 * static_cast<int64_t>(n) + c, pl);
      }
    }
  }
}

// One thread per (group, column): write the nonzero X-words, in word order,
// at packed[base[g][c] ...].
__global__ void isect_pack_kernel(const uint32_t* __restrict__ nb, int64_t n_ext, int32_t W,
                                  int32_t G, const uint32_t* __restrict__ dmask,
                                  const uint32_t* __restrict__ base,
                                  uint32_t* __restrict__ packed) {
  const int64_t total = static_cast<int64_t>(G) * n_ext;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(idx / n_ext);
    const int64_t c = idx - static_cast<int64_t>(g) * n_ext;
    uint32_t* out = packed + base[idx];
    for (int i = 0; i < 32; ++i) {
      const int w = 32 * g + i;
      if (w >= W) break;
      const uint32_t x = __ldg(nb + static_cast<int64_t>(w) * n_ext + c) ^ __ldg(dmask + w);
      if (x) *out++ = x;
    }
  }
}

// ---- the stripe kernel ----------------------------------------------------

struct IsectArgs {
  const uint32_t* occ;     // [G][n_ext]
  const uint32_t* base;    // [G*n_ext + 1]
  const uint32_t* packed;  // nonzero X-words
  const uint2* limbs;      // [G*1024] (hi, lo), zero past E
  const unsigned long long* colsum;  // [4][n]
  const unsigned long long* cacc;    // [2]
  int64_t n_ext;
  int32_t G;
  int32_t n;
  int32_t s_begin, s_end;
  int32_t scale;     // limbs hold round(L * 2^scale)
  int32_t finalize;  // write d/t (t == 0 -> 0) instead of d
  void* dist;        // (s_end - s_begin) x n
  void* tot;
  unsigned long long* exec_updates;
};

template <int RK, int RS, int NWK, int NWS>
struct IsectTile {
  static constexpr int NW = NWK * NWS;
  static constexpr int NT = 32 * NW;
  static constexpr int TK = NWK * RK;       // samples per CTA (u side)
  static constexpr int TS = NWS * 32 * RS;  // stripes per CTA
  static constexpr int VW = TK + TS;        // v columns staged
  static constexpr int OFF_L = 0;           // 1024 rows x (hi, lo)
  static constexpr int OFF_OU = OFF_L + 1024 * 8;
  static constexpr int OFF_OV = OFF_OU + TK * 4;
  static constexpr int OFF_FU = OFF_OV + VW * 4;
  static constexpr int OFF_FV = OFF_FU + TK * 4;
  static constexpr int OFF_PU = OFF_FV + VW * 4;
  static constexpr int OFF_PV = OFF_PU + 32 * TK * 4;
  static constexpr int BYTES = OFF_PV + 32 * VW * 4;
  static_assert(TK + VW <= NT, "one staging thread per column");
};

// Exact value v * 2^-scale (v >= 0, a 128-bit integer), correctly rounded.
__device__ __forceinline__ double fixed_to_double(__int128 v, int scale) {
  const unsigned __int128 u = static_cast<unsigned __int128>(v);
  const unsigned long long hi = static_cast<unsigned long long>(u >> 64);
  const unsigned long long lo = static_cast<unsigned long long>(u);
  if (hi == 0ull) return ldexp(__ull2double_rn(lo), -scale);
  const int sh = 64 - __clzll(static_cast<long long>(hi));  // 1..64 bits above the top 64
  unsigned long long top = static_cast<unsigned long long>(u >> sh);
  const unsigned long long rest = sh == 64 ? lo : (lo & ((1ull << sh) - 1ull));
  top |= rest != 0ull ? 1ull : 0ull;  // sticky bit below the rounding point
  return ldexp(__ull2double_rn(top), sh - scale);
}

template <class Real, int RK, int RS, int NWK, int NWS>
__global__ void __launch_bounds__(32 * NWK * NWS, 2) stripe_isect_kernel(const IsectArgs a) {
  using T = IsectTile<RK, RS, NWK, NWS>;
  extern __shared__ __align__(16) unsigned char smem[];
  uint2* sL = reinterpret_cast<uint2*>(smem + T::OFF_L);
  uint32_t* occU = reinterpret_cast<uint32_t*>(smem + T::OFF_OU);
  uint32_t* occV = reinterpret_cast<uint32_t*>(smem + T::OFF_OV);
  uint32_t* offU = reinterpret_cast<uint32_t*>(smem + T::OFF_FU);
  uint32_t* offV = reinterpret_cast<uint32_t*>(smem + T::OFF_FV);
  uint32_t* pkU = reinterpret_cast<uint32_t*>(smem + T::OFF_PU);
  uint32_t* pkV = reinterpret_cast<uint32_t*>(smem + T::OFF_PV);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wk = warp % NWK;
  const int ws = warp / NWK;
  const int n = a.n;
  const int k0 = blockIdx.x * T::TK;
  const int s0 = a.s_begin + blockIdx.y * T::TS;
  const int64_t P0 = static_cast<int64_t>(k0) + s0 + 1;

  // slot (j, i): sample k0 + wk*RK + j, stripe s0 + ws*32*RS + lane + 32*i
  unsigned long long GH[RK][RS], GL[RK][RS];
  uint32_t valid = 0u;
#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      GH[j][i] = 0ull;
      GL[j][i] = 0ull;
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      valid |= (k < n && s < a.s_end ? 1u : 0u) << (j * RS + i);
    }
  unsigned long long executed = 0;

  for (int g = 0; g < a.G; ++g) {
    const int64_t gb = static_cast<int64_t>(g) * a.n_ext;
    const uint32_t bu0 = __ldg(a.base + gb + k0);
    const uint32_t bv0 = __ldg(a.base + gb + P0);
    const int nu = static_cast<int>(__ldg(a.base + gb + k0 + T::TK) - bu0);
    const int nv = static_cast<int>(__ldg(a.base + gb + P0 + T::VW) - bv0);
    __syncthreads();
    if (tid < T::TK) {
      occU[tid] = __ldg(a.occ + gb + k0 + tid);
      offU[tid] = __ldg(a.base + gb + k0 + tid) - bu0;
    } else if (tid < T::TK + T::VW) {
      const int c = tid - T::TK;
      occV[c] = __ldg(a.occ + gb + P0 + c);
      offV[c] = __ldg(a.base + gb + P0 + c) - bv0;
    }
    for (int i = tid; i < nu; i += T::NT) pkU[i] = __ldg(a.packed + bu0 + i);
    for (int i = tid; i < nv; i += T::NT) pkV[i] = __ldg(a.packed + bv0 + i);
    for (int i = tid; i < 1024; i += T::NT) sL[i] = __ldg(a.limbs + static_cast<int64_t>(g) * 1024 + i);
    __syncthreads();

#pragma unroll
    for (int j = 0; j < RK; ++j) {
      const int cu = wk * RK + j;
      const uint32_t ou = occU[cu];
      const uint32_t* pu = pkU + offU[cu];
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        if (!(valid & (1u << (j * RS + i)))) continue;
        const int cv = cu + ws * 32 * RS + lane + 32 * i;
        const uint32_t ov = occV[cv];
        const uint32_t* pv = pkV + offV[cv];
        uint32_t o = ou & ov;
        unsigned long long gh = GH[j][i], gl = GL[j][i];
        while (o) {
          const int w = __clz(o);  // next word present in both columns
          o ^= 0x80000000u >> w;
          const uint32_t above = ~(0xffffffffu >> w);  // words before w
          uint32_t x = pu[__popc(ou & above)] & pv[__popc(ov & above)];
          executed += __popc(x);
          const uint2* Lw = sL + 32 * w;
          while (x) {
            const int r = __clz(x);
            x ^= 0x80000000u >> r;
            const uint2 L = Lw[r];
            gh += L.x;
            gl += L.y;
          }
        }
        GH[j][i] = gh;
        GL[j][i] = gl;
      }
    }
  }

  const unsigned long long* xs = a.colsum;
  const long long ch = static_cast<long long>(a.cacc[0]);
  const long long cl = static_cast<long long>(a.cacc[1]);
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      if (!(valid & (1u << (j * RS + i)))) continue;
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      int l = k + s + 1;
      if (l >= n) l -= n;
      const long long gh = static_cast<long long>(GH[j][i]);
      const long long gl = static_cast<long long>(GL[j][i]);
      const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + l]) + ch - gh;
      const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + l]) + cl - gl;
      const long long dh = static_cast<long long>(xs[k] + xs[l]) - 2 * gh;
      const long long dl = static_cast<long long>(xs[n + k] + xs[n + l]) - 2 * gl;
      const __int128 tv = (static_cast<__int128>(th) << 32) + tl;
      const __int128 dv = (static_cast<__int128>(dh) << 32) + dl;
      const Real t = static_cast<Real>(fixed_to_double(tv, a.scale));
      Real d = static_cast<Real>(fixed_to_double(dv, a.scale));
      if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
      const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
      dist[off] = d;
      tot[off] = t;
    }
  if (a.exec_updates) {
    for (int off = 16; off > 0; off >>= 1) executed += __shfl_down_sync(0xffffffffu, executed, off);
    if (lane == 0) atomicAdd(a.exec_updates, executed);
  }
}

}  // namespace sf
