// Weighted split (kernel 13, WN / WU): heavy rows dense, light rows
// scattered exactly.
//
// The weighted distance of a slot (k, l) is the sum over the rows present in
// u = column k or v = column l of fl(|u - v| L) (kernels.hpp:55-66; v = 0 when
// absent: the term is fl(u L)). The rows split by presence count m_r:
//
//  * heavy rows (m_r >= frac n): dense [H][ldh] values (0 = absent) and one
//    FP64 (fp32: FP32) DADD + DFMA per (row, slot), |u - v| folded into the
//    DFMA's operand modifier. All terms are >= 0 and added directly, so there
//    is no cancellation: d_heavy is within ~H eps of its exact value.
//  * light rows: with a = fix(e_u), b = fix(e_v) (e = fl(x L), converted
//    EXACTLY to 128-bit fixed point on the grid 2^-G, G ~ 100; only bits
//    below 2^-G are dropped), the slot's light part is
//        sum_{u only} a + sum_{v only} b + sum_{both} |a - b|
//      = AL_k + AL_l - 2 sum_{light rows in both} min(a, b)
//    with AL_c the column's sum of fix(e) over its light rows. The shared
//    row's term |a - b| is within one ulp of the reference's fl(|u - v| L)
//    (identical samples: exactly 0), and the sum itself is exact, rounded
//    once. Per (column k, slot tile) a CTA owns the tile's accumulators in
//    shared memory as balanced 16-bit digit planes (native 32-bit shared
//    reductions; carry-normalised every 2^15 rows) and walks column k's
//    light rows: per row, the members of the row's sorted (sample, e_v) list
//    inside the tile's window, one lane each: one conversion and ND
//    reductions per pair.
//
// The dense kernel's epilogue adds the light part (already rounded once to
// double), forms WN's separable total t = A_k + A_l (double-double column
// sums) and finalizes. Work per slot: H dense evaluations + the light shared
// rows, instead of the u-walk's (u row, slot) presence tests (C3: 7.5k u rows
// per column, 1.6k shared rows per slot, 22% of them).
#pragma once

#include <cstdint>

#include "bits.cuh"
#include "stripe_kernels.cuh"
#include "wsparse_kernels.cuh"

namespace sf {

// ---- exact double -> fixed point (grid 2^-G): floor(x 2^G), x >= 0 finite
__device__ __forceinline__ unsigned __int128 wx_to_fix(double x, int G) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const int ex = static_cast<int>((b >> 52) & 0x7ff);
  if (ex == 0 && (b << 1) == 0ull) return 0;
  const unsigned long long m = (b & ((1ull << 52) - 1ull)) | (ex ? (1ull << 52) : 0ull);
  const int sh = (ex ? ex : 1) - 1075 + G;
  if (sh >= 0) return static_cast<unsigned __int128>(m) << sh;
  if (sh > -64) return static_cast<unsigned __int128>(m >> (-sh));
  return 0;
}

// 64-bit shifts with PTX semantics: amounts >= 64 give 0.
__device__ __forceinline__ unsigned long long wx_shl(unsigned long long x, uint32_t s) {
  unsigned long long r;
  asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s));
  return r;
}
__device__ __forceinline__ unsigned long long wx_shr(unsigned long long x, uint32_t s) {
  unsigned long long r;
  asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s));
  return r;
}

// The same value as two 64-bit words (lo, hi), branch-free.
__device__ __forceinline__ void wx_fix2(double x, int G, unsigned long long& lo, unsigned long long& hi) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const int ex = static_cast<int>(b >> 52);  // x >= 0
  const unsigned long long m = (b & ((1ull << 52) - 1ull)) | (ex ? (1ull << 52) : 0ull);
  const int sh = (ex ? ex : 1) - 1075 + G;  // value = m 2^sh on the grid
  lo = sh >= 0 ? wx_shl(m, static_cast<uint32_t>(sh)) : wx_shr(m, static_cast<uint32_t>(-sh));
  hi = sh >= 64 ? wx_shl(m, static_cast<uint32_t>(sh - 64)) : wx_shr(m, static_cast<uint32_t>(64 - sh));
}

// Generalized UniFrac (extension) per-row terms, s = u + v > 0:
// d_s = w |u - v| / s, t_s = w with w = s^alpha L (stripe_kernels.cuh's
// update_generalized). SQ: alpha = 0.5 through one rsqrt (d_s = L |u-v| /
// sqrt(s), t_s = L sqrt(s)), within a few ulp of the sqrt + divide form.
// s = 0 (both absent) gives 0, 0.
template <class Real, bool SQ>
__device__ __forceinline__ void wx_gen_terms(Real u, Real v, Real L, Real alpha, Real& ds, Real& ts) {
  const Real s = u + v;
  const Real ad = u > v ? u - v : v - u;
  if (SQ) {
    const Real r = s > Real(0) ? rsqrt(s) : Real(0);
    ds = (ad * r) * L;
    ts = (s * r) * L;
  } else {
    const Real w = s > Real(0) ? pow_alpha(s, alpha) * L : Real(0);
    ds = s > Real(0) ? w * (ad / s) : Real(0);
    ts = w;
  }
}

// ---- build --------------------------------------------------------------------

// ---- sparse value build (no dense embedding rows) ---------------------------------
// The weighted rows are built from presence bits and the value pool alone:
// 1. presence bit rows [E][RW] (leaves: value != 0, internal: OR of the
//    children — exactly the rows whose dense value is nonzero);
// 2. presence words nb[w][c] (32 rows) + counts, scanned into pool offsets;
// 3. leaf values c / total[s] straight into the pool (table.cpp:208-214);
// 4. internal values, one launch per tree height: 0 + the present children's
//    values in postorder (a child absent from the column adds +0.0 in the
//    reference's fold, embed.cpp:71-79, so skipping it changes no bit).
// The pool, offsets and words are the chunked build's, bit for bit.

// Weighted leaf presence: the value c / total[s] is nonzero.
__global__ void wx_leaf_bits_kernel(uint32_t* __restrict__ bits, int64_t RW, const int32_t* __restrict__ leaf_rows,
                                    const int32_t* __restrict__ leaf_feat, int32_t n_leaf,
                                    const int64_t* __restrict__ feat_ptr, const int32_t* __restrict__ sidx,
                                    const double* __restrict__ counts, const double* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_leaf; i += nwarps) {
    uint32_t* row = bits + static_cast<int64_t>(leaf_rows[i]) * RW;
    const int f = leaf_feat[i];
    for (int64_t e = feat_ptr[f] + lane; e < feat_ptr[f + 1]; e += 32) {
      const int s = sidx[e];
      if (counts[e] / totals[s] != 0.0) atomicOr(row + (s >> 5), 1u << (s & 31));
    }
  }
}

// Presence words (row 32w + i at bit 31 - i) and their counts; columns past
// n count 0 (their words are copied in by ws_extend_kernel after the scan).
__global__ void wx_words_kernel(const uint32_t* __restrict__ bits, int64_t RW, int32_t E, int32_t n, int32_t W,
                                int64_t n_ext, uint32_t* __restrict__ nb, uint32_t* __restrict__ cnt) {
  const int64_t total = static_cast<int64_t>(W) * n_ext;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / n_ext;
    const int64_t c = i - w * n_ext;
    uint32_t x = 0u;
    if (c < n) {
      const int r_end = min(32, E - static_cast<int>(32 * w));
      const uint32_t* col = bits + 32 * w * RW + (c >> 5);
      const int b = static_cast<int>(c & 31);
      for (int r = 0; r < r_end; ++r)
        if ((__ldg(col + static_cast<int64_t>(r) * RW) >> b) & 1u) x |= 0x80000000u >> r;
    }
    nb[i] = x;
    cnt[i] = static_cast<uint32_t>(__popc(x));
  }
}

// Pool index of (row r, column c), r present in c.
__device__ __forceinline__ uint32_t wx_pos(const uint32_t* __restrict__ nb, const uint32_t* __restrict__ off,
                                           int64_t n_ext, int32_t r, int32_t c) {
  const int64_t cell = static_cast<int64_t>(r >> 5) * n_ext + c;
  const int i = r & 31;
  return __ldg(off + cell) + static_cast<uint32_t>(__popc(__ldg(nb + cell) & ~(0xffffffffu >> i)));
}

// Leaf values into the pool: warp per leaf row (embed_leaf_values' formula).
__global__ void wx_leaf_values_kernel(double* __restrict__ pool, const uint32_t* __restrict__ nb,
                                      const uint32_t* __restrict__ off, int64_t n_ext,
                                      const int32_t* __restrict__ leaf_rows, const int32_t* __restrict__ leaf_feat,
                                      int32_t n_leaf, const int64_t* __restrict__ feat_ptr,
                                      const int32_t* __restrict__ sidx, const double* __restrict__ counts,
                                      const double* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_leaf; i += nwarps) {
    const int32_t r = leaf_rows[i];
    const int f = leaf_feat[i];
    for (int64_t e = feat_ptr[f] + lane; e < feat_ptr[f + 1]; e += 32) {
      const int s = sidx[e];
      const double v = counts[e] / totals[s];
      if (v != 0.0) pool[wx_pos(nb, off, n_ext, r, s)] = v;
    }
  }
}

// Internal rows of one height: thread per (row, 32-column word); per present
// column, 0 + the present children's values in postorder (codes: child rows).
__global__ void wx_level_values_kernel(double* __restrict__ pool, const uint32_t* __restrict__ bits, int64_t RW,
                                       const uint32_t* __restrict__ nb, const uint32_t* __restrict__ off,
                                       int64_t n_ext, const int32_t* __restrict__ rows,
                                       const int32_t* __restrict__ cptr, const int32_t* __restrict__ codes,
                                       int32_t n_rows) {
  const int64_t total = static_cast<int64_t>(n_rows) * RW;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / RW;
    const int64_t cw = t - i * RW;
    const int32_t r = rows[i];
    uint32_t b = __ldg(bits + static_cast<int64_t>(r) * RW + cw);
    while (b) {
      const int j = __ffs(b) - 1;
      b &= b - 1u;
      const int32_t c = static_cast<int32_t>(32 * cw + j);
      double acc = 0.0;  // pending_ starts at zero (embed.cpp:75-76)
      for (int k = cptr[i]; k < cptr[i + 1]; ++k) {
        const int32_t ch = codes[k];
        if ((__ldg(bits + static_cast<int64_t>(ch) * RW + cw) >> j) & 1u) acc += pool[wx_pos(nb, off, n_ext, ch, c)];
      }
      pool[wx_pos(nb, off, n_ext, r, c)] = acc;
    }
  }
}

// Generalized: the u-walk's second pool (kernel 12's fallback), a = v^alpha L
// per present entry in pool order (wu_fill_kernel's formula).
template <class Real>
__global__ void wx_poola_kernel(const uint32_t* __restrict__ nb, const uint32_t* __restrict__ off, int64_t n_ext,
                                int32_t n, int32_t W, const double* __restrict__ lens, double alpha,
                                const Real* __restrict__ pool, Real* __restrict__ poola) {
  const int64_t total = static_cast<int64_t>(W) * n;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t / n;
    const int64_t c = t - w * n;
    uint32_t bits = nb[w * n_ext + c];
    uint32_t q = off[w * n_ext + c];
    while (bits) {
      const int r = __clz(bits);
      bits ^= 0x80000000u >> r;
      poola[q] = pow_alpha(pool[q], static_cast<Real>(alpha)) * static_cast<Real>(lens[32 * w + r]);
      ++q;
    }
  }
}

__global__ void wx_pool_to_float_kernel(const double* __restrict__ p64, const unsigned long long* __restrict__ total,
                                        float* __restrict__ p32) {
  const unsigned long long m = *total;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
    p32[i] = static_cast<float>(p64[i]);  // cast_batch: the fp64 row rounded once (embed.hpp:71-84)
}

// m_r: samples with row r present (presence words nb[w][c], row 32w+i at bit 31-i).
__global__ void wx_rowcount_kernel(const uint32_t* __restrict__ nb, int64_t n_ext, int32_t n, int32_t W,
                                   int32_t E, uint32_t* __restrict__ cnt) {
  __shared__ unsigned int sc[32];
  for (int32_t w = blockIdx.x; w < W; w += gridDim.x) {
    if (threadIdx.x < 32) sc[threadIdx.x] = 0u;
    __syncthreads();
    const uint32_t* row = nb + static_cast<int64_t>(w) * n_ext;
    for (int32_t c = threadIdx.x; c < n; c += blockDim.x) {
      uint32_t x = __ldg(row + c);
      while (x) {
        const int i = __clz(x);
        x ^= 0x80000000u >> i;
        atomicAdd(&sc[i], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32 && 32 * w + static_cast<int>(threadIdx.x) < E) cnt[32 * w + threadIdx.x] = sc[threadIdx.x];
    __syncthreads();
  }
}

// Heavy / light flags: heavy = present in >= thr samples; rows with L = 0
// add nothing and are dropped. hflag / lcnt are the scan inputs (E + 1
// entries, the last one 0); hmask / lmask the per-word bit masks.
__global__ void wx_classify_kernel(const uint32_t* __restrict__ cnt, const double* __restrict__ lens, int32_t E,
                                   int32_t W, uint32_t thr, uint32_t* __restrict__ hflag,
                                   unsigned long long* __restrict__ lcnt, uint32_t* __restrict__ hmask,
                                   uint32_t* __restrict__ lmask) {
  const int64_t total = static_cast<int64_t>(W) * 32;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = static_cast<int32_t>(i);
    const uint32_t m = r < E ? cnt[r] : 0u;
    const bool live = r < E && m > 0u && lens[r] != 0.0;
    const bool heavy = live && m >= thr;
    const bool light = live && !heavy;
    if (r < E) {
      hflag[r] = heavy ? 1u : 0u;
      lcnt[r] = light ? m : 0ull;
    }
    const uint32_t hb = __ballot_sync(0xffffffffu, heavy);
    const uint32_t lb = __ballot_sync(0xffffffffu, light);
    // lane j of the word holds row 32w + j: bit 31 - j in the presence words
    if ((threadIdx.x & 31) == 0) {
      hmask[r / 32] = __brev(hb);
      lmask[r / 32] = __brev(lb);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hflag[E] = 0u;
    lcnt[E] = 0ull;
  }
}

// Warp per presence word: heavy rows' values into the dense matrix UH (zeroed
// before), light rows' (sample, value) members in sample order at lptr[r].
template <class Real, bool GEN>
__global__ void wx_fill_kernel(const uint32_t* __restrict__ nb, const uint32_t* __restrict__ off,
                               const Real* __restrict__ pool, int64_t n_ext, int32_t n, int32_t W,
                               const uint32_t* __restrict__ hmask, const uint32_t* __restrict__ lmask,
                               const uint32_t* __restrict__ hidx, const unsigned long long* __restrict__ lptr,
                               int64_t ldh, const double* __restrict__ lens, double alpha, Real* __restrict__ UH,
                               int32_t* __restrict__ lmid, Real* __restrict__ lval, Real* __restrict__ lvala,
                               uint32_t* __restrict__ prank) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = warp; w < W; w += nwarps) {
    const uint32_t hm = hmask[w], lm = lmask[w];
    if (!(hm | lm)) continue;
    const int32_t rl = static_cast<int32_t>(32 * w + lane);
    // lane j: row 32w + j's heavy index / light list base (+ running count)
    const int64_t hrow = (hm & (0x80000000u >> lane)) ? static_cast<int64_t>(hidx[rl]) : 0;
    unsigned long long lnext = (lm & (0x80000000u >> lane)) ? lptr[rl] : 0ull;
    const unsigned long long lfirst = lnext;
    const uint32_t* nrow = nb + w * n_ext;
    const uint32_t* orow = off + w * n_ext;
    for (int32_t c0 = 0; c0 < n; c0 += 32) {
      const int32_t c = c0 + lane;
      const uint32_t x = c < n ? __ldg(nrow + c) : 0u;
      const uint32_t any = __reduce_or_sync(0xffffffffu, x) & (hm | lm);
      if (!any) continue;
      const uint32_t o = c < n ? __ldg(orow + c) : 0u;
      uint32_t bits = any;
      while (bits) {
        const int i = __clz(bits);
        const uint32_t bm = 0x80000000u >> i;
        bits ^= bm;
        const bool has = (x & bm) != 0u;
        Real v = Real(0);
        const uint32_t q = o + static_cast<uint32_t>(__popc(x & ~(0xffffffffu >> i)));
        if (has) v = pool[q];
        if (hm & bm) {
          const int64_t h = __shfl_sync(0xffffffffu, hrow, i);
          if (has) UH[h * ldh + c] = v;
        } else {
          const uint32_t bal = __ballot_sync(0xffffffffu, has);
          const unsigned long long base = __shfl_sync(0xffffffffu, lnext, i);
          const unsigned long long start = __shfl_sync(0xffffffffu, lfirst, i);
          if (has) {
            const unsigned long long p = base + static_cast<unsigned>(__popc(bal & ((1u << lane) - 1u)));
            lmid[p] = c;
            const Real L = static_cast<Real>(lens[32 * w + i]);
            if (GEN) {  // v itself and the one-sided term a_v = v^alpha L
              lval[p] = v;
              lvala[p] = pow_alpha(v, static_cast<Real>(alpha)) * L;
            } else {
              lval[p] = L * v;  // e_v = fl(v L), the light term's operand
            }
            prank[q] = static_cast<uint32_t>(p - start);  // the column's position in the row's list
          }
          if (lane == i) lnext += static_cast<unsigned>(__popc(bal));
        }
      }
    }
  }
}

// Heavy rows' lengths in heavy order (the dense kernel's L).
template <class Real>
__global__ void wx_heavylen_kernel(const uint32_t* __restrict__ hflag, const uint32_t* __restrict__ hidx,
                                   const double* __restrict__ lens, int32_t E, Real* __restrict__ LH) {
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < E; r += gridDim.x * blockDim.x)
    if (hflag[r]) LH[hidx[r]] = static_cast<Real>(lens[r]);
}

// Wrap columns of the dense heavy matrix: UH[h][c] = UH[h][c mod n], c >= n.
template <class Real>
__global__ void wx_extend_kernel(Real* __restrict__ UH, int64_t H, int64_t ldh, int32_t n) {
  const int64_t wcols = ldh - n;
  const int64_t total = H * wcols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t h = i / wcols;
    const int64_t c = n + (i - h * wcols);
    UH[h * ldh + c] = UH[h * ldh + c % n];
  }
}

// Light rows per column: warp per column, lanes over the 32-word groups of
// the column's nonzero-word masks.
__global__ void wx_colcount_kernel(const uint32_t* __restrict__ nb, const uint32_t* __restrict__ nz,
                                   const uint32_t* __restrict__ lmask, int64_t n_ext, int32_t n, int32_t W,
                                   unsigned long long* __restrict__ ccnt) {
  const int NG = (W + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = warp; k < n; k += nwarps) {
    unsigned long long c = 0;
    for (int g = lane; g < NG; g += 32) {
      uint32_t m = __ldg(nz + static_cast<int64_t>(g) * n + k);
      while (m) {
        const int w = 32 * g + __ffs(m) - 1;
        m &= m - 1u;
        c += static_cast<unsigned>(__popc(__ldg(nb + static_cast<int64_t>(w) * n_ext + k) & __ldg(lmask + w)));
      }
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) ccnt[k] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ccnt[n] = 0ull;
}

// Column k's light rows in ascending order (row, value, the column's rank in
// the row's member list) and AL_k = sum of fix(fl(u L)) over them. Warp per
// column: lane g takes the 32-word groups g, g + 32, ... in turn, each round
// placed after the previous round's entries by a warp scan.
template <class Real, bool GEN>
__global__ void wx_colfill_kernel(const uint32_t* __restrict__ nb, const uint32_t* __restrict__ off,
                                  const uint32_t* __restrict__ nz, const uint32_t* __restrict__ lmask,
                                  const Real* __restrict__ pool, const uint32_t* __restrict__ prank,
                                  const double* __restrict__ lens, double alpha, int64_t n_ext, int32_t n, int32_t W,
                                  int G,
                                  const unsigned long long* __restrict__ cptr, int32_t* __restrict__ crow,
                                  Real* __restrict__ cval, uint32_t* __restrict__ crank,
                                  unsigned long long* __restrict__ AL) {
  const int NG = (W + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = warp; k < n; k += nwarps) {
    unsigned long long base = cptr[k];
    unsigned __int128 acc = 0;
    for (int g0 = 0; g0 < NG; g0 += 32) {
      const int g = g0 + lane;
      const uint32_t m0 = g < NG ? __ldg(nz + static_cast<int64_t>(g) * n + k) : 0u;
      // this lane's light rows in the group
      unsigned cnt = 0;
      for (uint32_t m = m0; m;) {
        const int w = 32 * g + __ffs(m) - 1;
        m &= m - 1u;
        cnt += static_cast<unsigned>(__popc(__ldg(nb + static_cast<int64_t>(w) * n_ext + k) & __ldg(lmask + w)));
      }
      unsigned incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      unsigned long long p = base + (incl - cnt);
      for (uint32_t m = m0; m;) {
        const int w = 32 * g + __ffs(m) - 1;
        m &= m - 1u;
        const uint32_t x = __ldg(nb + static_cast<int64_t>(w) * n_ext + k);
        uint32_t lx = x & __ldg(lmask + w);
        if (!lx) continue;
        const uint32_t o = __ldg(off + static_cast<int64_t>(w) * n_ext + k);
        while (lx) {
          const int i = __clz(lx);
          lx ^= 0x80000000u >> i;
          const uint32_t q = o + static_cast<uint32_t>(__popc(x & ~(0xffffffffu >> i)));
          const Real u = pool[q];
          const int32_t r = 32 * w + i;
          crow[p] = r;
          cval[p] = u;
          crank[p] = prank[q];
          ++p;
          // the one-sided term: fl(u L) (weighted), u^alpha L (generalized)
          const Real e = GEN ? pow_alpha(u, static_cast<Real>(alpha)) * static_cast<Real>(lens[r])
                             : static_cast<Real>(lens[r]) * u;
          acc += wx_to_fix(static_cast<double>(e), G);
        }
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    // the column's sum: lanes' partial sums (exact integers, any order)
    unsigned long long lo = static_cast<unsigned long long>(acc), hi = static_cast<unsigned long long>(acc >> 64);
    for (int o = 16; o; o >>= 1) {
      const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o);
      const unsigned long long hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
      const unsigned long long s = lo + lo2;
      hi = hi + hi2 + (s < lo ? 1ull : 0ull);
      lo = s;
    }
    if (lane == 0) {
      AL[2 * k] = lo;
      AL[2 * k + 1] = hi;
    }
  }
}

// ---- light scatter ------------------------------------------------------------

struct WSLightArgs {
  const unsigned long long* cptr;  // [n + 1] column light lists
  const int32_t* crow;
  const void* cval;                // Real
  const uint32_t* crank;           // the column's position in each row's member list
  const unsigned long long* lptr;  // [E + 1] light rows' member lists (sorted samples)
  const int32_t* lmid;
  const void* lval;                // Real: e_v = fl(v L) (weighted) or v (generalized)
  const void* lvala;               // Real: a_v = v^alpha L (generalized), else null
  double alpha;
  const double* lens;
  const unsigned long long* AL;    // [n] x 2 (lo, hi)
  int32_t n;
  int32_t s_begin, s_end;          // stripes of this device
  int32_t out_begin;
  int32_t tile;                    // slots per CTA
  int32_t G;                       // fixed-point grid 2^-G
  int32_t nd;                      // 16-bit digit planes (<= 8)
  double* lightd;                  // [stripes][n] light part, rounded once
  double* lightt;                  // generalized: the totals' light part, else null
  unsigned long long* pairs;       // light (row, slot) pairs scattered (stats), or null
};

constexpr int kWSLightThreads = 1024;
constexpr int kWSLightSmem = 200 * 1024;  // digit planes: nd x tile x 4 bytes
constexpr int kWSFold = 32768;            // rows between carry normalisations (2^15 x 2^15 adds < 2^31)
#ifndef SF_WS_UNROLL
#define SF_WS_UNROLL 4
#endif
constexpr int kWSUnroll = SF_WS_UNROLL;   // member loads in flight per lane

// first index in [a, b) of the sorted ids with id >= x
__device__ __forceinline__ unsigned long long wx_lower(const int32_t* __restrict__ ids, unsigned long long a,
                                                       unsigned long long b, int32_t x) {
  while (a < b) {
    const unsigned long long mid = (a + b) >> 1;
    if (__ldg(ids + mid) < x)
      a = mid + 1;
    else
      b = mid;
  }
  return a;
}

// Members [p, ...) of one row with ids <= hi, slot = id + sh: the lanes take
// 32 x kWSUnroll at a time until the sorted ids pass hi. The member lists
// hold e_v = fl(v L) (the row's own length). With a = fix(e_u), b = fix(e_v)
// the shared row's term |a - b| plus the one-sided a + b already in the
// column sums leaves X = |a - b| - a - b = -2 min(a, b): one conversion per
// pair. X goes in as balanced 16-bit digits: Y = B - 2 min(a, b) with
// B = 2^15 in every 16-bit field, so digit j is field j of Y minus 2^15.
template <class Real, int ND>
__device__ __forceinline__ void wx_light_walk(const WSLightArgs& a, unsigned long long p, unsigned long long pe,
                                              int32_t hi, int32_t sh, Real eu, uint32_t planes_s, int T, int G,
                                              unsigned long long& pairs) {
  const int lane = threadIdx.x & 31;
  const Real* __restrict__ lval = static_cast<const Real*>(a.lval);
  constexpr unsigned long long kB = 0x8000800080008000ull;
  for (unsigned long long pb = p;; pb += 32 * kWSUnroll) {
    int32_t id[kWSUnroll];
    Real ev[kWSUnroll];
#pragma unroll
    for (int j = 0; j < kWSUnroll; ++j) {
      const unsigned long long m = pb + lane + 32 * j;
      id[j] = m < pe ? __ldg(a.lmid + m) : INT32_MAX;
      ev[j] = m < pe ? lval[m] : Real(0);
    }
    bool more = true;
#pragma unroll
    for (int j = 0; j < kWSUnroll; ++j) {
      if (id[j] > hi) {
        more = false;
        continue;
      }
      ++pairs;
      // shared-window address of the slot in digit plane 0
      const uint32_t cell = planes_s + 4u * static_cast<uint32_t>(id[j] + sh);
      unsigned long long ml, mh;
      wx_fix2(static_cast<double>(eu < ev[j] ? eu : ev[j]), G, ml, mh);
      // Y = B - 2 min (mod 2^128)
      const unsigned long long tl = ml << 1, th = (mh << 1) | (ml >> 63);
      const unsigned long long yl = kB - tl;
      const unsigned long long yh = kB - th - (kB < tl ? 1ull : 0ull);
      const uint32_t w[4] = {static_cast<uint32_t>(yl), static_cast<uint32_t>(yl >> 32), static_cast<uint32_t>(yh),
                             static_cast<uint32_t>(yh >> 32)};
      // the ND planes' digits (those above are 0: |X| < 2^(16 ND - 1)); a
      // zero digit is added too (cheaper than branching around it)
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        const int32_t dg = static_cast<int32_t>((w[d >> 1] >> (16 * (d & 1))) & 0xffffu) - 0x8000;
        asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(cell + 4u * static_cast<uint32_t>(d * T)), "r"(dg)
                     : "memory");
      }
    }
    if (!__all_sync(0xffffffffu, more)) break;
  }
}

// Generalized (extension): the shared row's d and t terms replace the
// one-sided a_u + a_v already in the column sums, X = fix(term) - fix(a_v) -
// fix(a_u) for each, two sets of digit planes (t at plane ND). The row
// constant c = B - fix(a_u).
template <class Real, int ND, bool SQ>
__device__ __forceinline__ void wx_light_walk_gen(const WSLightArgs& a, unsigned long long p, unsigned long long pe,
                                                  int32_t hi, int32_t sh, Real u, Real L, unsigned long long c_lo,
                                                  unsigned long long c_hi, uint32_t planes_s, int T, int G,
                                                  unsigned long long& pairs) {
  const int lane = threadIdx.x & 31;
  const Real* __restrict__ lval = static_cast<const Real*>(a.lval);
  const Real* __restrict__ lvala = static_cast<const Real*>(a.lvala);
  const Real alpha = static_cast<Real>(a.alpha);
  for (unsigned long long pb = p;; pb += 32 * kWSUnroll) {
    int32_t id[kWSUnroll];
    Real v[kWSUnroll], av[kWSUnroll];
#pragma unroll
    for (int j = 0; j < kWSUnroll; ++j) {
      const unsigned long long m = pb + lane + 32 * j;
      id[j] = m < pe ? __ldg(a.lmid + m) : INT32_MAX;
      v[j] = m < pe ? lval[m] : Real(0);
      av[j] = m < pe ? lvala[m] : Real(0);
    }
    bool more = true;
#pragma unroll
    for (int j = 0; j < kWSUnroll; ++j) {
      if (id[j] > hi) {
        more = false;
        continue;
      }
      ++pairs;
      const uint32_t cell = planes_s + 4u * static_cast<uint32_t>(id[j] + sh);
      Real ds, ts;
      wx_gen_terms<Real, SQ>(u, v[j], L, alpha, ds, ts);
      unsigned long long el, eh;
      wx_fix2(static_cast<double>(av[j]), G, el, eh);
      // c - fix(a_v), then + fix(term) for d and for t
      const unsigned long long bl = c_lo - el;
      const unsigned long long bh = c_hi - eh - (c_lo < el ? 1ull : 0ull);
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        unsigned long long tl, th;
        wx_fix2(static_cast<double>(which ? ts : ds), G, tl, th);
        const unsigned long long yl = bl + tl;
        const unsigned long long yh = bh + th + (yl < bl ? 1ull : 0ull);
        const uint32_t w[4] = {static_cast<uint32_t>(yl), static_cast<uint32_t>(yl >> 32), static_cast<uint32_t>(yh),
                               static_cast<uint32_t>(yh >> 32)};
        const uint32_t base = cell + 4u * static_cast<uint32_t>(which * ND * T);
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          const int32_t dg = static_cast<int32_t>((w[d >> 1] >> (16 * (d & 1))) & 0xffffu) - 0x8000;
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(base + 4u * static_cast<uint32_t>(d * T)), "r"(dg)
                       : "memory");
        }
      }
    }
    if (!__all_sync(0xffffffffu, more)) break;
  }
}

// Per (column k, tile of slots): column k's light rows, warp per row, the
// members of the row inside the tile's window (from the column's own
// position in the row's list when the window starts right after k), exact
// digit-plane accumulation; then each slot's exact light sum AL_k + AL_l +
// sum, rounded once.
template <class Real, int ND, int GENA>
__global__ void __launch_bounds__(kWSLightThreads, 1) wx_light_kernel(const WSLightArgs a) {
  constexpr bool GEN = GENA >= 0;
  constexpr int NP = GEN ? 2 : 1;      // plane sets: d (and t)
  extern __shared__ int32_t planes[];  // [NP][nd][tile]
  const int k = blockIdx.x;
  const int n = a.n;
  const int s_lo = a.s_begin + static_cast<int>(blockIdx.y) * a.tile;
  const int s_hi = min(a.s_end, s_lo + a.tile);
  const int T = a.tile;
  constexpr int nd = ND;
  const int G = a.G;
  const int lane = threadIdx.x & 31;
  const Real* __restrict__ cval = static_cast<const Real*>(a.cval);
  const unsigned long long r0 = a.cptr[k], r1 = a.cptr[k + 1];
  // the window l = k + s + 1, s in [s_lo, s_hi): ids in (k + s_lo, k + s_hi]
  // above k (part A) and, past n, wrapped below k (part B)
  const int64_t xa = static_cast<int64_t>(k) + s_lo + 1, xb = static_cast<int64_t>(k) + s_hi;
  const int32_t hiA = static_cast<int32_t>(xb < n ? xb : n - 1);
  const bool hasA = xa < n;
  const int32_t loB = static_cast<int32_t>(xa > n ? xa - n : 0);
  const int32_t hiB = static_cast<int32_t>(xb - n);
  const bool hasB = xb >= n;
  const int32_t shA = -k - 1 - s_lo, shB = n - k - 1 - s_lo;
  for (int i = threadIdx.x; i < NP * nd * T; i += kWSLightThreads) planes[i] = 0;
  const uint32_t planes_s = static_cast<uint32_t>(__cvta_generic_to_shared(planes));
  __syncthreads();
  unsigned long long pairs = 0;
  __shared__ unsigned int next_row;  // rows are taken dynamically: lists differ in length
  for (unsigned long long f0 = r0; f0 < r1; f0 += kWSFold) {
    const unsigned long long f1 = min(r1, f0 + kWSFold);
    if (threadIdx.x == 0) next_row = 0u;
    __syncthreads();
    for (;;) {
      unsigned int j = 0;
      if (lane == 0) j = atomicAdd(&next_row, 1u);
      const unsigned long long e = f0 + __shfl_sync(0xffffffffu, j, 0);
      if (e >= f1) break;
      const int32_t r = __ldg(a.crow + e);
      const Real u = cval[e];
      const uint32_t rank = __ldg(a.crank + e);
      const Real L = static_cast<Real>(__ldg(a.lens + r));
      const unsigned long long m0 = __ldg(a.lptr + r), m1 = __ldg(a.lptr + r + 1);
      const unsigned long long me = m0 + rank;  // the column itself
      const unsigned long long pa =
          hasA ? (s_lo == 0 ? me + 1 : wx_lower(a.lmid, me + 1, m1, static_cast<int32_t>(xa))) : 0ull;
      const unsigned long long pb = hasB ? (loB == 0 ? m0 : wx_lower(a.lmid, m0, me, loB)) : 0ull;
      if constexpr (GEN) {
        // c = B - fix(a_u), a_u = u^alpha L as in the column sums
        unsigned long long fl_, fh_;
        wx_fix2(static_cast<double>(pow_alpha(u, static_cast<Real>(a.alpha)) * L), G, fl_, fh_);
        const unsigned long long kB = 0x8000800080008000ull;
        const unsigned long long c_lo = kB - fl_, c_hi = kB - fh_ - (kB < fl_ ? 1ull : 0ull);
        if (hasA) wx_light_walk_gen<Real, ND, GENA == 1>(a, pa, m1, hiA, shA, u, L, c_lo, c_hi, planes_s, T, G, pairs);
        if (hasB) wx_light_walk_gen<Real, ND, GENA == 1>(a, pb, me, hiB, shB, u, L, c_lo, c_hi, planes_s, T, G, pairs);
      } else {
        const Real eu = L * u;  // fl(u L), as in the column sums
        if (hasA) wx_light_walk<Real, ND>(a, pa, m1, hiA, shA, eu, planes_s, T, G, pairs);
        if (hasB) wx_light_walk<Real, ND>(a, pb, me, hiB, shB, eu, planes_s, T, G, pairs);
      }
    }
    if (f1 < r1) {  // carry-normalise the planes before the next rows
      __syncthreads();
      for (int q = threadIdx.x; q < NP * T; q += kWSLightThreads) {
        int32_t* pl = planes + (q / T) * nd * T + (q % T);
        int32_t carry = 0;
        for (int d = 0; d + 1 < nd; ++d) {
          const int32_t v = pl[d * T] + carry;
          const int32_t lo = static_cast<int16_t>(static_cast<uint16_t>(v));
          carry = (v - lo) >> 16;
          pl[d * T] = lo;
        }
        pl[(nd - 1) * T] += carry;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  const unsigned __int128 ALk =
      (static_cast<unsigned __int128>(a.AL[2 * k + 1]) << 64) | static_cast<unsigned __int128>(a.AL[2 * k]);
  for (int q = threadIdx.x; q < T; q += kWSLightThreads) {
    const int s = s_lo + q;
    if (s >= s_hi) break;
    const int64_t li = static_cast<int64_t>(k) + s + 1;
    const int l = static_cast<int>(li >= n ? li - n : li);
    const unsigned __int128 ALl =
        (static_cast<unsigned __int128>(a.AL[2 * l + 1]) << 64) | static_cast<unsigned __int128>(a.AL[2 * l]);
#pragma unroll
    for (int set = 0; set < NP; ++set) {
      __int128 v = 0;
      for (int d = nd - 1; d >= 0; --d) v = v * 65536 + static_cast<__int128>(planes[(set * nd + d) * T + q]);
      const unsigned __int128 tot = ALk + ALl + static_cast<unsigned __int128>(v);  // >= 0: the exact light sum
      __stcs((set ? a.lightt : a.lightd) + static_cast<int64_t>(s - a.out_begin) * n + k,
             u128_to_real<double>(tot, false, -G));
    }
  }
  if (a.pairs) {
    for (int o = 16; o; o >>= 1) pairs += __shfl_down_sync(0xffffffffu, pairs, o);
    if (lane == 0 && pairs) atomicAdd(a.pairs, pairs);
  }
}

// ---- dense heavy rows + epilogue ----------------------------------------------

struct WSDenseArgs {
  const void* UH;         // Real [H][ldh]
  const void* LH;         // Real [H] heavy lengths
  int64_t H, ldh;
  int32_t n;
  int32_t s_begin, s_end;
  int32_t out_begin;
  int32_t finalize;
  const double* lightd;   // [stripes][n]
  const double* lightt;   // generalized: the totals' light part
  const double2* A;       // [n] WN column sums (double-double), t = A_k + A_l
  double alpha;           // generalized exponent
  void* dist;
  void* tot;              // null for WU
};

constexpr int kWSK = 128, kWSS = 128;  // tile: u columns x stripes
// u columns per CTA tile: generalized keeps d and t accumulators, so half
template <int M>
__host__ __device__ constexpr int wx_dense_kt() {
  return M == kGen ? kWSK / 2 : kWSK;
}
#ifndef SF_WS_R
#define SF_WS_R 16
#endif
constexpr int kWSR = SF_WS_R;          // heavy rows per cp.async stage
constexpr int kWSThreads = 256;        // 16 x 16 threads, 8 x 8 slots each (stride 16)

__device__ __forceinline__ void wx_cp8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void wx_cp4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem));
}

template <int M, class Real, bool SQ>
__global__ void __launch_bounds__(kWSThreads, 1) wx_dense_kernel(const WSDenseArgs a) {
  constexpr bool GEN = M == kGen;
  constexpr int KT = wx_dense_kt<M>();  // u columns of the tile
  constexpr int TI = KT / 16;           // per thread: TI u columns x 8 stripes
  constexpr int UW = KT, VW = KT + kWSS;  // staged values per row (VW - 1 used)
  constexpr int ROW = UW + VW;
  extern __shared__ __align__(16) unsigned char wx_smem[];
  Real* stage = reinterpret_cast<Real*>(wx_smem);  // [2][kWSR][ROW]
  Real* lstage = stage + 2 * kWSR * ROW;           // [2][kWSR]
  const int n = a.n;
  const int k0 = blockIdx.x * KT;
  const int s0 = a.s_begin + blockIdx.y * kWSS;
  const int tk = threadIdx.x & 15, ts = threadIdx.x >> 4;
  const Real* __restrict__ UH = static_cast<const Real*>(a.UH);
  const Real* __restrict__ LH = static_cast<const Real*>(a.LH);
  const int64_t vbase = static_cast<int64_t>(k0) + s0 + 1;
  const int64_t H = a.H;
  auto load = [&](int64_t h0, int buf) {
    Real* dst = stage + buf * kWSR * ROW;
    const int rows = H - h0 < kWSR ? static_cast<int>(H - h0) : kWSR;
    for (int i = threadIdx.x; i < kWSR * ROW; i += kWSThreads) {
      const int rr = i / ROW, c = i - rr * ROW;
      if (rr < rows) {
        const Real* src = UH + (h0 + rr) * a.ldh + (c < UW ? k0 + c : vbase + (c - UW));
        if (sizeof(Real) == 8)
          wx_cp8(dst + i, src);
        else
          wx_cp4(dst + i, src);
      } else {
        dst[i] = Real(0);
      }
    }
    if (threadIdx.x < kWSR) lstage[buf * kWSR + threadIdx.x] = threadIdx.x < rows ? LH[h0 + threadIdx.x] : Real(0);
    asm volatile("cp.async.commit_group;");
  };
  Real acc[TI][8], acct[GEN ? TI : 1][8];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      acc[i][j] = Real(0);
      if (GEN) acct[i][j] = Real(0);
    }
  const Real alpha = static_cast<Real>(a.alpha);
  if (H > 0) load(0, 0);
  int buf = 0;
  for (int64_t h0 = 0; h0 < H; h0 += kWSR) {
    if (h0 + kWSR < H) {
      load(h0 + kWSR, buf ^ 1);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();
    const Real* st = stage + buf * kWSR * ROW;
#pragma unroll 2
    for (int rr = 0; rr < kWSR; ++rr) {
      // thread (tk, ts) holds k = k0 + tk + 16 i, s = s0 + ts + 16 j: the
      // 16 lanes of a half-warp read consecutive values (no bank conflicts)
      const Real* ur = st + rr * ROW + tk;
      const Real* vr = st + rr * ROW + UW + tk + ts;
      const Real L = lstage[buf * kWSR + rr];
      Real win[TI + 7];
#pragma unroll
      for (int q = 0; q < TI + 7; ++q) win[q] = vr[16 * q];
#pragma unroll
      for (int i = 0; i < TI; ++i) {
        const Real u = ur[16 * i];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if constexpr (GEN) {
            Real ds, ts;
            wx_gen_terms<Real, SQ>(u, win[i + j], L, alpha, ds, ts);
            acc[i][j] += ds;
            acct[i][j] += ts;
          } else {
            acc[i][j] = fma(fabs(u - win[i + j]), L, acc[i][j]);
          }
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  // epilogue: + light part, totals, finalize
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int s = s0 + ts + 16 * j;
    if (s >= a.s_end) break;
#pragma unroll
    for (int i = 0; i < TI; ++i) {
      const int k = k0 + tk + 16 * i;
      if (k >= n) break;
      const int64_t o = static_cast<int64_t>(s - a.out_begin) * n + k;
      const double dv = static_cast<double>(acc[i][j]) + __ldcs(a.lightd + o);  // read once
      if (M == kWU) {
        __stcs(dist + o, static_cast<Real>(dv));
        continue;
      }
      if constexpr (GEN) {
        const Real tr = static_cast<Real>(static_cast<double>(acct[i][j]) + __ldcs(a.lightt + o));
        Real dr = static_cast<Real>(dv);
        if (a.finalize) dr = tr == Real(0) ? Real(0) : dr / tr;
        __stcs(dist + o, dr);
        __stcs(tot + o, tr);
        continue;
      }
      const int64_t li = static_cast<int64_t>(k) + s + 1;
      const int l = static_cast<int>(li >= n ? li - n : li);
      const double2 Ak = a.A[k], Al = a.A[l];
      double hi = Ak.x, lo = Ak.y;
      {
        const double sm = hi + Al.x;
        const double bb = sm - hi;
        lo += (hi - (sm - bb)) + (Al.x - bb);
        hi = sm;
      }
      const double tv = hi + (lo + Al.y);
      const Real tr = static_cast<Real>(tv);
      Real dr = static_cast<Real>(dv);
      if (a.finalize) dr = tr == Real(0) ? Real(0) : dr / tr;
      __stcs(dist + o, dr);  // final stripes: keep L2 for the staged heavy rows
      __stcs(tot + o, tr);
    }
  }
}

}  // namespace sf
