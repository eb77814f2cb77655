// K2-UW, split form (kernel 10, the default for the unweighted metric).
//
// update_entry<Unweighted> (kernels.hpp:55-66) summed over the rows gives
// t_kl = sum_{k in S_e or l in S_e} L_e and d_kl = sum_{k in S_e xor l in S_e} L_e.
// With X_e = S_e, or its complement when |S_e| > n/2 ("dense" rows),
//   t_kl = p_k + p_l + C - G_kl,   d_kl = x_k + x_l - 2 G_kl,
//   G_kl = sum_{e: k in X_e and l in X_e} L_e,
// x_k / p_k per-column sums (p: non-dense rows only), C the dense rows' sum.
//
// EXACT ARITHMETIC. Every length is an exact sum of fixed-point levels,
// L = sum_j v_j 2^-(scale + vb j), v_j < 2^vb integers (truncation, so every
// level is non-negative; the host splits each double until the remainder is
// zero: a length on the main grid has one level, a short branch far below
// the longest one may need two or more). Each level is an integer problem:
// its limbs (hi = v >> lo_bits, lo) sum below 2^53 over all rows, so every
// partial sum is exact in any order, and the epilogue assembles the exact
// rational value of t and d and rounds it once. The result is the correctly
// rounded exact sum for ANY double lengths.
//
//  * HEAVY rows (|X_e| >= heavy_min, ~15% of the rows and ~99% of the shared
//    rows at the EMP shape) are permuted to the front and node-packed in
//    64-row words nx[w][c]. A warp owns one u column k and 32*RS v columns;
//    it walks the set bits of its u words warp-uniformly and every lane adds
//    the row's main-level limbs to each of its slots whose v word has the bit.
//    The 0/1 factor is the AND of the v word and the bit mask itself, read as
//    the high word of a double (low word 0): 2^b for bit b is a power of two
//    (subnormal for b < 20), so fma(L * 2^-e_b, f, acc) adds L exactly or
//    adds +0. Per (u bit, slot): one LOP3 + 2 DFMA (the limbs are stored
//    pre-scaled by 2^-e_b). Bit 31 (the sign bit) goes through a shifted
//    factor of 2.0.
//  * LIGHT rows (|X_e| < heavy_min) share only ~5-10 rows per slot. Their
//    member lists are compacted once; each member pair's slot gets the row's
//    limbs with u64 atomics, band by band (L2-resident blocks).
//  * DEEP levels (lengths that are not on the main grid): their rows' member
//    lists are compacted and every member pair gets the deeper levels' limbs
//    with u64 atomics into a per-slot, per-level accumulator (typically no
//    row at all: synthetic lengths are multiples of 2^-52).
//
// The heavy kernel's epilogue adds the light (and deep) sums, forms t, d in
// exact integers and applies finalize (kernels.hpp:251-259).
#pragma once

#include <cstdint>

#include "bits.cuh"

namespace sf {

// ---- preparation ------------------------------------------------------------

// One warp per row: |S_e|, dense flag, and the sort key that puts the heavy
// rows first (stable radix sort: postorder kept among the heavy rows — subtree
// locality, 25% fewer nonzero words per column at the EMP shape — and among
// the light rows, whose key is 1).
__global__ void sp_row_key_kernel(const uint32_t* __restrict__ rows, int64_t stride, int32_t E,
                                  int32_t n, int32_t heavy_min, uint32_t* __restrict__ keys,
                                  int32_t* __restrict__ vals, uint8_t* __restrict__ dense,
                                  unsigned int* __restrict__ n_heavy, int32_t* __restrict__ mcount) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < E; r += nwarps) {
    const uint32_t* row = rows + r * stride;
    int m = 0;
    for (int64_t i = lane; i < stride; i += 32) m += __popc(__ldg(row + i));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m += __shfl_xor_sync(0xffffffffu, m, off);
    if (lane == 0) {
      const bool dn = 2 * m > n;
      const int x = dn ? n - m : m;
      keys[r] = x >= heavy_min ? 0u : 1u;
      vals[r] = static_cast<int32_t>(r);
      dense[r] = dn ? 1 : 0;
      mcount[r] = m;
      if (x >= heavy_min) atomicAdd(n_heavy, 1u);
    }
  }
}

// Exponent e_b of the factor the heavy walk builds for bit b of a 32-bit v
// half: the double whose high word is 1 << b (low word 0). b < 20: subnormal
// 2^(b-1042); 20 <= b <= 30: 2^(2^(b-20) - 1023); b = 31 is the sign bit
// (-0.0), so that bit uses the factor 2.0 = hi word 0x40000000 instead.
__host__ __device__ __forceinline__ int factor_exp(int b) {
  if (b < 20) return b - 1042;
  if (b < 31) return (1 << (b - 20)) - 1023;
  return 1;
}

// Limb value stored for the heavy walk: integer limb c (< 2^32) as c * 2^-52
// (so every accumulator is an exact multiple of 2^-52 below 2), divided by the
// bit's factor. c * 2^(-52 - e_b) is at most 2^32 * 2^990 and at least
// 2^-53 (b = 31), both normal doubles.
__device__ __forceinline__ double scaled_limb(unsigned long long c, int b) {
  return ldexp(static_cast<double>(c), -52 - factor_exp(b));
}

// Permuted row i <- original row perm[i]: dense mask, the pre-scaled limbs
// by bit position for the heavy walk, the integer limbs by bit position (for
// the column sums), and C = the dense rows' main-level limb sums.
__global__ void sp_perm_kernel(const int32_t* __restrict__ perm, int32_t E, int64_t rows_pad,
                               const uint8_t* __restrict__ dense, const unsigned long long* __restrict__ fix,
                               int32_t lo_bits, unsigned long long* __restrict__ dmask64,
                               double2* __restrict__ limbs, unsigned long long* __restrict__ fixbit,
                               unsigned long long* __restrict__ cacc) {
  const unsigned long long lo_mask = (1ull << lo_bits) - 1ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows_pad;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = 63 - static_cast<int>(i & 63);  // bit position in the 64-row word
    const int64_t slot = (i & ~int64_t{63}) + p;
    if (i >= E) {
      limbs[slot] = make_double2(0.0, 0.0);
      fixbit[slot] = 0ull;
      continue;
    }
    const int r = perm[i];
    const unsigned long long v = fix[r];
    const unsigned long long hi = v >> lo_bits, lo = v & lo_mask;
    limbs[slot] = make_double2(scaled_limb(hi, p & 31), scaled_limb(lo, p & 31));
    fixbit[slot] = v;
    if (dense[r]) {
      atomicOr(dmask64 + (i >> 6), 1ull << p);
      atomicAdd(cacc, hi);
      atomicAdd(cacc + 1, lo);
    }
  }
}

// Heavy words only: sample-packed rows -> node-packed X words of the permuted
// heavy rows (w < Hw). One warp per (word, 32-sample block).
__global__ void sp_transpose_kernel(const uint32_t* __restrict__ rows, int64_t stride,
                                    const int32_t* __restrict__ perm,
                                    const unsigned int* __restrict__ n_heavy, int32_t n,
                                    const unsigned long long* __restrict__ dmask64,
                                    unsigned long long* __restrict__ nx, int64_t n_ext) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t H = *n_heavy;
  const int64_t Hw = (H + 63) / 64;
  const int64_t blocks = Hw * stride;
  for (int64_t bidx = warp; bidx < blocks; bidx += nwarps) {
    const int64_t w = bidx / stride;
    const int64_t cb = bidx - w * stride;
    const int64_t r1 = 64 * w + lane, r2 = r1 + 32;
    const uint32_t a = r1 < H ? __ldg(rows + static_cast<int64_t>(perm[r1]) * stride + cb) : 0u;
    const uint32_t b = r2 < H ? __ldg(rows + static_cast<int64_t>(perm[r2]) * stride + cb) : 0u;
    unsigned long long out = 0ull;
#pragma unroll
    for (int bit = 0; bit < 32; ++bit) {
      const uint32_t v1 = __ballot_sync(0xffffffffu, (a >> bit) & 1u);
      const uint32_t v2 = __ballot_sync(0xffffffffu, (b >> bit) & 1u);
      if (bit == lane)
        out = (static_cast<unsigned long long>(__brev(v1)) << 32) | static_cast<unsigned long long>(__brev(v2));
    }
    const int64_t s = cb * 32 + lane;
    // complement only the heavy rows of the word: the light rows that share
    // its last word (dense ones included) must stay zero here
    const int64_t h = H - 64 * w;
    const unsigned long long heavy_bits = h >= 64 ? ~0ull : ~(~0ull >> h);
    if (s < n) nx[w * n_ext + s] = out ^ (dmask64[w] & heavy_bits);
  }
}

// Wrap columns of the heavy words: nx[w][c] = nx[w][c mod n], n <= c < n_ext.
__global__ void sp_extend_kernel(unsigned long long* __restrict__ nx, int64_t n_ext, int32_t n,
                                 const unsigned int* __restrict__ n_heavy) {
  const int64_t Hw = (static_cast<int64_t>(*n_heavy) + 63) / 64;
  const int64_t extra = n_ext - n;
  const int64_t total = Hw * extra;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / extra;
    const int64_t col = n + i % extra;
    nx[w * n_ext + col] = nx[w * n_ext + col % n];
  }
}

// Column sums over the heavy words: thread per column (coalesced over c).
// colsum layout [4][n] = x_hi, x_lo, p_hi, p_lo (p: rows that are not dense).
constexpr int kHeavyColSlices = 16;
__global__ void sp_heavy_colsum_kernel(const unsigned long long* __restrict__ nx, int64_t n_ext,
                                       int32_t n, const unsigned int* __restrict__ n_heavy,
                                       const unsigned long long* __restrict__ dmask64,
                                       const unsigned long long* __restrict__ fixbit, int32_t lo_bits,
                                       unsigned long long* __restrict__ colsum) {
  // thread per (column, slice of the heavy words): coalesced along the
  // columns, kHeavyColSlices partial sums per column (exact u64 atomics)
  const int64_t Hw = (static_cast<int64_t>(*n_heavy) + 63) / 64;
  const unsigned long long lo_mask = (1ull << lo_bits) - 1ull;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < kHeavyColSlices * n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t z = t / n, c = t - z * n;
    unsigned long long xh = 0, xl = 0, ph = 0, pl = 0;
    for (int64_t w = Hw * z / kHeavyColSlices; w < Hw * (z + 1) / kHeavyColSlices; ++w) {
      const unsigned long long x = __ldg(nx + w * n_ext + c);
      if (!x) continue;
      const unsigned long long dm = __ldg(dmask64 + w);
      unsigned long long b = x;
      while (b) {
        const int p = 63 - __clzll(static_cast<long long>(b));  // bit position
        const unsigned long long m = 1ull << p;
        b ^= m;
        const unsigned long long v = __ldg(fixbit + 64 * w + p);
        const unsigned long long h = v >> lo_bits, l = v & lo_mask;
        xh += h;
        xl += l;
        if (!(dm & m)) {
          ph += h;
          pl += l;
        }
      }
    }
    if (xh | xl) {
      atomicAdd(colsum + c, xh);
      atomicAdd(colsum + n + c, xl);
    }
    if (ph | pl) {
      atomicAdd(colsum + 2 * static_cast<int64_t>(n) + c, ph);
      atomicAdd(colsum + 3 * static_cast<int64_t>(n) + c, pl);
    }
  }
}

// ---- light rows ---------------------------------------------------------------

// Light sums are u64 limb pairs (hi, lo): every limb and partial sum is an
// integer below 2^53, so integer atomics are exact and order-free (measured
// as fast as fp64 atomic adds in L2: profiles/r01_ab_c3_light_u64_atomics.jsonl).
__device__ __forceinline__ void light_add(unsigned long long* cell, ulonglong2 L) {
  atomicAdd(cell, L.x);
  atomicAdd(cell + 1, L.y);
}

__device__ __forceinline__ ulonglong2 ilimbs_of(unsigned long long v, int lo_bits) {
  return make_ulonglong2(v >> lo_bits, v & ((1ull << lo_bits) - 1ull));
}

__device__ __forceinline__ void sp_add_pair(int a, int b, int n, int S, int s_begin, int s_end,
                                            ulonglong2 L, unsigned long long* __restrict__ gl,
                                            unsigned long long& pairs) {
  const int d = b - a;
  int s = d - 1;
  if (s < S && s >= s_begin && s < s_end) {
    light_add(gl + 2 * (static_cast<int64_t>(s - s_begin) * n + a), L);
    ++pairs;
  }
  s = n - d - 1;
  if (s < S && s >= s_begin && s < s_end) {
    light_add(gl + 2 * (static_cast<int64_t>(s - s_begin) * n + b), L);
    ++pairs;
  }
}

// One-shot light scatter (used when the banded form's u32/u16 indexing does
// not fit): one warp per light row, members listed in shared memory in sample
// order, every member pair's slot(s) in [s_begin, s_end) gets the limbs.
// Pair {a < b}, d = b - a: slot (s = d-1, k = a) when d-1 < S, and slot
// (s = n-d-1, k = b) when n-d-1 < S (both for d = n/2, n even: the
// reference's duplicated half stripe).
template <int NW, int MAXT>
__global__ void __launch_bounds__(32 * NW) sp_light_scatter_kernel(
    const uint32_t* __restrict__ rows, int64_t stride, int32_t E, int32_t n,
    const int32_t* __restrict__ perm, const unsigned int* __restrict__ n_heavy,
    const int32_t* __restrict__ mcount, const unsigned long long* __restrict__ fix, int32_t lo_bits,
    int32_t s_begin, int32_t s_end, unsigned long long* __restrict__ gl, unsigned long long* __restrict__ colsum,
    unsigned long long* __restrict__ pairs_out, int32_t list_cap) {
  extern __shared__ int32_t sp_members[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int32_t* mem = sp_members + static_cast<int64_t>(wib) * list_cap;
  const int S = n / 2;
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * NW + wib;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * NW;
  const uint32_t tail = (n & 31) ? ((1u << (n & 31)) - 1u) : 0xffffffffu;
  const int64_t H = *n_heavy;
  unsigned long long pairs = 0;
  for (int64_t idx = H + warp; idx < E; idx += nwarps) {
    const int r = perm[idx];
    const int m = mcount[r];
    const bool dense = 2 * m > n;
    const int x = dense ? n - m : m;
    if (x == 0) continue;  // adds nothing anywhere
    const uint32_t* row = rows + static_cast<int64_t>(r) * stride;
    int count = 0;
    for (int64_t base = 0; base < stride && count < x; base += 32) {
      const int64_t i = base + lane;
      uint32_t wd = 0u;
      if (i < stride) {
        wd = __ldg(row + i);
        if (dense) wd = ~wd & (i == stride - 1 ? tail : 0xffffffffu);
      }
      const int c = __popc(wd);
      int incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      int at = count + incl - c;
      while (wd) {
        const int b = __ffs(wd) - 1;
        wd &= wd - 1u;
        mem[at++] = static_cast<int32_t>(i * 32 + b);
      }
      count += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const ulonglong2 L = ilimbs_of(fix[r], lo_bits);
    for (int i = lane; colsum && i < x; i += 32) {  // colsum null on later passes
      const int c = mem[i];
      atomicAdd(colsum + c, L.x);
      atomicAdd(colsum + n + c, L.y);
      if (!dense) {
        atomicAdd(colsum + 2 * static_cast<int64_t>(n) + c, L.x);
        atomicAdd(colsum + 3 * static_cast<int64_t>(n) + c, L.y);
      }
    }
    if (x <= 32 * MAXT) {
      int bv[MAXT];
#pragma unroll
      for (int t = 0; t < MAXT; ++t) bv[t] = (lane + 32 * t < x) ? mem[lane + 32 * t] : 0;
      for (int i = 0; i + 1 < x; ++i) {
        const int a = mem[i];  // broadcast
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          const int j = lane + 32 * t;
          if (j > i && j < x) sp_add_pair(a, bv[t], n, S, s_begin, s_end, L, gl, pairs);
        }
      }
    } else {
      for (int i = 0; i + 1 < x; ++i) {
        const int a = mem[i];
        for (int j = i + 1 + lane; j < x; j += 32) sp_add_pair(a, mem[j], n, S, s_begin, s_end, L, gl, pairs);
      }
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) pairs += __shfl_down_sync(0xffffffffu, pairs, off);
  if (lane == 0 && pairs) atomicAdd(pairs_out, pairs);
}

// ---- Banded light scatter (default). The one-shot scatter sends each pair's
// atomics to a random sector of the whole (stripes x n) light-sum array
// (5 GB at C3): every atomic is an HBM read-modify-write (ncu: 2.3 TB/s of
// DRAM traffic, 5% issue). Here the member lists are compacted once (CSR,
// ascending samples), and the pairs are emitted band by band — a band is a
// (stripe range x column range) block of the light-sum array sized to stay
// resident in L2.

// Members per permuted position (0 for heavy rows): cnt[idx], idx < E.
__global__ void sp_light_count_kernel(const int32_t* __restrict__ perm, int32_t E, int32_t n,
                                      const unsigned int* __restrict__ n_heavy,
                                      const int32_t* __restrict__ mcount, uint32_t* __restrict__ cnt) {
  const int64_t H = *n_heavy;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= E;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t x = 0;
    if (i >= H && i < E) {
      const int m = mcount[perm[i]];
      x = static_cast<uint32_t>(2 * m > n ? n - m : m);
    }
    cnt[i] = x;
  }
}

// Warp-wide compaction of the members of X_e (row words, complemented when
// dense) into out[0, x), ascending; calls visit(sample) once per member.
template <class Visit>
__device__ __forceinline__ void list_members(const uint32_t* __restrict__ row, int64_t stride, bool dense,
                                             uint32_t tail, int x, int lane, int32_t* __restrict__ out,
                                             Visit visit) {
  int count = 0;
  for (int64_t base = 0; base < stride && count < x; base += 32) {
    const int64_t i = base + lane;
    uint32_t wd = 0u;
    if (i < stride) {
      wd = __ldg(row + i);
      if (dense) wd = ~wd & (i == stride - 1 ? tail : 0xffffffffu);
    }
    const int c = __popc(wd);
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    int at = count + incl - c;
    while (wd) {
      const int b = __ffs(wd) - 1;
      wd &= wd - 1u;
      const int smp = static_cast<int>(i * 32 + b);
      out[at++] = smp;
      visit(smp);
    }
    count += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// Members of every light row, ascending, at lmem[lptr[idx] ...]; the light
// rows' column sums are added here (once per run).
__global__ void sp_light_members_kernel(const uint32_t* __restrict__ rows, int64_t stride, int32_t E,
                                        int32_t n, const int32_t* __restrict__ perm,
                                        const unsigned int* __restrict__ n_heavy,
                                        const int32_t* __restrict__ mcount,
                                        const uint32_t* __restrict__ lptr,
                                        const unsigned long long* __restrict__ fix, int32_t lo_bits,
                                        int32_t* __restrict__ lmem, unsigned long long* __restrict__ colsum,
                                        int32_t gather_min) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t tail = (n & 31) ? ((1u << (n & 31)) - 1u) : 0xffffffffu;
  const int64_t H = *n_heavy;
  for (int64_t idx = H + warp; idx < E; idx += nwarps) {
    const int r = perm[idx];
    const int m = mcount[r];
    const bool dense = 2 * m > n;
    const int x = dense ? n - m : m;
    if (x == 0) continue;
    // rows with >= gather_min members reach the column sums through the
    // column entries (sp_light_colsum_kernel): no per-member atomics here
    if (x >= gather_min) {
      list_members(rows + static_cast<int64_t>(r) * stride, stride, dense, tail, x, lane, lmem + lptr[idx],
                   [](int) {});
      continue;
    }
    const ulonglong2 L = ilimbs_of(fix[r], lo_bits);
    list_members(rows + static_cast<int64_t>(r) * stride, stride, dense, tail, x, lane, lmem + lptr[idx],
                 [&](int smp) {
                   atomicAdd(colsum + smp, L.x);
                   atomicAdd(colsum + n + smp, L.y);
                   if (!dense) {
                     atomicAdd(colsum + 2 * static_cast<int64_t>(n) + smp, L.x);
                     atomicAdd(colsum + 3 * static_cast<int64_t>(n) + smp, L.y);
                   }
                 });
  }
}

// The light rows' column sums from the column entries (rows with >= 2
// members): warp per column, exact u64 limb sums, four atomics per column
// (the heavy rows and the single-member rows add theirs elsewhere).
__global__ void sp_light_colsum_kernel(const uint32_t* __restrict__ cptr, const uint2* __restrict__ cent,
                                       const int32_t* __restrict__ perm, const int32_t* __restrict__ mcount,
                                       const unsigned long long* __restrict__ fix, int32_t lo_bits, int32_t n,
                                       unsigned long long* __restrict__ colsum) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = warp; c < n; c += nwarps) {
    unsigned long long xh = 0, xl = 0, ph = 0, pl = 0;
    for (uint32_t e = cptr[c] + lane; e < cptr[c + 1]; e += 32) {
      const int r = perm[cent[e].x];
      const ulonglong2 L = ilimbs_of(fix[r], lo_bits);
      xh += L.x;
      xl += L.y;
      if (2 * mcount[r] <= n) {
        ph += L.x;
        pl += L.y;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      xh += __shfl_down_sync(0xffffffffu, xh, off);
      xl += __shfl_down_sync(0xffffffffu, xl, off);
      ph += __shfl_down_sync(0xffffffffu, ph, off);
      pl += __shfl_down_sync(0xffffffffu, pl, off);
    }
    if (lane == 0) {
      atomicAdd(colsum + c, xh);
      atomicAdd(colsum + n + c, xl);
      atomicAdd(colsum + 2 * static_cast<int64_t>(n) + c, ph);
      atomicAdd(colsum + 3 * static_cast<int64_t>(n) + c, pl);
    }
  }
}

// First index j in [lo, hi) with mem[j] >= key (mem ascending).
template <class M>
__device__ __forceinline__ int lower_bound_i32(const M* __restrict__ mem, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (static_cast<int>(mem[mid]) < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One band: slots with stripe in [s0, s1) and column in [k0, k1). gl rows are
// relative to the light pass start p0 (layout unchanged: (s - p0) * n + k).
// Every slot of a pair {a < b}, d = b - a, is owned by one member:
//   slot (s = d - 1,     k = a): a's partners above, b in [a + s0 + 1, a + se];
//   slot (s = n - d - 1, k = b): b's partners below, a in [b - n + 1 + s0, b - n + se].
// A member works only in the column band holding it, and both partner
// ranges move upward as the stripe bands advance, so two per-member cursors
// (u16, next partner index) replace the binary searches after the first band
// of a pass (FIRST: search, then store the cursors).
template <int NW, bool FIRST>
__global__ void __launch_bounds__(32 * NW) sp_light_band_kernel(
    const int32_t* __restrict__ perm, int32_t E, int32_t n, const unsigned int* __restrict__ n_heavy,
    const uint32_t* __restrict__ lptr, const int32_t* __restrict__ lmem, uint16_t* __restrict__ cur,
    const unsigned long long* __restrict__ fix, int32_t lo_bits, int32_t p0, int32_t s0, int32_t s1,
    int32_t k0, int32_t k1, unsigned long long* __restrict__ gl, unsigned long long* __restrict__ pairs_out,
    int32_t list_cap) {
  extern __shared__ int32_t sp_band_members[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int32_t* mem = sp_band_members + static_cast<int64_t>(wib) * list_cap;
  const int S = n / 2;
  const int se = min(s1, S);  // stripes past S do not exist
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * NW + wib;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * NW;
  const int64_t H = *n_heavy;
  unsigned long long pairs = 0;
  for (int64_t idx = H + warp; idx < E; idx += nwarps) {
    const uint32_t b0 = lptr[idx];
    const int x = static_cast<int>(lptr[idx + 1] - b0);
    if (x < 2) continue;
    for (int i = lane; i < x; i += 32) mem[i] = __ldg(lmem + b0 + i);
    __syncwarp();
    const ulonglong2 L = ilimbs_of(fix[perm[idx]], lo_bits);
    uint16_t* c = cur + 2 * static_cast<int64_t>(b0);
    for (int i = lane; i < x; i += 32) {
      const int a = mem[i];
      if (a < k0 || a >= k1) continue;
      int j1, j2;
      if (FIRST) {
        j1 = lower_bound_i32(mem, i + 1, x, a + s0 + 1);
        j2 = lower_bound_i32(mem, 0, i, a - n + 1 + s0);
      } else {
        const uint32_t cc = reinterpret_cast<const uint32_t*>(c)[i];
        j1 = static_cast<int>(cc & 0xffffu);
        j2 = static_cast<int>(cc >> 16);
      }
      // partners above: slot (b - a - 1, a)
      for (; j1 < x && mem[j1] <= a + se; ++j1) {
        const int s = mem[j1] - a - 1;
        light_add(gl + 2 * (static_cast<int64_t>(s - p0) * n + a), L);
        ++pairs;
      }
      // partners below: slot (n - (a - a') - 1, a)
      for (; j2 < i && mem[j2] <= a - n + se; ++j2) {
        const int s = n - (a - mem[j2]) - 1;
        light_add(gl + 2 * (static_cast<int64_t>(s - p0) * n + a), L);
        ++pairs;
      }
      reinterpret_cast<uint32_t*>(c)[i] = static_cast<uint32_t>(j1) | (static_cast<uint32_t>(j2) << 16);
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) pairs += __shfl_down_sync(0xffffffffu, pairs, off);
  if (lane == 0 && pairs) atomicAdd(pairs_out, pairs);
}

// ---- Column-owned light scatter (default). Every slot (s, k) of a light
// pair is owned by one member, the column k (slot (b - a - 1, a) by a for its
// partners above, slot (n - (a - b) - 1, a) by a for its partners below), so
// one CTA per column can accumulate all of that column's light sums in
// shared memory: the light rows containing the column are its entries (a
// column-major CSR of the light member lists), each entry walks its row's
// sorted members from its own position — partners above while the stripe is
// below the window's end, partners below from the start of the list — and
// the window (up to kLightWin stripes of (hi, lo) limbs) is written to the
// light-sum array once. No global atomics; the limb sums are exact integers,
// so the order of the shared-memory atomics does not change the bits.
#ifndef SF_LIGHT_WIN
#define SF_LIGHT_WIN 12800
#endif
#ifndef SF_LIGHT_UNROLL
#define SF_LIGHT_UNROLL 4
#endif
constexpr int kLightWin = SF_LIGHT_WIN;        // stripes per shared-memory window (16 B each)
// a column entry is read once per window: streaming (evict-first) load
__device__ __forceinline__ uint2 ld_entry(const uint2* p) {
#if SF_LIGHT_STREAM
  return __ldcs(p);
#else
  return *p;
#endif
}
constexpr int kLightUnroll = SF_LIGHT_UNROLL;  // member loads in flight per lane
#ifndef SF_LIGHT_CHUNK
#define SF_LIGHT_CHUNK 1  // three 21-bit limbs for all columns, carries folded per entry chunk (0: limb mode by entry count)
#endif


// 16-bit copy of the light member lists (n <= 65536) for the column kernel.
__global__ void sp_narrow_members_kernel(const int32_t* __restrict__ lmem, const uint32_t* __restrict__ total,
                                         uint16_t* __restrict__ lmem16) {
  const uint32_t m = *total;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    lmem16[i] = static_cast<uint16_t>(lmem[i]);
}

// Entries per column: one count per light member (rows with >= 2 members).
__global__ void sp_col_count_kernel(const int32_t* __restrict__ lmem, const uint32_t* __restrict__ lptr,
                                    int32_t E, const unsigned int* __restrict__ n_heavy,
                                    uint32_t* __restrict__ ccnt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t idx = *n_heavy + warp; idx < E; idx += nwarps) {
    const uint32_t b0 = lptr[idx];
    const int x = static_cast<int>(lptr[idx + 1] - b0);
    if (x < 2) continue;
    for (int i = lane; i < x; i += 32) atomicAdd(ccnt + lmem[b0 + i], 1u);
  }
}

// Column entries: (permuted light row idx, position of the column in the
// row's member list). Warp per light row, one claim per member.
__global__ void sp_col_fill_kernel(const int32_t* __restrict__ lmem, const uint32_t* __restrict__ lptr,
                                   int32_t E, const unsigned int* __restrict__ n_heavy,
                                   uint32_t* __restrict__ cfill, uint2* __restrict__ cent) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t idx = *n_heavy + warp; idx < E; idx += nwarps) {
    const uint32_t b0 = lptr[idx];
    const int x = static_cast<int>(lptr[idx + 1] - b0);
    if (x < 2) continue;  // no pair
    for (int i = lane; i < x; i += 32) {
      const uint32_t pos = atomicAdd(cfill + lmem[b0 + i], 1u);
      cent[pos] = make_uint2(static_cast<uint32_t>(idx), static_cast<uint32_t>(i));
    }
  }
}

// One light contribution into the shared-memory window, planes of
// kLightWin cells (structure of arrays: the cells of different stripes fall
// in different banks). The row's value v (< 2^63) goes in as limbs into
// 32-bit native shared atomic adds, exact while no cell overflows: a cell
// takes one addition per light row holding the column, so MODE 0 (three
// 21-bit limbs) is exact for up to 2048 entries — the column kernel walks
// longer columns in chunks of 2048 entries and folds the planes' carries
// into a fourth plane between chunks (SF_LIGHT_CHUNK, default). MODE 1
// (four 16-bit limbs, <= 65535 entries) and MODE 2 ((hi, lo) limbs with
// 64-bit compare-and-swap adds, any count) are the unchunked alternatives
// (SF_LIGHT_CHUNK=0, or the SF_LIGHT_LIMB_MODE test hook). The kernel is
// bound by these atomics (L1 data pipe, profiles/r02_ncu_light_column_c3_v3.txt):
// three limbs instead of four is 2.6% of the C3 step.
template <int MODE>
__device__ __forceinline__ void window_add(uint32_t* acc, int cell, unsigned long long v, ulonglong2 L) {
  if (MODE == 2) {
    unsigned long long* a64 = reinterpret_cast<unsigned long long*>(acc);
    atomicAdd(a64 + cell, L.x);
    atomicAdd(a64 + kLightWin + cell, L.y);
  } else if (MODE == 1) {
    atomicAdd(acc + cell, static_cast<uint32_t>(v & 0xffffu));
    atomicAdd(acc + kLightWin + cell, static_cast<uint32_t>((v >> 16) & 0xffffu));
    atomicAdd(acc + 2 * kLightWin + cell, static_cast<uint32_t>((v >> 32) & 0xffffu));
    atomicAdd(acc + 3 * kLightWin + cell, static_cast<uint32_t>(v >> 48));
  } else {
    atomicAdd(acc + cell, static_cast<uint32_t>(v & 0x1fffffu));
    atomicAdd(acc + kLightWin + cell, static_cast<uint32_t>((v >> 21) & 0x1fffffu));
    atomicAdd(acc + 2 * kLightWin + cell, static_cast<uint32_t>(v >> 42));
  }
}

// The window cell's exact sum as (hi, lo) with hi * 2^lo_bits + lo = sum.
template <int MODE>
__device__ __forceinline__ ulonglong2 window_cell(const uint32_t* acc, int cell, int lo_bits) {
  if (MODE == 2) {
    const unsigned long long* a64 = reinterpret_cast<const unsigned long long*>(acc);
    return make_ulonglong2(a64[cell], a64[kLightWin + cell]);
  }
  unsigned __int128 v;
  if (MODE == 1)
    v = static_cast<unsigned __int128>(acc[cell]) + (static_cast<unsigned __int128>(acc[kLightWin + cell]) << 16) +
        (static_cast<unsigned __int128>(acc[2 * kLightWin + cell]) << 32) +
        (static_cast<unsigned __int128>(acc[3 * kLightWin + cell]) << 48);
  else  // three 21-bit limbs and the folded carries (zero without chunks)
    v = static_cast<unsigned __int128>(acc[cell]) + (static_cast<unsigned __int128>(acc[kLightWin + cell]) << 21) +
        (static_cast<unsigned __int128>(acc[2 * kLightWin + cell]) << 42) +
        (static_cast<unsigned __int128>(acc[3 * kLightWin + cell]) << 63);
  return make_ulonglong2(static_cast<unsigned long long>(v >> lo_bits),
                         static_cast<unsigned long long>(v) & ((1ull << lo_bits) - 1ull));
}

// Per light row (by permuted index): member list offset and length, and its
// main-level value — one 16-byte record, L2-resident (C3: ~8 MB).
struct LightRowInfo {
  uint32_t b0, x;
  unsigned long long v;
};

__global__ void sp_light_rowinfo_kernel(const int32_t* __restrict__ perm, int32_t E,
                                        const unsigned int* __restrict__ n_heavy, const uint32_t* __restrict__ lptr,
                                        const unsigned long long* __restrict__ fix, LightRowInfo* __restrict__ info) {
  for (int64_t idx = *n_heavy + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < E;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
    info[idx] = LightRowInfo{lptr[idx], lptr[idx + 1] - lptr[idx], fix[perm[idx]]};
}

// One warp per entry (light row holding the column): the lanes walk the
// row's sorted members 32 at a time from the entry's own position. The next
// entry's record is loaded while the current one is walked.
template <int MODE, class M>
__device__ __forceinline__ void light_column_window(const uint32_t e0, const uint32_t e1, const uint2* __restrict__ cent,
                                                    const LightRowInfo* __restrict__ info,
                                                    const M* __restrict__ lmem, int32_t lo_bits, int k, int n,
                                                    int w0, int w1, uint32_t* __restrict__ acc,
                                                    unsigned long long& pairs) {
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t e = e0 + wid;
  uint2 en = e < e1 ? ld_entry(cent + e) : make_uint2(0u, 0u);
  LightRowInfo ri{0u, 0u, 0ull};
  if (e < e1) ri = info[en.x];
  for (; e < e1; e += nw) {
    // prefetch the next entry of this warp
    const uint32_t en_next = e + nw;
    uint2 nen = make_uint2(0u, 0u);
    if (en_next < e1) nen = ld_entry(cent + en_next);
    const int x = static_cast<int>(ri.x);
    const int i = static_cast<int>(en.y);
    const M* mem = lmem + ri.b0;
    const unsigned long long v = ri.v;
    const ulonglong2 L = ilimbs_of(v, lo_bits);
    // partners above: slot (b - k - 1, k), b in [k + w0 + 1, k + w1]; the
    // member loads are issued kUnroll x 32 at a time (the kernel is bound by
    // their latency: each row's list is read once per member column)
    int j0 = w0 > 0 ? lower_bound_i32(mem, i + 1, x, k + w0 + 1) : i + 1;
    for (int jb = j0;; jb += 32 * kLightUnroll) {
      int s[kLightUnroll];
#pragma unroll
      for (int u = 0; u < kLightUnroll; ++u) {
        const int j = jb + lane + 32 * u;
        s[u] = j < x ? static_cast<int>(__ldg(mem + j)) - k - 1 : w1;
      }
      bool all_live = true;
#pragma unroll
      for (int u = 0; u < kLightUnroll; ++u) {
        const bool live = s[u] < w1;
        all_live = all_live && live;
        if (live) {
          window_add<MODE>(acc, s[u] - w0, v, L);
          ++pairs;
        }
      }
      if (!__all_sync(0xffffffffu, all_live)) break;  // sorted: later members are past the window
    }
    // partners below: slot (n - (k - b) - 1, k), b in [k - n + 1 + w0, k - n + w1]
    j0 = w0 > 0 ? lower_bound_i32(mem, 0, i, k - n + 1 + w0) : 0;
    for (int jb = j0;; jb += 32 * kLightUnroll) {
      int s[kLightUnroll];
#pragma unroll
      for (int u = 0; u < kLightUnroll; ++u) {
        const int j = jb + lane + 32 * u;
        s[u] = j < i ? n - (k - static_cast<int>(__ldg(mem + j))) - 1 : w1;
      }
      bool all_live = true;
#pragma unroll
      for (int u = 0; u < kLightUnroll; ++u) {
        const bool live = s[u] < w1;
        all_live = all_live && live;
        if (live) {
          window_add<MODE>(acc, s[u] - w0, v, L);
          ++pairs;
        }
      }
      if (!__all_sync(0xffffffffu, all_live)) break;
    }
    en = nen;
    if (en_next < e1) ri = info[en.x];
  }
}

// One CTA per column k: stripes [s0, s1) of the light sums (rows relative to
// the pass start p0), in windows of kLightWin stripes.
// M: the member type, uint16_t when n <= 65536 (half the bytes of the
// member lists each column re-reads: the kernel is bound by those reads).
template <int NT, class M>
__global__ void __launch_bounds__(NT) sp_light_column_kernel(
    const uint32_t* __restrict__ cptr, const uint2* __restrict__ cent, const LightRowInfo* __restrict__ info,
    const M* __restrict__ lmem, int32_t lo_bits, int32_t n, int32_t k_begin, int32_t k_end, int32_t p0,
    int32_t s0, int32_t s1, unsigned long long* __restrict__ gl, unsigned long long* __restrict__ pairs_out,
    int32_t min_mode, int32_t chunk) {
  extern __shared__ uint32_t lacc[];  // 4 planes of kLightWin u32 cells (or 2 of u64)
  const int S = n / 2;
  const int send = min(s1, S);
  unsigned long long pairs = 0;
  for (int k = k_begin + blockIdx.x; k < k_end; k += gridDim.x) {
    const uint32_t e0 = cptr[k], e1 = cptr[k + 1];
#if SF_LIGHT_CHUNK
    // three 21-bit limbs for every column: entries in chunks of <= 2048 (one
    // addition per entry per cell keeps every plane below 2^32), the planes'
    // carries folded into the fourth plane between chunks
    const int mode = min_mode;  // test hook: 1 / 2 select the wide limb modes
    const uint32_t step = mode == 0 ? static_cast<uint32_t>(chunk) : 0xffffffffu;
#else
    // one addition per entry per cell: pick the narrowest exact limb mode
    const int mode = max(min_mode, e1 - e0 <= 2048u ? 0 : e1 - e0 <= 65535u ? 1 : 2);
    const uint32_t step = 0xffffffffu;
#endif
    for (int w0 = s0; w0 < send; w0 += kLightWin) {
      const int w1 = min(send, w0 + kLightWin);
      const int ww = w1 - w0;
      for (int t = threadIdx.x; t < 4 * kLightWin; t += NT) lacc[t] = 0u;
      __syncthreads();
      for (uint32_t c0 = e0;;) {
        const uint32_t c1 = e1 - c0 > step ? c0 + step : e1;
        if (mode == 0)
          light_column_window<0, M>(c0, c1, cent, info, lmem, lo_bits, k, n, w0, w1, lacc, pairs);
        else if (mode == 1)
          light_column_window<1, M>(c0, c1, cent, info, lmem, lo_bits, k, n, w0, w1, lacc, pairs);
        else
          light_column_window<2, M>(c0, c1, cent, info, lmem, lo_bits, k, n, w0, w1, lacc, pairs);
        __syncthreads();
        if (c1 >= e1) break;
        for (int t = threadIdx.x; t < ww; t += NT) {  // fold the carries before the next chunk
          uint32_t a0 = lacc[t], a1 = lacc[kLightWin + t], a2 = lacc[2 * kLightWin + t];
          a1 += a0 >> 21;
          a2 += a1 >> 21;
          lacc[t] = a0 & 0x1fffffu;
          lacc[kLightWin + t] = a1 & 0x1fffffu;
          lacc[2 * kLightWin + t] = a2 & 0x1fffffu;
          lacc[3 * kLightWin + t] += a2 >> 21;
        }
        __syncthreads();
        c0 = c1;
      }
      for (int t = threadIdx.x; t < ww; t += NT) {
        const ulonglong2 out = mode == 0 ? window_cell<0>(lacc, t, lo_bits)
                                         : mode == 1 ? window_cell<1>(lacc, t, lo_bits) : window_cell<2>(lacc, t, lo_bits);
        ulonglong2* cell = reinterpret_cast<ulonglong2*>(gl) + static_cast<int64_t>(w0 + t - p0) * n + k;
#if SF_LIGHT_STREAM
        // written once, read once by the epilogue much later: streaming
        // stores keep the 5 GB of light sums from evicting the member lists
        __stcs(reinterpret_cast<longlong2*>(cell), make_longlong2(static_cast<long long>(out.x),
                                                                   static_cast<long long>(out.y)));
#else
        *cell = out;
#endif
      }
      __syncthreads();
    }
  }
  for (int off = 16; off > 0; off >>= 1) pairs += __shfl_down_sync(0xffffffffu, pairs, off);
  if ((threadIdx.x & 31) == 0 && pairs) atomicAdd(pairs_out, pairs);
}

// ---- deeper fixed-point levels ---------------------------------------------------
// drows[i] (original row ids, i < R) are the rows with a nonzero value below
// the main level; dfix[i * (J-1) + (j-1)] their level-j values (j >= 1).

__global__ void sp_deep_count_kernel(const int32_t* __restrict__ drows, int32_t R, int32_t n,
                                     const int32_t* __restrict__ mcount, uint32_t* __restrict__ cnt) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= R;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t x = 0;
    if (i < R) {
      const int m = mcount[drows[i]];
      x = static_cast<uint32_t>(2 * m > n ? n - m : m);
    }
    cnt[i] = x;
  }
}

// Members of every deep row at dmem[dptr[i] ...] (ascending), the owning deep
// row of every entry, and the deeper levels' column sums and dense totals:
// dcolsum [J-1][4][n] as colsum, dcacc [J-1][2].
__global__ void sp_deep_members_kernel(const uint32_t* __restrict__ rows, int64_t stride, int32_t n,
                                       const int32_t* __restrict__ drows, int32_t R,
                                       const int32_t* __restrict__ mcount, const uint32_t* __restrict__ dptr,
                                       const unsigned long long* __restrict__ dfix, int32_t J, int32_t lo_bits,
                                       int32_t* __restrict__ dmem, uint32_t* __restrict__ dent,
                                       unsigned long long* __restrict__ dcolsum,
                                       unsigned long long* __restrict__ dcacc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t tail = (n & 31) ? ((1u << (n & 31)) - 1u) : 0xffffffffu;
  const int64_t n4 = 4 * static_cast<int64_t>(n);
  for (int64_t i = warp; i < R; i += nwarps) {
    const int r = drows[i];
    const int m = mcount[r];
    const bool dense = 2 * m > n;
    const int x = dense ? n - m : m;
    const unsigned long long* v = dfix + i * (J - 1);
    if (dense && lane < J - 1) {
      const ulonglong2 L = ilimbs_of(v[lane], lo_bits);
      atomicAdd(dcacc + 2 * lane, L.x);
      atomicAdd(dcacc + 2 * lane + 1, L.y);
    }
    const uint32_t b0 = dptr[i];
    for (int q = lane; q < x; q += 32) dent[b0 + q] = static_cast<uint32_t>(i);
    if (x == 0) continue;
    list_members(rows + static_cast<int64_t>(r) * stride, stride, dense, tail, x, lane, dmem + b0, [&](int smp) {
      for (int j = 0; j < J - 1; ++j) {
        if (!v[j]) continue;
        const ulonglong2 L = ilimbs_of(v[j], lo_bits);
        unsigned long long* cs = dcolsum + j * n4;
        atomicAdd(cs + smp, L.x);
        atomicAdd(cs + n + smp, L.y);
        if (!dense) {
          atomicAdd(cs + 2 * static_cast<int64_t>(n) + smp, L.x);
          atomicAdd(cs + 3 * static_cast<int64_t>(n) + smp, L.y);
        }
      }
    });
  }
}

__device__ __forceinline__ void deep_add(unsigned long long* __restrict__ dacc, int64_t cell, int32_t J,
                                         const unsigned long long* __restrict__ v, int lo_bits) {
  for (int j = 0; j < J - 1; ++j) {
    if (!v[j]) continue;
    light_add(dacc + 2 * (cell * (J - 1) + j), ilimbs_of(v[j], lo_bits));
  }
}

// Warp per deep-row member entry a, lanes over its partners above (b after
// a in the row's sorted list): both slots of the pair as in sp_add_pair, the
// deeper levels' limbs into dacc [(s - s_begin) * n + k][J-1] (hi, lo). (A
// thread per entry walked up to a whole row alone: rows of thousands of
// members serialised the kernel.)
__global__ void sp_deep_scatter_kernel(const uint32_t* __restrict__ dptr, const int32_t* __restrict__ dmem,
                                       const uint32_t* __restrict__ dent, int64_t M,
                                       const unsigned long long* __restrict__ dfix, int32_t J, int32_t lo_bits,
                                       int32_t n, int32_t s_begin, int32_t s_end,
                                       unsigned long long* __restrict__ dacc) {
  const int S = n / 2;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t g = warp; g < M; g += nwarps) {
    const uint32_t i = dent[g];
    const int64_t end = dptr[i + 1];
    const unsigned long long* v = dfix + static_cast<int64_t>(i) * (J - 1);
    const int a = dmem[g];
    for (int64_t q = g + 1 + lane; q < end; q += 32) {
      const int b = __ldg(dmem + q);
      const int d = b - a;
      int s = d - 1;
      if (s < S && s >= s_begin && s < s_end) deep_add(dacc, static_cast<int64_t>(s - s_begin) * n + a, J, v, lo_bits);
      s = n - d - 1;
      if (s < S && s >= s_begin && s < s_end) deep_add(dacc, static_cast<int64_t>(s - s_begin) * n + b, J, v, lo_bits);
    }
  }
}

// ---- heavy walk + epilogue ----------------------------------------------------------

struct SplitArgs {
  const unsigned long long* nx;      // [Hw][n_ext] heavy X words
  const double2* limbs;              // permuted heavy rows, by bit position, pre-scaled (scaled_limb)
  const unsigned int* n_heavy;
  unsigned long long* gl;            // light sums per slot (hi, lo limbs, u64); deep levels: G out
  const unsigned long long* colsum;  // [4][n]
  const unsigned long long* cacc;    // [2]
  const unsigned long long* dacc;    // deeper levels: [(s - gl_begin) * n + k][J-1] (hi, lo)
  const unsigned long long* dcolsum; // [J-1][4][n]
  const unsigned long long* dcacc;   // [J-1][2]
  int64_t n_ext;
  int32_t n;
  int32_t s_begin, s_end;  // stripes computed by this launch
  int32_t out_begin;       // stripe held by row 0 of dist / tot
  int32_t gl_begin;        // stripe held by row 0 of gl / dacc (the light-sum pass)
  int32_t lo_bits, scale, finalize;
  int32_t levels, vb;      // fixed-point levels (1: every length on the main grid), bits per level
  int32_t k_begin = 0, k_end = 0;  // sp_deep_epilogue_kernel: columns of this launch
  void* dist;
  void* tot;
  unsigned long long* counters;  // [0] slot x u-bit FMA pairs (+ light pairs, added by host), [1] fp64 ops
};

// One 32-bit half of a heavy u word, two bits per step, branch-free: per
// bit and slot one LOP3 (v & m, the factor's high word) and two DFMA. The
// factors of FG slots are formed before their DFMAs, so a DFMA does not wait
// on the LOP3 just before it.
template <int V, int FG>
__device__ __forceinline__ void heavy_half(uint32_t hu, const double2* __restrict__ Lb,
                                           const uint32_t (&vv)[V], double (&gh)[V], double (&gl)[V]) {
  static_assert(V % FG == 0, "factor groups must tile the slots");
  if (hu & 0x80000000u) {  // sign bit: factor 2.0 from the bit shifted to 30
    const double2 L = __ldg(Lb + 31);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const double f = __hiloint2double(static_cast<int>((vv[i] >> 1) & 0x40000000u), 0);
      gh[i] = fma(L.x, f, gh[i]);
      gl[i] = fma(L.y, f, gl[i]);
    }
    hu &= 0x7fffffffu;
  }
  while (hu) {
    const int b1 = msb_pos(hu);
    const uint32_t m1 = 1u << b1;
    hu ^= m1;
    const int b2 = msb_pos(hu | 1u);
    const uint32_t m2 = hu ? (1u << b2) : 0u;
    hu ^= m2;
    const double2 L1 = __ldg(Lb + b1);
    const double2 L2 = __ldg(Lb + b2);
#pragma unroll
    for (int i0 = 0; i0 < V; i0 += FG) {
      double f1[FG], f2[FG];
#pragma unroll
      for (int j = 0; j < FG; ++j) {
        f1[j] = __hiloint2double(static_cast<int>(vv[i0 + j] & m1), 0);
        f2[j] = __hiloint2double(static_cast<int>(vv[i0 + j] & m2), 0);
      }
#pragma unroll
      for (int j = 0; j < FG; ++j) {
        gh[i0 + j] = fma(L1.x, f1[j], gh[i0 + j]);
        gl[i0 + j] = fma(L1.y, f1[j], gl[i0 + j]);
      }
#pragma unroll
      for (int j = 0; j < FG; ++j) {
        gh[i0 + j] = fma(L2.x, f2[j], gh[i0 + j]);
        gl[i0 + j] = fma(L2.y, f2[j], gl[i0 + j]);
      }
    }
  }
}

// Exact t and d of one slot at fixed-point level j >= 1 (128-bit integers).
__device__ __forceinline__ void deep_level_td(const SplitArgs& a, int j, int64_t cell, int k, int lm, __int128& tv,
                                              __int128& dv) {
  const int n = a.n;
  const unsigned long long* xs = a.dcolsum + static_cast<int64_t>(j - 1) * 4 * n;
  const ulonglong2 G = reinterpret_cast<const ulonglong2*>(a.dacc)[cell * (a.levels - 1) + (j - 1)];
  const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm] + a.dcacc[2 * (j - 1)] - G.x);
  const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm] + a.dcacc[2 * (j - 1) + 1] - G.y);
  const long long dh = static_cast<long long>(xs[k] + xs[lm] - 2 * G.x);
  const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm] - 2 * G.y);
  tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
  dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
}

// sum_j V_j 2^-(scale + vb j) over the slot's levels, correctly rounded:
// carries are normalized from the deepest level up (every level's value is
// non-negative), then the leading 64+ bits are gathered from the first
// nonzero digit down, with a sticky bit for the rest.
template <class Real>
__device__ Real combine_levels(const SplitArgs& a, __int128 V0, bool is_t, int64_t cell, int k, int lm) {
  constexpr int kMaxLevels = 40;
  unsigned long long dig[kMaxLevels];
  const int J = a.levels;
  const unsigned __int128 mask = (static_cast<unsigned __int128>(1) << a.vb) - 1;
  unsigned __int128 carry = 0;
  for (int j = J - 1; j >= 1; --j) {
    __int128 tv, dv;
    deep_level_td(a, j, cell, k, lm, tv, dv);
    const unsigned __int128 x = static_cast<unsigned __int128>(is_t ? tv : dv) + carry;
    dig[j] = static_cast<unsigned long long>(x & mask);
    carry = x >> a.vb;
  }
  unsigned __int128 acc = static_cast<unsigned __int128>(V0) + carry;
  int e = 0;  // acc's unit is 2^-(scale + vb e)
  bool sticky = false;
  for (int j = 1; j < J; ++j) {
    if ((acc >> 64) == 0) {
      acc = (acc << a.vb) | dig[j];
      e = j;
    } else if (dig[j]) {
      sticky = true;
    }
  }
  return u128_to_real<Real>(acc, sticky, -(a.scale + a.vb * e));
}

// Epilogue when some length has deeper levels: the heavy kernel left the
// slot's main-level pair sum G (hi, lo limbs as int64) in its light-sum cell.
template <class Real>
__global__ void sp_deep_epilogue_kernel(const SplitArgs a) {
  const int n = a.n;
  const int kw = a.k_end - a.k_begin;
  const int64_t total = static_cast<int64_t>(a.s_end - a.s_begin) * kw;
  const unsigned long long* xs = a.colsum;
  const long long ch = static_cast<long long>(a.cacc[0]);
  const long long cl = static_cast<long long>(a.cacc[1]);
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = a.s_begin + static_cast<int>(i / kw);
    const int k = a.k_begin + static_cast<int>(i % kw);
    const int lm = static_cast<int>((static_cast<int64_t>(k) + s + 1) % n);
    const int64_t cell = static_cast<int64_t>(s - a.gl_begin) * n + k;
    const longlong2 G = reinterpret_cast<const longlong2*>(a.gl)[cell];
    const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - G.x;
    const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - G.y;
    const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * G.x;
    const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * G.y;
    const Real t = combine_levels<Real>(a, (static_cast<__int128>(th) << a.lo_bits) + tl, true, cell, k, lm);
    Real d = combine_levels<Real>(a, (static_cast<__int128>(dh) << a.lo_bits) + dl, false, cell, k, lm);
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    const int64_t off = static_cast<int64_t>(s - a.out_begin) * n + k;
    dist[off] = d;
    tot[off] = t;
  }
}

// Warp tile: UC consecutive u columns k0 .. k0+UC-1 x the 32 V v columns
// l = k0 + s0 + 1 + lane + 32 i (i < V). Slot (k0 + c, l) is stripe
// s = s0 + lane + 32 i - c, so a tile's stripes shift by one per u column:
// the grid's y tiles cover [s_begin - UC + 1, s_end) and slots outside
// [s_begin, s_end) are computed but not written. Every v word a lane loads
// serves UC u columns.
template <class Real, int V, int UC, int NW, int MINB, int FG>
__global__ void __launch_bounds__(32 * NW, MINB) stripe_split_kernel(const SplitArgs a) {
  const int lane = threadIdx.x & 31;
  const int k0 = (blockIdx.x * NW + (threadIdx.x >> 5)) * UC;
  const int n = a.n;
  if (k0 >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * V;
  const int64_t n_ext = a.n_ext;
  const int Hw = static_cast<int>((*a.n_heavy + 63u) / 64u);
  // v column of slot i: l0 + 32 i (< n_ext for every i: n_ext covers a whole
  // tile past the last stripe, so dead slots read real words and are dropped)
  const int64_t l0 = static_cast<int64_t>(k0) + s0 + 1 + lane;
  int nvalid[UC];
  int wvalid[UC];
#pragma unroll
  for (int c = 0; c < UC; ++c) {
    nvalid[c] = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int s = s0 + lane + 32 * i - c;
      nvalid[c] += (k0 + c < n && s >= a.s_begin && s < a.s_end) ? 1 : 0;
    }
    wvalid[c] = __reduce_add_sync(0xffffffffu, nvalid[c]);  // live slots of the warp in column c
  }
  unsigned long long work = 0;  // sum over columns of u bits x live slots

  double gh[UC][V], gl[UC][V];
#pragma unroll
  for (int c = 0; c < UC; ++c)
#pragma unroll
    for (int i = 0; i < V; ++i) {
      gh[c][i] = 0.0;
      gl[c][i] = 0.0;
    }
#pragma unroll 1
  for (int w = 0; w < Hw; ++w) {
    const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
    unsigned long long u[UC];
    unsigned long long any = 0ull;
#pragma unroll
    for (int c = 0; c < UC; ++c) {
      u[c] = k0 + c < n ? __ldg(row + k0 + c) : 0ull;
      any |= u[c];
    }
    if (any == 0ull) continue;
    const double2* Lw = a.limbs + 64 * static_cast<int64_t>(w);
#pragma unroll
    for (int c = 0; c < UC; ++c) work += static_cast<unsigned long long>(__popcll(u[c])) * wvalid[c];
    // one 32-bit half of the v words live at a time (fewer registers)
    const uint32_t* row32 = reinterpret_cast<const uint32_t*>(row);
    uint32_t vv[V];
    if (static_cast<uint32_t>(any >> 32)) {
#pragma unroll
      for (int i = 0; i < V; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i) + 1);
#pragma unroll
      for (int c = 0; c < UC; ++c)
        if (static_cast<uint32_t>(u[c] >> 32)) heavy_half<V, FG>(static_cast<uint32_t>(u[c] >> 32), Lw + 32, vv, gh[c], gl[c]);
    }
    if (static_cast<uint32_t>(any)) {
#pragma unroll
      for (int i = 0; i < V; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i));
#pragma unroll
      for (int c = 0; c < UC; ++c)
        if (static_cast<uint32_t>(u[c])) heavy_half<V, FG>(static_cast<uint32_t>(u[c]), Lw, vv, gh[c], gl[c]);
    }
  }

  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;
  const long long ch = static_cast<long long>(a.cacc[0]);
  const long long cl = static_cast<long long>(a.cacc[1]);
#pragma unroll
  for (int c = 0; c < UC; ++c) {
    const int k = k0 + c;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int s = s0 + lane + 32 * i - c;
      if (k >= n || s < a.s_begin || s >= a.s_end) continue;
      const int64_t li = l0 + 32 * i;
      const int lm = li >= n ? static_cast<int>(li - n) : static_cast<int>(li);
      const int64_t off = static_cast<int64_t>(s - a.out_begin) * n + k;
      const int64_t cell = static_cast<int64_t>(s - a.gl_begin) * n + k;
      const ulonglong2 light = reinterpret_cast<const ulonglong2*>(a.gl)[cell];
      // accumulators hold exact multiples of 2^-52 below 2
      const long long Gh_ = __double2ll_rn(gh[c][i] * 0x1p52) + static_cast<long long>(light.x);
      const long long Gl_ = __double2ll_rn(gl[c][i] * 0x1p52) + static_cast<long long>(light.y);
      if (a.levels > 1) {  // sp_deep_epilogue_kernel finishes the slot
        reinterpret_cast<longlong2*>(a.gl)[cell] = make_longlong2(Gh_, Gl_);
        continue;
      }
      const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - Gh_;
      const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - Gl_;
      const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * Gh_;
      const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * Gl_;
      const __int128 tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
      const __int128 dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
      const Real t = fixed_to_real<Real>(tv, a.scale);
      Real d = fixed_to_real<Real>(dv, a.scale);
      if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
      dist[off] = d;
      tot[off] = t;
    }
  }
  if (a.counters && lane == 0) {
    // work is warp-uniform: the warp issued work FMA pairs on live slots
    atomicAdd(a.counters, work);
    atomicAdd(a.counters + 1, 2ull * work);
  }
}

}  // namespace sf
