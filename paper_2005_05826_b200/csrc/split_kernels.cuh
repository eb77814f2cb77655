// K2-UW, split form (kernel 10, the default for the unweighted metric).
//
// Same exact algebra as isect_kernels.cuh: with X_e = S_e, or its complement
// when |S_e| > n/2, and fixed-point lengths (hi, lo limbs),
//   t_kl = p_k + p_l + C - G_kl,   d_kl = x_k + x_l - 2 G_kl,
//   G_kl = sum_{e: k in X_e and l in X_e} L_e.
// The rows are split by |X_e| at heavy_min (~0.01 n):
//
//  * HEAVY rows (|X_e| >= heavy_min, ~15% of rows at the EMP shape, ~99% of
//    the shared rows): permuted to the front, node-packed in 64-row X-words
//    nx[w][c]. A warp owns one u column k and 32*RS consecutive v columns;
//    it walks the bits of its u words (uniform control flow) and every lane
//    adds the row's limbs into each of its RS slots whose v word has that bit,
//    as DFMA with a 0/1 factor: 2 FP64 instructions per u bit per slot, no
//    divergence. The walk is FP64-pipe bound by construction.
//  * LIGHT rows (|X_e| < heavy_min): a slot shares only ~5-10 of them, but
//    finding them by walking per slot costs far more than they carry. They are
//    scattered instead: the light rows' member lists are compacted once and
//    each member pair's slot gets the row's limbs with u64 atomics, band by
//    band (L2-resident blocks). Every value added is an integer below 2^53
//    and so is every partial sum, so the atomics are exact and the result
//    does not depend on their order.
//
// The heavy kernel's epilogue adds the light sums and forms t, d (and d/t).
#pragma once

#include <cstdint>

#include "isect2_kernels.cuh"

namespace sf {

// (hi, lo) limbs of fixed-point length v, as exactly representable doubles.
__device__ __forceinline__ double2 limbs_of(unsigned long long v, int lo_bits) {
  return make_double2(static_cast<double>(v >> lo_bits),
                      static_cast<double>(v & ((1ull << lo_bits) - 1ull)));
}

// Heavy words only: sample-packed rows -> node-packed X words of the permuted
// heavy rows (w < Hw, Hw read on device). One warp per (word, 32-sample block).
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
__global__ void sp_heavy_colsum_kernel(const unsigned long long* __restrict__ nx, int64_t n_ext,
                                       int32_t n, const unsigned int* __restrict__ n_heavy,
                                       const unsigned long long* __restrict__ dmask64,
                                       const double2* __restrict__ limbs,
                                       unsigned long long* __restrict__ colsum) {
  const int64_t Hw = (static_cast<int64_t>(*n_heavy) + 63) / 64;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    unsigned long long xh = 0, xl = 0, ph = 0, pl = 0;
    for (int64_t w = 0; w < Hw; ++w) {
      const unsigned long long x = __ldg(nx + w * n_ext + c);
      if (!x) continue;
      const unsigned long long dm = __ldg(dmask64 + w);
      unsigned long long b = x;
      while (b) {
        const int p = 63 - __clzll(static_cast<long long>(b));  // bit position
        const unsigned long long m = 1ull << p;
        b ^= m;
        const double2 L = __ldg(limbs + 64 * w + p);
        const unsigned long long h = static_cast<unsigned long long>(L.x);
        const unsigned long long l = static_cast<unsigned long long>(L.y);
        xh += h;
        xl += l;
        if (!(dm & m)) {
          ph += h;
          pl += l;
        }
      }
    }
    atomicAdd(colsum + c, xh);
    atomicAdd(colsum + n + c, xl);
    atomicAdd(colsum + 2 * static_cast<int64_t>(n) + c, ph);
    atomicAdd(colsum + 3 * static_cast<int64_t>(n) + c, pl);
  }
}

// Light rows: one warp per row, over the light tail perm[H..E) of the row
// permutation (|S_e| from the row-key kernel). Lists the members of X_e (in
// sample order) in shared memory, adds the row to its members' column sums,
// and adds its limbs to the slot of every member pair whose stripe lies in
// [s_begin, s_end). gl: (s_end - s_begin) x n x (hi, lo) doubles.
// Pair {a < b}, d = b - a: slot (s = d-1, k = a) when d-1 < S, and slot
// (s = n-d-1, k = b) when n-d-1 < S (both for d = n/2, n even: the
// reference's duplicated half stripe). Rows with up to 32*MAXT members keep
// them in registers (lane j holds members j, j+32, ...) so the pair loop
// needs one broadcast shared load per a instead of one per pair.
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
    // members in sample order: warp-wide compaction of the (possibly
    // complemented) row words
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
    const unsigned long long lh = L.x;
    const unsigned long long ll = L.y;
    for (int i = lane; colsum && i < x; i += 32) {  // colsum null on later passes
      const int c = mem[i];
      atomicAdd(colsum + c, lh);
      atomicAdd(colsum + n + c, ll);
      if (!dense) {
        atomicAdd(colsum + 2 * static_cast<int64_t>(n) + c, lh);
        atomicAdd(colsum + 3 * static_cast<int64_t>(n) + c, ll);
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

// ---- Banded light scatter (default). The one-shot scatter above sends each
// pair's two fp64 atomics to a random 32-byte sector of the whole (stripes x
// n) light-sum array (5 GB at C3): every atomic is an HBM read-modify-write
// (ncu: 2.3 TB/s of DRAM traffic, 5% issue). Here the member lists are
// compacted once (CSR, ascending samples), and the pairs are emitted band by
// band — a band is a (stripe range x column range) block of the light-sum
// array sized to stay resident in L2 — by binary-searching, for each member
// a, the partners b whose slot falls in the band. Atomics then hit L2, and
// HBM sees each light-sum line about once.

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

// Members of every light row, ascending, at lmem[lptr[idx] ...]; the light
// rows' column sums are added here (once per run).
__global__ void sp_light_members_kernel(const uint32_t* __restrict__ rows, int64_t stride, int32_t E,
                                        int32_t n, const int32_t* __restrict__ perm,
                                        const unsigned int* __restrict__ n_heavy,
                                        const int32_t* __restrict__ mcount,
                                        const uint32_t* __restrict__ lptr,
                                        const unsigned long long* __restrict__ fix, int32_t lo_bits,
                                        int32_t* __restrict__ lmem, unsigned long long* __restrict__ colsum) {
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
    const uint32_t* row = rows + static_cast<int64_t>(r) * stride;
    int32_t* out = lmem + lptr[idx];
    const double2 L = limbs_of(fix[r], lo_bits);
    const unsigned long long lh = static_cast<unsigned long long>(L.x);
    const unsigned long long ll = static_cast<unsigned long long>(L.y);
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
        atomicAdd(colsum + smp, lh);
        atomicAdd(colsum + n + smp, ll);
        if (!dense) {
          atomicAdd(colsum + 2 * static_cast<int64_t>(n) + smp, lh);
          atomicAdd(colsum + 3 * static_cast<int64_t>(n) + smp, ll);
        }
      }
      count += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// First index j in [lo, hi) with mem[j] >= key (mem ascending).
__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ mem, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (mem[mid] < key)
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
    int32_t list_cap, int32_t dry) {
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
        if (!dry) light_add(gl + 2 * (static_cast<int64_t>(s - p0) * n + a), L);
        ++pairs;
      }
      // partners below: slot (n - (a - a') - 1, a)
      for (; j2 < i && mem[j2] <= a - n + se; ++j2) {
        const int s = n - (a - mem[j2]) - 1;
        if (!dry) light_add(gl + 2 * (static_cast<int64_t>(s - p0) * n + a), L);
        ++pairs;
      }
      reinterpret_cast<uint32_t*>(c)[i] = static_cast<uint32_t>(j1) | (static_cast<uint32_t>(j2) << 16);
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) pairs += __shfl_down_sync(0xffffffffu, pairs, off);
  if (lane == 0 && pairs) atomicAdd(pairs_out, pairs);
}

// ---- Entry lists per column band (default band scatter). The warp-per-row
// band kernel above rereads every light row's member list in every band
// launch (C3: ~190 launches, C5: ~3,000); here each launch only visits the
// members whose column lies in its band: one thread per (row, member) entry
// of the column band's list, row data precomputed.
struct LightRow {
  uint32_t b0, x;        // member list offset and length
  unsigned long long lh, ll;  // fixed-point limbs of the row's length
};

__global__ void sp_light_rowinfo_kernel(const int32_t* __restrict__ perm, int32_t E,
                                        const unsigned int* __restrict__ n_heavy,
                                        const uint32_t* __restrict__ lptr,
                                        const unsigned long long* __restrict__ fix, int32_t lo_bits,
                                        LightRow* __restrict__ info) {
  const int64_t H = *n_heavy;
  for (int64_t idx = H + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < E;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const ulonglong2 L = ilimbs_of(fix[perm[idx]], lo_bits);
    info[idx] = LightRow{lptr[idx], lptr[idx + 1] - lptr[idx], L.x, L.y};
  }
}

// Entries per column band (block histogram in shared memory, <= 1024 bands).
__global__ void sp_entry_hist_kernel(const int32_t* __restrict__ lmem, const uint32_t* __restrict__ lptr,
                                     int32_t E, int32_t KB, int32_t nkb, uint32_t* __restrict__ kcnt) {
  extern __shared__ uint32_t hist[];
  for (int i = threadIdx.x; i < nkb; i += blockDim.x) hist[i] = 0u;
  __syncthreads();
  const int64_t M = lptr[E];
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < M;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&hist[lmem[g] / KB], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < nkb; i += blockDim.x)
    if (hist[i]) atomicAdd(kcnt + i, hist[i]);
}

// Entries (member g, row idx) into their band's list; warp per light row,
// warp-aggregated slot claims (a row's members are ascending, so a warp's
// lanes mostly share one or two bands).
__global__ void sp_entry_fill_kernel(const int32_t* __restrict__ lmem, const uint32_t* __restrict__ lptr,
                                     int32_t E, const unsigned int* __restrict__ n_heavy, int32_t KB,
                                     uint32_t* __restrict__ kfill, uint2* __restrict__ ent) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t H = *n_heavy;
  for (int64_t idx = H + warp; idx < E; idx += nwarps) {
    const uint32_t b0 = lptr[idx];
    const int x = static_cast<int>(lptr[idx + 1] - b0);  // every entry listed (the histogram counts all)
    for (int base = 0; base < x; base += 32) {
      const int i = base + lane;
      const bool live = i < x;
      const int K = live ? lmem[b0 + i] / KB : -1;
      const uint32_t act = __ballot_sync(0xffffffffu, live);
      if (!live) continue;
      const uint32_t same = __match_any_sync(act, K);
      const int leader = __ffs(same) - 1;
      uint32_t pos = 0;
      if (lane == leader) pos = atomicAdd(kfill + K, static_cast<uint32_t>(__popc(same)));
      pos = __shfl_sync(same, pos, leader) + static_cast<uint32_t>(__popc(same & ((1u << lane) - 1u)));
      ent[pos] = make_uint2(b0 + static_cast<uint32_t>(i), static_cast<uint32_t>(idx));
    }
  }
}

// One band (stripes [s0, s1), the column band whose entries are ent[t0, t1)):
// same slot ownership and cursors as sp_light_band_kernel.
template <bool FIRST>
__global__ void __launch_bounds__(256) sp_light_entry_kernel(
    const uint2* __restrict__ ent, uint32_t t0, uint32_t t1, const LightRow* __restrict__ info,
    const int32_t* __restrict__ lmem, uint32_t* __restrict__ cur, int32_t n, int32_t p0, int32_t s0,
    int32_t s1, unsigned long long* __restrict__ gl, unsigned long long* __restrict__ pairs_out) {
  const int S = n / 2;
  const int se = min(s1, S);
  unsigned long long pairs = 0;
  for (uint32_t t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x) {
    const uint2 e = ent[t];
    const LightRow r = info[e.y];
    const int32_t* mem = lmem + r.b0;
    const int x = static_cast<int>(r.x);
    const int i = static_cast<int>(e.x - r.b0);
    const int a = mem[i];
    const ulonglong2 L = make_ulonglong2(r.lh, r.ll);
    int j1, j2;
    if (FIRST) {
      j1 = lower_bound_i32(mem, i + 1, x, a + s0 + 1);
      j2 = lower_bound_i32(mem, 0, i, a - n + 1 + s0);
    } else {
      const uint32_t cc = cur[e.x];
      j1 = static_cast<int>(cc & 0xffffu);
      j2 = static_cast<int>(cc >> 16);
    }
    for (; j1 < x; ++j1) {  // partners above: slot (b - a - 1, a)
      const int b = __ldg(mem + j1);
      if (b > a + se) break;
      light_add(gl + 2 * (static_cast<int64_t>(b - a - 1 - p0) * n + a), L);
      ++pairs;
    }
    for (; j2 < i; ++j2) {  // partners below: slot (n - (a - a') - 1, a)
      const int a2 = __ldg(mem + j2);
      if (a2 > a - n + se) break;
      light_add(gl + 2 * (static_cast<int64_t>(n - (a - a2) - 1 - p0) * n + a), L);
      ++pairs;
    }
    cur[e.x] = static_cast<uint32_t>(j1) | (static_cast<uint32_t>(j2) << 16);
  }
  for (int off = 16; off > 0; off >>= 1) pairs += __shfl_down_sync(0xffffffffu, pairs, off);
  if ((threadIdx.x & 31) == 0 && pairs) atomicAdd(pairs_out, pairs);
}

// bfind: position of the most significant set bit (x != 0).
__device__ __forceinline__ int msb_pos(uint32_t x) {
  int b;
  asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(x));
  return b;
}

// Nonzero heavy words per column: bit j of nz[g][c] = (nx[32g + j][c] != 0).
// Thread per (group, column), coalesced over columns.
__global__ void sp_nzmask_kernel(const unsigned long long* __restrict__ nx, int64_t n_ext, int32_t n,
                                 const unsigned int* __restrict__ n_heavy, uint32_t* __restrict__ nz) {
  const int64_t Hw = (static_cast<int64_t>(*n_heavy) + 63) / 64;
  const int64_t G = (Hw + 31) / 32;
  const int64_t total = G * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / n;
    const int64_t c = i - g * n;
    uint32_t m = 0u;
    const int64_t left = Hw - 32 * g;
    const int jmax = left < 32 ? static_cast<int>(left) : 32;
    for (int j = 0; j < jmax; ++j)
      if (__ldg(nx + (32 * g + j) * n_ext + c)) m |= 1u << j;
    nz[g * n + c] = m;
  }
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct SplitArgs {
  const unsigned long long* nx;      // [Hw][n_ext] heavy X words
  const double2* limbs;              // permuted heavy rows, by bit position
  const unsigned int* n_heavy;
  const unsigned long long* gl;      // light sums per slot (hi, lo limbs, u64)
  const unsigned long long* colsum;  // [4][n]
  const unsigned long long* cacc;    // [2]
  int64_t n_ext;
  int32_t n;
  int32_t s_begin, s_end;  // stripes computed by this launch
  int32_t out_begin;       // stripe held by row 0 of dist / tot
  int32_t gl_begin;        // stripe held by row 0 of gl (the light-sum pass)
  int32_t lo_bits, scale, finalize;
  void* dist;
  void* tot;
  unsigned long long* counters;  // [0] slot x u-bit FMAs (+ light pairs, added by host), [1] fp64 ops
  const uint32_t* nz;            // [ceil(Hw/32)][n] nonzero-word masks (LIST variants)
};

// The next (up to) two set bits of hu, highest first: positions b1, b2 and
// masks m1, m2 (0 when absent; the position then points at a valid entry).
__device__ __forceinline__ void next_two(uint32_t& hu, int& b1, uint32_t& m1, int& b2, uint32_t& m2) {
  b1 = msb_pos(hu | 1u);
  m1 = hu ? (1u << b1) : 0u;
  hu ^= m1;
  b2 = msb_pos(hu | 1u);
  m2 = hu ? (1u << b2) : 0u;
  hu ^= m2;
}

// Add the limbs of one pair of u bits to every slot whose v half has the bit
// (the bit is set in u, so v need not be masked with u first). BITMAJOR: bit
// 1 for all slots, then bit 2; else slot by slot.
template <int RS, bool BITMAJOR>
__device__ __forceinline__ void heavy_fma2(const double2 L1, uint32_t m1, const double2 L2, uint32_t m2,
                                           const uint32_t (&vv)[RS], double (&gh)[RS],
                                           double (&gl)[RS]) {
  if (BITMAJOR) {
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const double f1 = unit_if(vv[i] & m1);
      gh[i] = fma(L1.x, f1, gh[i]);
      gl[i] = fma(L1.y, f1, gl[i]);
    }
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const double f2 = unit_if(vv[i] & m2);
      gh[i] = fma(L2.x, f2, gh[i]);
      gl[i] = fma(L2.y, f2, gl[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const double f1 = unit_if(vv[i] & m1);
      const double f2 = unit_if(vv[i] & m2);
      gh[i] = fma(L1.x, f1, gh[i]);
      gl[i] = fma(L1.y, f1, gl[i]);
      gh[i] = fma(L2.x, f2, gh[i]);
      gl[i] = fma(L2.y, f2, gl[i]);
    }
  }
}

// One 32-bit half of a heavy u word, two bits per step, branch-free.
// (A ping-pong prefetch of the next step's limbs measured slower: the extra
// registers cost more occupancy than the hidden L1 latency was worth.)
template <int RS, bool BITMAJOR>
__device__ __forceinline__ void heavy_half(uint32_t hu, const double2* __restrict__ Lb,
                                           const uint32_t (&vv)[RS], double (&gh)[RS],
                                           double (&gl)[RS]) {
  while (hu) {
    int b1, b2;
    uint32_t m1, m2;
    next_two(hu, b1, m1, b2, m2);
    const double2 L1 = __ldg(Lb + b1);
    const double2 L2 = __ldg(Lb + b2);
    heavy_fma2<RS, BITMAJOR>(L1, m1, L2, m2, vv, gh, gl);
  }
}

// One nonzero heavy word (u != 0) of the warp's column, HALVES layout.
template <int RS>
__device__ __forceinline__ void heavy_word(unsigned long long u, const unsigned long long* row,
                                           const double2* Lw, int64_t l0, double (&gh)[RS], double (&gl)[RS]) {
  const uint32_t* row32 = reinterpret_cast<const uint32_t*>(row);
  uint32_t vv[RS];
  if (static_cast<uint32_t>(u >> 32)) {
#pragma unroll
    for (int i = 0; i < RS; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i) + 1);
    heavy_half<RS, false>(static_cast<uint32_t>(u >> 32), Lw + 32, vv, gh, gl);
  }
  if (static_cast<uint32_t>(u)) {
#pragma unroll
    for (int i = 0; i < RS; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i));
    heavy_half<RS, false>(static_cast<uint32_t>(u), Lw, vv, gh, gl);
  }
}

template <class Real, int RS, int NW, bool BITMAJOR = false, bool UPREF = false, bool HALVES = false,
          int MINB = 1, bool LIST = false, bool PREF = false, bool PIPE = false>
__global__ void __launch_bounds__(32 * NW, MINB) stripe_split_kernel(const SplitArgs a) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  const int Hw = static_cast<int>((*a.n_heavy + 63u) / 64u);
  // v column of slot i: l0 + 32 i (< n_ext for every i: n_ext covers a whole
  // tile past the last stripe, so dead slots read real words and are dropped)
  const int64_t l0 = static_cast<int64_t>(k) + s0 + 1 + lane;
  int nvalid = 0;
#pragma unroll
  for (int i = 0; i < RS; ++i) nvalid += (s0 + lane + 32 * i < a.s_end) ? 1 : 0;
  const int wvalid = __reduce_add_sync(0xffffffffu, nvalid);  // live slots of the warp
  unsigned long long ubits = 0;

  double gh[RS], gl[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    gh[i] = 0.0;
    gl[i] = 0.0;
  }
  if (PIPE) {
    // software-pipelined walk of the nonzero words (per-column masks): the
    // next word's u and 64-bit v words are loaded into registers while the
    // current word is walked
    const int G = (Hw + 31) / 32;
    int g = 0;
    uint32_t m = 0u;
    auto next_w = [&]() -> int {  // next nonzero word index, or -1
      while (!m) {
        if (g >= G) return -1;
        m = __ldg(a.nz + static_cast<int64_t>(g) * n + k);
        ++g;
      }
      const int w = 32 * (g - 1) + (__ffs(m) - 1);
      m &= m - 1u;
      return w;
    };
    int w = next_w();
    unsigned long long u = 0ull, v[RS];
    if (w >= 0) {
      const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
      u = __ldg(row + k);
#pragma unroll
      for (int i = 0; i < RS; ++i) v[i] = __ldg(row + l0 + 32 * i);
    }
#pragma unroll 1
    while (w >= 0) {
      const int wn = next_w();
      unsigned long long un = 0ull, vn[RS];
      if (wn >= 0) {
        const unsigned long long* nrow = a.nx + static_cast<int64_t>(wn) * n_ext;
        un = __ldg(nrow + k);
#pragma unroll
        for (int i = 0; i < RS; ++i) vn[i] = __ldg(nrow + l0 + 32 * i);
      }
      ubits += static_cast<unsigned>(__popcll(u));
      const double2* Lw = a.limbs + 64 * static_cast<int64_t>(w);
      uint32_t vh[RS], vl[RS];
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        vh[i] = static_cast<uint32_t>(v[i] >> 32);
        vl[i] = static_cast<uint32_t>(v[i]);
      }
      heavy_half<RS, false>(static_cast<uint32_t>(u >> 32), Lw + 32, vh, gh, gl);
      heavy_half<RS, false>(static_cast<uint32_t>(u), Lw, vl, gh, gl);
      w = wn;
      u = un;
#pragma unroll
      for (int i = 0; i < RS; ++i) v[i] = vn[i];
    }
  }
  if (LIST) {
    // walk only the nonzero words of column k (per-column masks), and pull
    // the next word's u and v lines into L1 while this word is walked
    const int G = (Hw + 31) / 32;
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      uint32_t m = __ldg(a.nz + static_cast<int64_t>(g) * n + k);
      while (m) {
        const int w = 32 * g + (__ffs(m) - 1);
        m &= m - 1u;
        const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
        if (PREF && m) {
          const unsigned long long* nrow = a.nx + static_cast<int64_t>(32 * g + (__ffs(m) - 1)) * n_ext;
          if (lane == 0) prefetch_l1(nrow + k);
#pragma unroll
          for (int i = 0; i < RS; ++i) prefetch_l1(nrow + l0 + 32 * i);
        }
        const unsigned long long u = __ldg(row + k);
        ubits += static_cast<unsigned>(__popcll(u));
        heavy_word<RS>(u, row, a.limbs + 64 * static_cast<int64_t>(w), l0, gh, gl);
      }
    }
  }
  unsigned long long u_next = (UPREF && Hw > 0) ? __ldg(a.nx + k) : 0ull;
#pragma unroll 1
  for (int w = 0; (LIST || PIPE) ? false : w < Hw; ++w) {
    const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
    unsigned long long u;
    if (UPREF) {
      u = u_next;  // loaded one word ahead
      if (w + 1 < Hw) u_next = __ldg(row + n_ext + k);
    } else {
      u = __ldg(row + k);
    }
    if (u == 0ull) continue;
    const double2* Lw = a.limbs + 64 * static_cast<int64_t>(w);
    ubits += static_cast<unsigned>(__popcll(u));
    if (HALVES) {  // one 32-bit half of the v words live at a time (fewer registers)
      const uint32_t* row32 = reinterpret_cast<const uint32_t*>(row);
      uint32_t vv[RS];
      if (static_cast<uint32_t>(u >> 32)) {
#pragma unroll
        for (int i = 0; i < RS; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i) + 1);
        heavy_half<RS, BITMAJOR>(static_cast<uint32_t>(u >> 32), Lw + 32, vv, gh, gl);
      }
      if (static_cast<uint32_t>(u)) {
#pragma unroll
        for (int i = 0; i < RS; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i));
        heavy_half<RS, BITMAJOR>(static_cast<uint32_t>(u), Lw, vv, gh, gl);
      }
    } else {
      uint32_t vh[RS], vl[RS];
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const unsigned long long v = __ldg(row + l0 + 32 * i);
        vh[i] = static_cast<uint32_t>(v >> 32);
        vl[i] = static_cast<uint32_t>(v);
      }
      heavy_half<RS, BITMAJOR>(static_cast<uint32_t>(u >> 32), Lw + 32, vh, gh, gl);
      heavy_half<RS, BITMAJOR>(static_cast<uint32_t>(u), Lw, vl, gh, gl);
    }
  }

  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;
  const long long ch = static_cast<long long>(a.cacc[0]);
  const long long cl = static_cast<long long>(a.cacc[1]);
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    if (i >= nvalid) break;
    const int s = s0 + lane + 32 * i;
    const int64_t li = l0 + 32 * i;
    const int lm = li >= n ? static_cast<int>(li - n) : static_cast<int>(li);
    const int64_t off = static_cast<int64_t>(s - a.out_begin) * n + k;
    const ulonglong2 light =
        reinterpret_cast<const ulonglong2*>(a.gl)[static_cast<int64_t>(s - a.gl_begin) * n + k];
    const long long Gh_ = static_cast<long long>(gh[i]) + static_cast<long long>(light.x);
    const long long Gl_ = static_cast<long long>(gl[i]) + static_cast<long long>(light.y);
    const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - Gh_;
    const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - Gl_;
    const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * Gh_;
    const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * Gl_;
    const __int128 tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
    const __int128 dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
    const Real t = static_cast<Real>(i2_fixed_to_double(tv, a.scale));
    Real d = static_cast<Real>(i2_fixed_to_double(dv, a.scale));
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    dist[off] = d;
    tot[off] = t;
  }
  if (a.counters && lane == 0) {
    // ubits is warp-uniform: the warp issued ubits x (live slots) FMA pairs
    atomicAdd(a.counters, ubits * static_cast<unsigned long long>(wvalid));
    atomicAdd(a.counters + 1, 2ull * ubits * static_cast<unsigned long long>(wvalid));
  }
}

// ---- Integer-accumulator variant (A/B: SF_SPLIT_VARIANT=16). Same walk,
// but each slot accumulates the row's 63-bit fixed-point length as two
// 32-bit limbs with IMAD.WIDE.U32 (0/1 bit x limb + u64 accumulator) on the
// integer/FMA pipes instead of DFMA on the FP64 pipe. Exact: a column has at
// most ~2^14 heavy bits, so each 64-bit limb sum stays below 2^46.
__global__ void sp_ilimbs_kernel(const double2* __restrict__ limbs, int64_t count, int32_t lo_bits,
                                 uint2* __restrict__ il) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 L = limbs[i];
    const unsigned long long v = (static_cast<unsigned long long>(L.x) << lo_bits) +
                                 static_cast<unsigned long long>(L.y);
    il[i] = make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
  }
}

template <int RS>
__device__ __forceinline__ void heavy_half_int(uint32_t hu, const uint2* __restrict__ Lb,
                                               const uint32_t (&vv)[RS], unsigned long long (&al)[RS],
                                               unsigned long long (&ah)[RS]) {
  while (hu) {
    int b1, b2;
    uint32_t m1, m2;
    next_two(hu, b1, m1, b2, m2);
    const uint2 L1 = __ldg(Lb + b1);
    const uint2 L2 = __ldg(Lb + b2);
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const uint32_t f1 = (vv[i] & m1) ? 1u : 0u;
      const uint32_t f2 = (vv[i] & m2) ? 1u : 0u;
      // acc += f * L as one IMAD.WIDE.U32 each (the compiler would otherwise
      // select and add in two 32-bit halves)
      asm("mad.wide.u32 %0, %2, %3, %0;\n\tmad.wide.u32 %1, %2, %4, %1;"
          : "+l"(al[i]), "+l"(ah[i]) : "r"(f1), "r"(L1.x), "r"(L1.y));
      asm("mad.wide.u32 %0, %2, %3, %0;\n\tmad.wide.u32 %1, %2, %4, %1;"
          : "+l"(al[i]), "+l"(ah[i]) : "r"(f2), "r"(L2.x), "r"(L2.y));
    }
  }
}

template <class Real, int RS, int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB) stripe_split_int_kernel(const SplitArgs a, const uint2* il) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  const int Hw = static_cast<int>((*a.n_heavy + 63u) / 64u);
  const int64_t l0 = static_cast<int64_t>(k) + s0 + 1 + lane;
  int nvalid = 0;
#pragma unroll
  for (int i = 0; i < RS; ++i) nvalid += (s0 + lane + 32 * i < a.s_end) ? 1 : 0;
  const int wvalid = __reduce_add_sync(0xffffffffu, nvalid);
  unsigned long long ubits = 0;
  unsigned long long al[RS], ah[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    al[i] = 0ull;
    ah[i] = 0ull;
  }
#pragma unroll 1
  for (int w = 0; w < Hw; ++w) {
    const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
    const unsigned long long u = __ldg(row + k);
    if (u == 0ull) continue;
    const uint2* Lw = il + 64 * static_cast<int64_t>(w);
    ubits += static_cast<unsigned>(__popcll(u));
    const uint32_t* row32 = reinterpret_cast<const uint32_t*>(row);
    uint32_t vv[RS];
    if (static_cast<uint32_t>(u >> 32)) {
#pragma unroll
      for (int i = 0; i < RS; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i) + 1);
      heavy_half_int<RS>(static_cast<uint32_t>(u >> 32), Lw + 32, vv, al, ah);
    }
    if (static_cast<uint32_t>(u)) {
#pragma unroll
      for (int i = 0; i < RS; ++i) vv[i] = __ldg(row32 + 2 * (l0 + 32 * i));
      heavy_half_int<RS>(static_cast<uint32_t>(u), Lw, vv, al, ah);
    }
  }
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;
  const int lb = a.lo_bits;
  const __int128 C = (static_cast<__int128>(a.cacc[0]) << lb) + static_cast<__int128>(a.cacc[1]);
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    if (i >= nvalid) break;
    const int s = s0 + lane + 32 * i;
    const int64_t li = l0 + 32 * i;
    const int lm = li >= n ? static_cast<int>(li - n) : static_cast<int>(li);
    const int64_t off = static_cast<int64_t>(s - a.out_begin) * n + k;
    const ulonglong2 light =
        reinterpret_cast<const ulonglong2*>(a.gl)[static_cast<int64_t>(s - a.gl_begin) * n + k];
    const __int128 G = (static_cast<__int128>(ah[i]) << 32) + static_cast<__int128>(al[i]) +
                       (static_cast<__int128>(light.x) << lb) + static_cast<__int128>(light.y);
    const __int128 P = (static_cast<__int128>(xs[2 * n + k] + xs[2 * n + lm]) << lb) +
                       static_cast<__int128>(xs[3 * n + k] + xs[3 * n + lm]);
    const __int128 X = (static_cast<__int128>(xs[k] + xs[lm]) << lb) + static_cast<__int128>(xs[n + k] + xs[n + lm]);
    const __int128 tv = P + C - G;
    const __int128 dv = X - 2 * G;
    const Real t = static_cast<Real>(i2_fixed_to_double(tv, a.scale));
    Real d = static_cast<Real>(i2_fixed_to_double(dv, a.scale));
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    dist[off] = d;
    tot[off] = t;
  }
  if (a.counters && lane == 0) {
    atomicAdd(a.counters, ubits * static_cast<unsigned long long>(wvalid));
    atomicAdd(a.counters + 1, 2ull * ubits * static_cast<unsigned long long>(wvalid));
  }
}

}  // namespace sf
