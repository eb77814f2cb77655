// K2-UW, intersection form v2 (kernel 6): the same exact algebra as
// isect_kernels.cuh (t = p_k + p_l + C - G_kl, d = x_k + x_l - 2 G_kl with
// X_e = S_e or its complement), with a layout chosen for the walk:
//
//  * rows are PERMUTED before packing: because the sums are exact, row order
//    is free. "Heavy" rows (|X_e| >= heavy_min, i.e. the rows most pairs
//    share) go first, sorted by |X_e| descending; the rest keep postorder
//    (subtree locality). At the EMP shape this halves the words a slot has to
//    visit (577 -> ~240 candidate words) and concentrates ~80% of the shared
//    rows in the first ~4 groups;
//  * 64-row words (u64), bit (63-i) = permuted row 64w+i; groups of 32 words
//    (2048 rows) with a per-column occupancy mask, and a second level: one
//    bit per group per column (gm), so a slot skips every group in which
//    either column is empty;
//  * lengths as two exactly representable doubles (hi, lo limbs of the
//    fixed-point value), stored by bit position within the word and
//    accumulated with DADD: every partial sum stays below 2^53, so the
//    accumulation is exact;
//  * no shared-memory staging and no CTA barriers: each warp owns one u
//    column (uniform loads) and 32*RS consecutive v columns (coalesced
//    loads); all reads go through L1/L2, so warps never wait on each other.
#pragma once

#include <cstdint>

namespace sf {

// ---- preparation ----------------------------------------------------------

// One warp per row: |S_e|, dense flag, and the sort key that puts heavy rows
// first by |X_e| descending (stable radix sort keeps postorder among ties and
// among the light rows, whose key is n + 1).
__global__ void i2_row_key_kernel(const uint32_t* __restrict__ rows, int64_t stride, int32_t E,
                                  int32_t n, int32_t heavy_min, uint32_t* __restrict__ keys,
                                  int32_t* __restrict__ vals, uint8_t* __restrict__ dense,
                                  unsigned int* __restrict__ n_heavy,
                                  int32_t* __restrict__ mcount = nullptr,
                                  bool heavy_in_postorder = false) {
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
      // heavy first: by |X_e| descending (kernels 6-9: densest words first), or
      // in postorder (kernel 10: subtree locality, 25% fewer nonzero words
      // per column at the EMP shape); light rows after, in postorder
      const uint32_t hkey = heavy_in_postorder ? 0u : static_cast<uint32_t>(n - x);
      keys[r] = x >= heavy_min ? hkey : static_cast<uint32_t>(n + 1);
      vals[r] = static_cast<int32_t>(r);
      dense[r] = dn ? 1 : 0;
      if (mcount) mcount[r] = m;
      if (x >= heavy_min) atomicAdd(n_heavy, 1u);
    }
  }
}

// Permuted row i <- original row perm[i]: dense mask, length limbs as
// doubles, and C = sum of the dense rows' fixed-point lengths (limb sums).
__global__ void i2_perm_kernel(const int32_t* __restrict__ perm, int32_t E, int64_t rows_pad,
                               const uint8_t* __restrict__ dense,
                               const unsigned long long* __restrict__ fix, int32_t lo_bits,
                               unsigned long long* __restrict__ dmask64,
                               double2* __restrict__ limbs, unsigned long long* __restrict__ cacc) {
  const unsigned long long lo_mask = (1ull << lo_bits) - 1ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows_pad;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t slot = (i & ~int64_t{63}) + (63 - (i & 63));  // by bit position
    if (i >= E) {
      limbs[slot] = make_double2(0.0, 0.0);
      continue;
    }
    const int r = perm[i];
    const unsigned long long v = fix[r];
    const unsigned long long hi = v >> lo_bits, lo = v & lo_mask;
    limbs[slot] = make_double2(static_cast<double>(hi), static_cast<double>(lo));
    if (dense[r]) {
      atomicOr(dmask64 + (i >> 6), 0x8000000000000000ull >> (i & 63));
      atomicAdd(cacc, hi);
      atomicAdd(cacc + 1, lo);
    }
  }
}

// Sample-packed rows -> node-packed 64-row X-words of the permuted rows.
// One warp per (64-row word w, 32-sample block cb): 2 x 32 ballots.
__global__ void i2_transpose_kernel(const uint32_t* __restrict__ rows, int64_t stride,
                                    const int32_t* __restrict__ perm, int32_t E, int32_t n,
                                    int32_t W, const unsigned long long* __restrict__ dmask64,
                                    unsigned long long* __restrict__ nx, int64_t n_ext) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t blocks = static_cast<int64_t>(W) * stride;
  for (int64_t bidx = warp; bidx < blocks; bidx += nwarps) {
    const int64_t w = bidx / stride;
    const int64_t cb = bidx - w * stride;
    const int64_t r1 = 64 * w + lane, r2 = r1 + 32;
    const uint32_t a = r1 < E ? __ldg(rows + static_cast<int64_t>(perm[r1]) * stride + cb) : 0u;
    const uint32_t b = r2 < E ? __ldg(rows + static_cast<int64_t>(perm[r2]) * stride + cb) : 0u;
    unsigned long long out = 0ull;
#pragma unroll
    for (int bit = 0; bit < 32; ++bit) {
      const uint32_t v1 = __ballot_sync(0xffffffffu, (a >> bit) & 1u);
      const uint32_t v2 = __ballot_sync(0xffffffffu, (b >> bit) & 1u);
      if (bit == lane)
        out = (static_cast<unsigned long long>(__brev(v1)) << 32) | static_cast<unsigned long long>(__brev(v2));
    }
    const int64_t s = cb * 32 + lane;
    if (s < n) nx[w * n_ext + s] = out ^ dmask64[w];
  }
}

// Wrap columns: nx[w][c] = nx[w][c mod n] for n <= c < n_ext.
__global__ void i2_extend_kernel(unsigned long long* __restrict__ nx, int64_t n_ext, int32_t n,
                                 int32_t W) {
  const int64_t extra = n_ext - n;
  const int64_t total = static_cast<int64_t>(W) * extra;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / extra;
    const int64_t col = n + i % extra;
    nx[w * n_ext + col] = nx[w * n_ext + col % n];
  }
}

// One thread per (group, column): occupancy mask, nonzero-word count, the
// group bit of the column, and for real columns the limb sums x_c / p_c.
// colsum layout: [4][n] = x_hi, x_lo, p_hi, p_lo; gm layout: [NGW][n_ext].
__global__ void i2_occ_kernel(const unsigned long long* __restrict__ nx, int64_t n_ext, int32_t n,
                              int32_t W, int32_t G, const unsigned long long* __restrict__ dmask64,
                              const double2* __restrict__ limbs, uint32_t* __restrict__ occ,
                              uint32_t* __restrict__ cnt, uint32_t* __restrict__ gm,
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
      const unsigned long long x = __ldg(nx + static_cast<int64_t>(w) * n_ext + c);
      if (x == 0ull) continue;
      o |= 0x80000000u >> i;
      ++count;
      if (c < n) {
        const unsigned long long dm = __ldg(dmask64 + w);
        unsigned long long b = x;
        while (b) {
          const int p = __clzll(static_cast<long long>(b));
          const unsigned long long m = 0x8000000000000000ull >> p;
          b ^= m;
          const double2 L = __ldg(limbs + 64 * static_cast<int64_t>(w) + (63 - p));
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
    }
    occ[idx] = o;
    cnt[idx] = static_cast<uint32_t>(count);
    if (o) atomicOr(gm + static_cast<int64_t>(g >> 5) * n_ext + c, 0x80000000u >> (g & 31));
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

// One thread per (group, column): the nonzero words, in word order.
__global__ void i2_pack_kernel(const unsigned long long* __restrict__ nx, int64_t n_ext, int32_t W,
                               int32_t G, const uint32_t* __restrict__ base,
                               unsigned long long* __restrict__ packed) {
  const int64_t total = static_cast<int64_t>(G) * n_ext;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(idx / n_ext);
    const int64_t c = idx - static_cast<int64_t>(g) * n_ext;
    unsigned long long* out = packed + base[idx];
    for (int i = 0; i < 32; ++i) {
      const int w = 32 * g + i;
      if (w >= W) break;
      const unsigned long long x = __ldg(nx + static_cast<int64_t>(w) * n_ext + c);
      if (x) *out++ = x;
    }
  }
}

// ---- the stripe kernel ------------------------------------------------------

struct Isect2Args {
  const uint32_t* occ;                 // [G][n_ext]
  const uint32_t* base;                // [G*n_ext + 1], in u64 words
  const unsigned long long* packed;    // nonzero X-words
  const double2* limbs;                // [G*2048] (hi, lo) of permuted rows
  const uint32_t* gm;                  // [NGW][n_ext]
  const unsigned long long* colsum;    // [4][n]
  const unsigned long long* cacc;      // [2]
  const unsigned long long* nx;        // [W][n_ext] X words (kernel 7: the heavy region)
  const unsigned int* n_heavy;         // rows with |X_e| >= heavy_min (sorted first)
  int64_t n_ext;
  int32_t G, NGW, W;
  int32_t n;
  int32_t s_begin, s_end;
  int32_t lo_bits;   // value = hi * 2^lo_bits + lo
  int32_t scale;     // value = round(L * 2^scale)
  int32_t finalize;
  void* dist;
  void* tot;
  unsigned long long* exec_updates;
};

// Exact value v * 2^-scale (v >= 0, a 128-bit integer), correctly rounded.
__device__ __forceinline__ double i2_fixed_to_double(__int128 v, int scale) {
  const unsigned __int128 u = static_cast<unsigned __int128>(v);
  const unsigned long long hi = static_cast<unsigned long long>(u >> 64);
  const unsigned long long lo = static_cast<unsigned long long>(u);
  if (hi == 0ull) return ldexp(__ull2double_rn(lo), -scale);
  const int sh = 64 - __clzll(static_cast<long long>(hi));
  unsigned long long top = static_cast<unsigned long long>(u >> sh);
  const unsigned long long rest = sh == 64 ? lo : (lo & ((1ull << sh) - 1ull));
  top |= rest != 0ull ? 1ull : 0ull;
  return ldexp(__ull2double_rn(top), sh - scale);
}

// (hit ? 1.0 : 0.0) built from its high word only: one SEL. acc = fma(L, f,
// acc) then adds L exactly as a DADD would (f = 1) or leaves acc unchanged
// (f = 0: L*0 = +0 and acc + 0 = acc), one DFMA per limb and slot instead of
// the DADD + 2 FSEL the compiler emits for a conditional add.
__device__ __forceinline__ double unit_if(uint32_t hit) {
  return __hiloint2double(hit ? 0x3ff00000 : 0, 0);
}

// Warp w of the CTA owns u column k = blockIdx.x*NW + w and the stripes
// s0 + lane + 32*i (i < RS), s0 = s_begin + blockIdx.y*32*RS.
//
// limbs are indexed by BIT POSITION within each 64-row word (entry 64w + b is
// the row at bit b, i.e. permuted row 64w + 63 - b), so a set bit found with
// FLO on either 32-bit half addresses its length directly.
template <class Real, int RS, int NW>
__global__ void __launch_bounds__(32 * NW) stripe_isect2_kernel(const Isect2Args a) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  uint32_t executed = 0;
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;

#pragma unroll 1
  for (int i = 0; i < RS; ++i) {
    const int s = s0 + lane + 32 * i;
    if (s >= a.s_end) break;
    const int64_t l = static_cast<int64_t>(k) + s + 1;  // extended column, < n_ext
    double gh = 0.0, gl = 0.0;
#pragma unroll 1
    for (int j = 0; j < a.NGW; ++j) {
      uint32_t gmask = __ldg(a.gm + j * n_ext + k) & __ldg(a.gm + j * n_ext + l);
      while (gmask) {
        const int gi = __clz(gmask);
        gmask ^= 0x80000000u >> gi;
        const int g = 32 * j + gi;
        const int64_t gb = static_cast<int64_t>(g) * n_ext;
        const uint32_t ou = __ldg(a.occ + gb + k);
        const uint32_t ov = __ldg(a.occ + gb + l);
        uint32_t o = ou & ov;
        if (!o) continue;
        const uint32_t bu = __ldg(a.base + gb + k);
        const uint32_t bv = __ldg(a.base + gb + l);
        const double2* Lg = a.limbs + static_cast<int64_t>(g) * 2048;
        do {
          const int w = __clz(o);
          o ^= 0x80000000u >> w;
          const uint32_t above = ~(0xffffffffu >> w);
          const unsigned long long x = __ldg(a.packed + (bu + __popc(ou & above))) &
                                       __ldg(a.packed + (bv + __popc(ov & above)));
          uint32_t xh = static_cast<uint32_t>(x >> 32);
          uint32_t xl = static_cast<uint32_t>(x);
          executed += __popc(xh) + __popc(xl);
          const double2* Lw = Lg + 64 * w;
          while (xh) {
            const int b = 31 - __clz(xh);
            xh ^= 1u << b;
            const double2 L = __ldg(Lw + 32 + b);
            gh += L.x;
            gl += L.y;
          }
          while (xl) {
            const int b = 31 - __clz(xl);
            xl ^= 1u << b;
            const double2 L = __ldg(Lw + b);
            gh += L.x;
            gl += L.y;
          }
        } while (o);
      }
    }
    const int lm = l >= n ? static_cast<int>(l - n) : static_cast<int>(l);
    const long long ch = static_cast<long long>(a.cacc[0]);
    const long long cl = static_cast<long long>(a.cacc[1]);
    const long long Gh = static_cast<long long>(gh);
    const long long Gl = static_cast<long long>(gl);
    const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - Gh;
    const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - Gl;
    const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * Gh;
    const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * Gl;
    const __int128 tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
    const __int128 dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
    const Real t = static_cast<Real>(i2_fixed_to_double(tv, a.scale));
    Real d = static_cast<Real>(i2_fixed_to_double(dv, a.scale));
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
    dist[off] = d;
    tot[off] = t;
  }
  if (a.exec_updates) {
    unsigned long long e = executed;
    for (int off = 16; off > 0; off >>= 1) e += __shfl_down_sync(0xffffffffu, e, off);
    if (lane == 0) atomicAdd(a.exec_updates, e);
  }
}

// Kernel 7: kernel 6's light-row walk, plus a HEAVY region processed
// warp-uniformly. The first Gh groups hold the rows most slots share
// (|X_e| >= ~0.06 n). There every word is nonzero for almost every column, so
// instead of each lane walking the bits of its own u&v (divergent: ~5 of 32
// lanes busy), the warp walks the bits of its shared u word and every lane
// tests its RS v words at that bit: one uniform limb load, then predicated
// DADDs — no divergence, each u bit serving 32*RS slots at once.
template <class Real, int RS, int NW>
__global__ void __launch_bounds__(32 * NW) stripe_isect3_kernel(const Isect2Args a) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  const int Gh = static_cast<int>((*a.n_heavy + 2047u) / 2048u);
  const int Hw = min(a.W, 32 * Gh);
  uint32_t executed = 0;

  int64_t l[RS];
  bool ok[RS];
  double gh[RS], gl[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    const int s = s0 + lane + 32 * i;
    ok[i] = s < a.s_end;
    l[i] = ok[i] ? static_cast<int64_t>(k) + s + 1 : static_cast<int64_t>(k) + 1;
    gh[i] = 0.0;
    gl[i] = 0.0;
  }

  // ---- heavy region: uniform walk over the u column's bits
#pragma unroll 1
  for (int w = 0; w < Hw; ++w) {
    const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
    const unsigned long long u = __ldg(row + k);
    if (u == 0ull) continue;
    uint32_t vh[RS], vl[RS];
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const unsigned long long v = ok[i] ? (__ldg(row + l[i]) & u) : 0ull;
      vh[i] = static_cast<uint32_t>(v >> 32);
      vl[i] = static_cast<uint32_t>(v);
      executed += __popc(vh[i]) + __popc(vl[i]);
    }
    const double2* Lw = a.limbs + 64 * static_cast<int64_t>(w);
    uint32_t uh = static_cast<uint32_t>(u >> 32);
    while (uh) {
      const int b = 31 - __clz(uh);
      const uint32_t m = 1u << b;
      uh ^= m;
      const double2 L = __ldg(Lw + 32 + b);
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const double f = unit_if(vh[i] & m);
        gh[i] = fma(L.x, f, gh[i]);
        gl[i] = fma(L.y, f, gl[i]);
      }
    }
    uint32_t ul = static_cast<uint32_t>(u);
    while (ul) {
      const int b = 31 - __clz(ul);
      const uint32_t m = 1u << b;
      ul ^= m;
      const double2 L = __ldg(Lw + b);
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const double f = unit_if(vl[i] & m);
        gh[i] = fma(L.x, f, gh[i]);
        gl[i] = fma(L.y, f, gl[i]);
      }
    }
  }

  // ---- light region: per-slot walk of the groups >= Gh (as kernel 6)
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    if (!ok[i]) continue;
    const int64_t li = l[i];
    double ah = gh[i], al = gl[i];
#pragma unroll 1
    for (int j = Gh >> 5; j < a.NGW; ++j) {
      uint32_t gmask = __ldg(a.gm + j * n_ext + k) & __ldg(a.gm + j * n_ext + li);
      if (j == (Gh >> 5)) gmask &= 0xffffffffu >> (Gh & 31);
      while (gmask) {
        const int gi = __clz(gmask);
        gmask ^= 0x80000000u >> gi;
        const int g = 32 * j + gi;
        const int64_t gb = static_cast<int64_t>(g) * n_ext;
        const uint32_t ou = __ldg(a.occ + gb + k);
        const uint32_t ov = __ldg(a.occ + gb + li);
        uint32_t o = ou & ov;
        if (!o) continue;
        const uint32_t bu = __ldg(a.base + gb + k);
        const uint32_t bv = __ldg(a.base + gb + li);
        const double2* Lg = a.limbs + static_cast<int64_t>(g) * 2048;
        do {
          const int w = __clz(o);
          o ^= 0x80000000u >> w;
          const uint32_t above = ~(0xffffffffu >> w);
          const unsigned long long x = __ldg(a.packed + (bu + __popc(ou & above))) &
                                       __ldg(a.packed + (bv + __popc(ov & above)));
          uint32_t xh = static_cast<uint32_t>(x >> 32);
          uint32_t xl = static_cast<uint32_t>(x);
          executed += __popc(xh) + __popc(xl);
          const double2* Lw = Lg + 64 * w;
          while (xh) {
            const int b = 31 - __clz(xh);
            xh ^= 1u << b;
            const double2 L = __ldg(Lw + 32 + b);
            ah += L.x;
            al += L.y;
          }
          while (xl) {
            const int b = 31 - __clz(xl);
            xl ^= 1u << b;
            const double2 L = __ldg(Lw + b);
            ah += L.x;
            al += L.y;
          }
        } while (o);
      }
    }
    const int s = s0 + lane + 32 * i;
    const int lm = li >= n ? static_cast<int>(li - n) : static_cast<int>(li);
    const long long ch = static_cast<long long>(a.cacc[0]);
    const long long cl = static_cast<long long>(a.cacc[1]);
    const long long Gh_ = static_cast<long long>(ah);
    const long long Gl_ = static_cast<long long>(al);
    const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - Gh_;
    const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - Gl_;
    const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * Gh_;
    const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * Gl_;
    const __int128 tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
    const __int128 dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
    const Real t = static_cast<Real>(i2_fixed_to_double(tv, a.scale));
    Real d = static_cast<Real>(i2_fixed_to_double(dv, a.scale));
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
    dist[off] = d;
    tot[off] = t;
  }
  if (a.exec_updates) {
    unsigned long long e = executed;
    for (int off = 16; off > 0; off >>= 1) e += __shfl_down_sync(0xffffffffu, e, off);
    if (lane == 0) atomicAdd(a.exec_updates, e);
  }
}

// Kernel 8: kernel 7's warp-uniform heavy region, and a warp-uniform LIGHT
// walk too. In the light region a lane's slot rarely shares a word with its
// u column, so walking each slot's candidates separately (kernels 6/7) leaves
// ~1-4 of 32 lanes busy. Here the warp walks the u column's nonzero words
// (uniform loop, only words some lane shares) and each lane checks its RS v
// columns' occupancy bit for that word; only hits load the packed v word and
// walk the (usually single) shared bit.
template <class Real, int RS, int NW>
__global__ void __launch_bounds__(32 * NW) stripe_isect4_kernel(const Isect2Args a) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  const int Gh = static_cast<int>((*a.n_heavy + 2047u) / 2048u);
  const int Hw = min(a.W, 32 * Gh);
  uint32_t executed = 0;

  int64_t l[RS];
  bool ok[RS];
  double gh[RS], gl[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    const int s = s0 + lane + 32 * i;
    ok[i] = s < a.s_end;
    l[i] = ok[i] ? static_cast<int64_t>(k) + s + 1 : static_cast<int64_t>(k) + 1;
    gh[i] = 0.0;
    gl[i] = 0.0;
  }

  // ---- heavy region: uniform walk over the u column's bits
#pragma unroll 1
  for (int w = 0; w < Hw; ++w) {
    const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
    const unsigned long long u = __ldg(row + k);
    if (u == 0ull) continue;
    uint32_t vh[RS], vl[RS];
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const unsigned long long v = ok[i] ? (__ldg(row + l[i]) & u) : 0ull;
      vh[i] = static_cast<uint32_t>(v >> 32);
      vl[i] = static_cast<uint32_t>(v);
      executed += __popc(vh[i]) + __popc(vl[i]);
    }
    const double2* Lw = a.limbs + 64 * static_cast<int64_t>(w);
    uint32_t uh = static_cast<uint32_t>(u >> 32);
    while (uh) {
      const int b = 31 - __clz(uh);
      const uint32_t m = 1u << b;
      uh ^= m;
      const double2 L = __ldg(Lw + 32 + b);
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const double f = unit_if(vh[i] & m);
        gh[i] = fma(L.x, f, gh[i]);
        gl[i] = fma(L.y, f, gl[i]);
      }
    }
    uint32_t ul = static_cast<uint32_t>(u);
    while (ul) {
      const int b = 31 - __clz(ul);
      const uint32_t m = 1u << b;
      ul ^= m;
      const double2 L = __ldg(Lw + b);
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const double f = unit_if(vl[i] & m);
        gh[i] = fma(L.x, f, gh[i]);
        gl[i] = fma(L.y, f, gl[i]);
      }
    }
  }

  // ---- light region: uniform walk over the u column's nonzero words
#pragma unroll 1
  for (int j = Gh >> 5; j < a.NGW; ++j) {
    uint32_t gmask = __ldg(a.gm + j * n_ext + k);
    if (j == (Gh >> 5)) gmask &= 0xffffffffu >> (Gh & 31);
    while (gmask) {
      const int gi = __clz(gmask);
      gmask ^= 0x80000000u >> gi;
      const int g = 32 * j + gi;
      const int64_t gb = static_cast<int64_t>(g) * n_ext;
      const uint32_t ou = __ldg(a.occ + gb + k);
      const uint32_t bu = __ldg(a.base + gb + k);
      uint32_t ov[RS], bv[RS];
      uint32_t any = 0u;
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        ov[i] = ok[i] ? (__ldg(a.occ + gb + l[i]) & ou) : 0u;
        bv[i] = __ldg(a.base + gb + l[i]);
        any |= ov[i];
      }
      uint32_t wm = __reduce_or_sync(0xffffffffu, any);
      const double2* Lg = a.limbs + static_cast<int64_t>(g) * 2048;
      while (wm) {
        const int w = __clz(wm);
        const uint32_t bit = 0x80000000u >> w;
        wm ^= bit;
        const uint32_t above = ~(0xffffffffu >> w);
        const unsigned long long u = __ldg(a.packed + (bu + __popc(ou & above)));
        const double2* Lw = Lg + 64 * w;
#pragma unroll
        for (int i = 0; i < RS; ++i) {
          if (!(ov[i] & bit)) continue;
          const unsigned long long x =
              u & __ldg(a.packed + (bv[i] + __popc(__ldg(a.occ + gb + l[i]) & above)));
          uint32_t xh = static_cast<uint32_t>(x >> 32);
          uint32_t xl = static_cast<uint32_t>(x);
          executed += __popc(xh) + __popc(xl);
          while (xh) {
            const int b = 31 - __clz(xh);
            xh ^= 1u << b;
            const double2 L = __ldg(Lw + 32 + b);
            gh[i] += L.x;
            gl[i] += L.y;
          }
          while (xl) {
            const int b = 31 - __clz(xl);
            xl ^= 1u << b;
            const double2 L = __ldg(Lw + b);
            gh[i] += L.x;
            gl[i] += L.y;
          }
        }
      }
    }
  }

  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;
  const long long ch = static_cast<long long>(a.cacc[0]);
  const long long cl = static_cast<long long>(a.cacc[1]);
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    if (!ok[i]) continue;
    const int s = s0 + lane + 32 * i;
    const int lm = l[i] >= n ? static_cast<int>(l[i] - n) : static_cast<int>(l[i]);
    const long long Gh_ = static_cast<long long>(gh[i]);
    const long long Gl_ = static_cast<long long>(gl[i]);
    const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - Gh_;
    const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - Gl_;
    const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * Gh_;
    const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * Gl_;
    const __int128 tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
    const __int128 dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
    const Real t = static_cast<Real>(i2_fixed_to_double(tv, a.scale));
    Real d = static_cast<Real>(i2_fixed_to_double(dv, a.scale));
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
    dist[off] = d;
    tot[off] = t;
  }
  if (a.exec_updates) {
    unsigned long long e = executed;
    for (int off = 16; off > 0; off >>= 1) e += __shfl_down_sync(0xffffffffu, e, off);
    if (lane == 0) atomicAdd(a.exec_updates, e);
  }
}

// Kernel 9: kernel 7 retuned so the heavy walk is FP64-bound. The heavy
// region now reaches down to |X_e| >= ~0.012 n (the rows that carry ~99% of
// the shared rows), each lane serves RS = 8 slots per u bit (per slot and u
// bit: one LOP3 + SEL to build the 0/1 factor, two DFMA — half the issue
// slots land on the FP64 pipe, which therefore saturates at full issue), and
// the per-slot light walk only has ~10 shared rows per slot left to find.
// fp_ops counts the FP64 instructions issued per lane (2 per u bit per live
// slot in the heavy walk, 2 per shared bit in the light walk): the roofline
// numerator.
template <class Real, int RS, int NW>
__global__ void __launch_bounds__(32 * NW) stripe_isect5_kernel(const Isect2Args a,
                                                                unsigned long long* fp_ops) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  const int Gh = static_cast<int>((*a.n_heavy + 2047u) / 2048u);
  const int Hw = min(a.W, 32 * Gh);
  const int64_t l0 = static_cast<int64_t>(k) + s0 + 1 + lane;  // v column of slot i: l0 + 32 i
  int nvalid = 0;  // slots i < nvalid are inside [s_begin, s_end)
#pragma unroll
  for (int i = 0; i < RS; ++i) nvalid += (s0 + lane + 32 * i < a.s_end) ? 1 : 0;
  uint32_t executed = 0;
  unsigned long long fops = 0;

  double gh[RS], gl[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    gh[i] = 0.0;
    gl[i] = 0.0;
  }

  // ---- heavy region: uniform walk over the u column's bits
#pragma unroll 1
  for (int w = 0; w < Hw; ++w) {
    const unsigned long long* row = a.nx + static_cast<int64_t>(w) * n_ext;
    const unsigned long long u = __ldg(row + k);
    if (u == 0ull) continue;
    uint32_t vh[RS], vl[RS];
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const unsigned long long v = i < nvalid ? (__ldg(row + l0 + 32 * i) & u) : 0ull;
      vh[i] = static_cast<uint32_t>(v >> 32);
      vl[i] = static_cast<uint32_t>(v);
    }
    const double2* Lw = a.limbs + 64 * static_cast<int64_t>(w);
    uint32_t uh = static_cast<uint32_t>(u >> 32);
    uint32_t ul = static_cast<uint32_t>(u);
    fops += static_cast<unsigned long long>(2 * nvalid) * static_cast<unsigned>(__popcll(u));
    while (uh) {
      const int b = 31 - __clz(uh);
      const uint32_t m = 1u << b;
      uh ^= m;
      const double2 L = __ldg(Lw + 32 + b);
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const double f = unit_if(vh[i] & m);
        gh[i] = fma(L.x, f, gh[i]);
        gl[i] = fma(L.y, f, gl[i]);
      }
    }
    while (ul) {
      const int b = 31 - __clz(ul);
      const uint32_t m = 1u << b;
      ul ^= m;
      const double2 L = __ldg(Lw + b);
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const double f = unit_if(vl[i] & m);
        gh[i] = fma(L.x, f, gh[i]);
        gl[i] = fma(L.y, f, gl[i]);
      }
    }
  }

  // ---- light region: per-slot walk of the groups >= Gh (as kernel 6)
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const unsigned long long* xs = a.colsum;
  const long long ch = static_cast<long long>(a.cacc[0]);
  const long long cl = static_cast<long long>(a.cacc[1]);
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    if (i >= nvalid) break;
    const int64_t li = l0 + 32 * i;
    double ah = gh[i], al = gl[i];
#pragma unroll 1
    for (int j = Gh >> 5; j < a.NGW; ++j) {
      uint32_t gmask = __ldg(a.gm + j * n_ext + k) & __ldg(a.gm + j * n_ext + li);
      if (j == (Gh >> 5)) gmask &= 0xffffffffu >> (Gh & 31);
      while (gmask) {
        const int gi = __clz(gmask);
        gmask ^= 0x80000000u >> gi;
        const int g = 32 * j + gi;
        const int64_t gb = static_cast<int64_t>(g) * n_ext;
        const uint32_t ou = __ldg(a.occ + gb + k);
        const uint32_t ov = __ldg(a.occ + gb + li);
        uint32_t o = ou & ov;
        if (!o) continue;
        const uint32_t bu = __ldg(a.base + gb + k);
        const uint32_t bv = __ldg(a.base + gb + li);
        const double2* Lg = a.limbs + static_cast<int64_t>(g) * 2048;
        do {
          const int w = __clz(o);
          o ^= 0x80000000u >> w;
          const uint32_t above = ~(0xffffffffu >> w);
          const unsigned long long x = __ldg(a.packed + (bu + __popc(ou & above))) &
                                       __ldg(a.packed + (bv + __popc(ov & above)));
          uint32_t xh = static_cast<uint32_t>(x >> 32);
          uint32_t xl = static_cast<uint32_t>(x);
          executed += __popc(xh) + __popc(xl);
          const double2* Lw = Lg + 64 * w;
          while (xh) {
            const int b = 31 - __clz(xh);
            xh ^= 1u << b;
            const double2 L = __ldg(Lw + 32 + b);
            ah += L.x;
            al += L.y;
          }
          while (xl) {
            const int b = 31 - __clz(xl);
            xl ^= 1u << b;
            const double2 L = __ldg(Lw + b);
            ah += L.x;
            al += L.y;
          }
        } while (o);
      }
    }
    const int s = s0 + lane + 32 * i;
    const int lm = li >= n ? static_cast<int>(li - n) : static_cast<int>(li);
    const long long Gh_ = static_cast<long long>(ah);
    const long long Gl_ = static_cast<long long>(al);
    const long long th = static_cast<long long>(xs[2 * n + k] + xs[2 * n + lm]) + ch - Gh_;
    const long long tl = static_cast<long long>(xs[3 * n + k] + xs[3 * n + lm]) + cl - Gl_;
    const long long dh = static_cast<long long>(xs[k] + xs[lm]) - 2 * Gh_;
    const long long dl = static_cast<long long>(xs[n + k] + xs[n + lm]) - 2 * Gl_;
    const __int128 tv = (static_cast<__int128>(th) << a.lo_bits) + tl;
    const __int128 dv = (static_cast<__int128>(dh) << a.lo_bits) + dl;
    const Real t = static_cast<Real>(i2_fixed_to_double(tv, a.scale));
    Real d = static_cast<Real>(i2_fixed_to_double(dv, a.scale));
    if (a.finalize) d = t == Real(0) ? Real(0) : d / t;
    const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
    dist[off] = d;
    tot[off] = t;
  }
  fops += 2ull * executed;
  if (a.exec_updates) {
    unsigned long long e = executed;
    for (int off = 16; off > 0; off >>= 1) {
      e += __shfl_down_sync(0xffffffffu, e, off);
      fops += __shfl_down_sync(0xffffffffu, fops, off);
    }
    if (lane == 0) {
      atomicAdd(a.exec_updates, e);
      atomicAdd(fp_ops, fops);
    }
  }
}

}  // namespace sf
