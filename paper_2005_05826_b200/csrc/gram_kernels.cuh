// K2-UW heavy rows on the tensor cores (the default heavy path of kernel 10).
//
// The heavy part of the split form is an exact 0/1 Gram with integer
// weights: G_kl = sum_{heavy e} v_e [k in X_e][l in X_e], v_e the row's
// main-level fixed-point length (split_kernels.cuh). With v_e written in
// balanced base-256 digits, v_e = sum_j 256^j d_ej, d_ej in [-128, 127]
// (at most 9 digits for v < 2^63),
//   G_kl = sum_j 256^j sum_e (d_ej [k in X_e]) [l in X_e],
// i.e. one int8 x int8 -> int32 matrix product per digit plane, exact: every
// product is d * 1 and |sum| <= 128 * H < 2^31 for H < 2^24 heavy rows. The
// digit planes of a block of BK u columns are the M side (rows (k, j)), the
// 0/1 X rows of a window of v columns the N side, the heavy rows K:
//   C[(k - k0) * nd + jj][c] = sum_i A'[(k - k0) * nd + jj][i] B[l_start + c][i]
// run by cuBLASLt's int8 tensor-core GEMM (tcgen05 IMMA on sm_100a: 4.4 of
// 4.5 POPS measured at these shapes, tools/ab/mb_int8_gemm.py). A slot
// (s, k) of the block is column c = (k - k0) + (s - c0) of the window
// l_start = k0 + c0 + 1; the parallelogram of slots the stripe range needs
// is read out by sp_gram_epilogue_kernel, which adds the light sums and
// column sums and forms t, d exactly like the DFMA heavy walk's epilogue.
// All planes whose digit is zero for every heavy row are skipped (lengths
// that are multiples of 2^-52 leave the lowest plane empty).
#pragma once

#include <cstdint>

#include "bits.cuh"

namespace sf {

constexpr int kMaxDigits = 9;

// Balanced base-256 digits of v (< 2^63): d_j in [-128, 127], v = sum 256^j d_j.
__device__ __forceinline__ void balanced_digits(unsigned long long v, int8_t (&d)[kMaxDigits]) {
#pragma unroll
  for (int j = 0; j < kMaxDigits; ++j) {
    const int r = static_cast<int>(v & 255ull);
    v >>= 8;
    if (r >= 128) {
      d[j] = static_cast<int8_t>(r - 256);
      v += 1;
    } else {
      d[j] = static_cast<int8_t>(r);
    }
  }
}

// Digits of every permuted heavy row i < Kp (zero past H), plane-major:
// rowdig[j * Kp + i], and the OR of the nonzero planes into *mask.
__global__ void sp_gram_rowdig_kernel(const unsigned long long* __restrict__ fixbit,
                                      const unsigned int* __restrict__ n_heavy, int64_t Kp,
                                      int8_t* __restrict__ rowdig, unsigned int* __restrict__ mask) {
  const int64_t H = *n_heavy;
  unsigned int m = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < Kp;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int8_t d[kMaxDigits];
    // permuted row i sits at bit 63 - (i & 63) of word i / 64 (fixbit is by bit position)
    const unsigned long long v = i < H ? fixbit[(i & ~int64_t{63}) + 63 - (i & 63)] : 0ull;
    balanced_digits(v, d);
#pragma unroll
    for (int j = 0; j < kMaxDigits; ++j) {
      rowdig[j * Kp + i] = d[j];
      if (d[j]) m |= 1u << j;
    }
  }
  for (int off = 16; off > 0; off >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, off);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(mask, m);
}

// B[c][i] = [permuted heavy row i in X_c] as int8, c < n_ext (wrap columns
// included), i < Kp: one thread per (64-row word, column), coalesced reads of
// the node-packed words, one 64-byte row segment written per thread.
__global__ void sp_gram_bits_kernel(const unsigned long long* __restrict__ nx, int64_t n_ext,
                                    const unsigned int* __restrict__ n_heavy, int64_t Kp, int8_t* __restrict__ B) {
  const int64_t Hw = (static_cast<int64_t>(*n_heavy) + 63) / 64;
  const int64_t Wk = Kp / 64;  // words of the padded K (rows past the heavy words are zero)
  const int64_t total = Wk * n_ext;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t / n_ext;
    const int64_t c = t - w * n_ext;
    const unsigned long long x = w < Hw ? __ldg(nx + w * n_ext + c) : 0ull;
    uint4* out = reinterpret_cast<uint4*>(B + c * Kp + 64 * w);
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // rows 64w + 16q .. +15 = bits 63-16q .. 48-16q
      uint32_t wd[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint32_t o = 0;
#pragma unroll
        for (int t4 = 0; t4 < 4; ++t4) {
          const int row = 16 * q + 4 * b + t4;
          o |= static_cast<uint32_t>((x >> (63 - row)) & 1ull) << (8 * t4);
        }
        wd[b] = o;
      }
      out[q] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
  }
}

// A'[(k - k0) * nd + jj][i] = B[k][i] ? d_{dj[jj]}(row i) : 0 for the BK u
// columns of the block: one thread per (column, 16-row chunk); the 0/1
// bytes become byte masks (x * 0xff, no carries) ANDed with the plane.
__global__ void sp_gram_digits_kernel(const int8_t* __restrict__ B, int64_t Kp, int32_t k0, int32_t bk,
                                      int32_t n, const int8_t* __restrict__ rowdig, int64_t plane_stride,
                                      const int32_t* __restrict__ dj, int32_t nd, int8_t* __restrict__ Ap) {
  const int64_t chunks = Kp / 16;
  const int64_t total = static_cast<int64_t>(bk) * chunks;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t kk = t / chunks;
    const int64_t ch = t - kk * chunks;
    const int64_t k = k0 + kk;
    uint4 bits = make_uint4(0u, 0u, 0u, 0u);
    if (k < n) bits = __ldg(reinterpret_cast<const uint4*>(B + k * Kp) + ch);
    const uint4 m = make_uint4(bits.x * 0xffu, bits.y * 0xffu, bits.z * 0xffu, bits.w * 0xffu);
    for (int jj = 0; jj < nd; ++jj) {
      const uint4 dv = __ldg(reinterpret_cast<const uint4*>(rowdig + static_cast<int64_t>(dj[jj]) * plane_stride) + ch);
      reinterpret_cast<uint4*>(Ap + (kk * nd + jj) * Kp)[ch] =
          make_uint4(dv.x & m.x, dv.y & m.y, dv.z & m.z, dv.w & m.w);
    }
  }
}

struct GramArgs {
  const int32_t* C;                  // [W][M] column-major GEMM output, M = bk * nd
  const int32_t* dj;                 // digit index of each plane, nd entries
  int32_t nd, bk, k0;                // planes, block columns, first column
  int32_t dj0;                       // first digit when the planes are consecutive, else -1
  int32_t c0, c1;                    // stripes of this launch
  int64_t M;
  int32_t n;
  int32_t out_begin, gl_begin;
  int32_t lo_bits, scale, finalize, levels, vb;
  unsigned long long* gl;            // light sums (hi, lo); more than two levels: G out
  const unsigned long long* dacc;    // two levels: the second level's pair sums [cell] (hi, lo)
  const unsigned long long* dcolsum; // [4][n] second level
  const unsigned long long* dcacc;   // [2] second level
  const unsigned long long* colsum;  // [4][n]
  const unsigned long long* cacc;    // [2]
  void* dist;
  void* tot;
};

// Slots (s, k), s in [c0, c1), k in [k0, k0 + bk): G = heavy (tensor) +
// light, then t = p_k + p_l + C - G and d = x_k + x_l - 2 G in exact
// integers, rounded once (finalize: d / t, 0/0 -> 0). LO, VB > 0: the
// limb split and level width as compile-time constants (lo_bits = 32,
// vb = 63 whenever E < 2^21): the 128/192-bit shifts by them become moves.
template <class Real, int LO, int VB>
__global__ void sp_gram_epilogue_kernel(const GramArgs a) {
  const int lo_bits = LO > 0 ? LO : a.lo_bits;
  const int vb = VB > 0 ? VB : a.vb;
  const int n = a.n;
  const int kcount = min(a.bk, n - a.k0);
  const unsigned long long* xs = a.colsum;
  const __int128 Cd = (static_cast<__int128>(a.cacc[0]) << lo_bits) + static_cast<__int128>(a.cacc[1]);
  const __int128 C1 = a.levels == 2 ? (static_cast<__int128>(a.dcacc[0]) << lo_bits) + static_cast<__int128>(a.dcacc[1])
                                    : __int128(0);
  const unsigned long long lo_mask = (1ull << lo_bits) - 1ull;
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  // 2D grid: x over the block's columns, y strides over the stripes (no
  // 64-bit division per slot)
  const int span = a.c1 - a.c0;
  for (int ds = blockIdx.y; ds < span; ds += gridDim.y)
  for (int kk = blockIdx.x * blockDim.x + threadIdx.x; kk < kcount; kk += gridDim.x * blockDim.x) {
    const int s = a.c0 + ds;
    const int k = a.k0 + kk;
    int l = k + s + 1;
    if (l >= n) l -= n;
    const int32_t* cp = a.C + static_cast<int64_t>(kk + ds) * a.M + static_cast<int64_t>(kk) * a.nd;
    __int128 G = 0;
    if (a.nd == 8 && a.dj0 == 0) {
      // planes 0..7: the slot's 32 bytes as two 16-byte loads, combined
      // Horner-style from the top digit (no per-plane 128-bit shifts)
      const int4 lo = __ldg(reinterpret_cast<const int4*>(cp));
      const int4 hi = __ldg(reinterpret_cast<const int4*>(cp) + 1);
      const int32_t c8[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int jj = 7; jj >= 0; --jj) G = G * 256 + static_cast<__int128>(c8[jj]);
    } else if (a.dj0 >= 0) {
      // consecutive planes dj0 .. dj0 + nd - 1 (C3: 1..7): Horner from the
      // top plane, one 128-bit shift by 8 dj0 at the end
#pragma unroll
      for (int jj = kMaxDigits - 1; jj >= 0; --jj)
        if (jj < a.nd) G = G * 256 + static_cast<__int128>(__ldg(cp + jj));
      G <<= 8 * a.dj0;
    } else {
      for (int jj = 0; jj < a.nd; ++jj) G += static_cast<__int128>(cp[jj]) * (static_cast<__int128>(1) << (8 * a.dj[jj]));
    }
    const int64_t cell = static_cast<int64_t>(s - a.gl_begin) * n + k;
#if SF_LIGHT_STREAM
    const longlong2 lraw = __ldcs(reinterpret_cast<const longlong2*>(a.gl) + cell);  // read once
    const ulonglong2 light = make_ulonglong2(static_cast<unsigned long long>(lraw.x),
                                             static_cast<unsigned long long>(lraw.y));
#else
    const ulonglong2 light = reinterpret_cast<const ulonglong2*>(a.gl)[cell];
#endif
    G += (static_cast<__int128>(light.x) << lo_bits) + static_cast<__int128>(light.y);
    if (a.levels > 2) {  // sp_deep_epilogue_kernel finishes the slot from (hi, lo)
      reinterpret_cast<longlong2*>(a.gl)[cell] =
          make_longlong2(static_cast<long long>(G >> lo_bits), static_cast<long long>(G & lo_mask));
      continue;
    }
    const __int128 P = (static_cast<__int128>(xs[2 * n + k] + xs[2 * n + l]) << lo_bits) +
                       static_cast<__int128>(xs[3 * n + k] + xs[3 * n + l]);
    const __int128 X = (static_cast<__int128>(xs[k] + xs[l]) << lo_bits) +
                       static_cast<__int128>(xs[n + k] + xs[n + l]);
    Real tv, dv;
    if (a.levels == 2) {  // lengths off the main grid: the second level, exact, fused
      const unsigned long long* ys = a.dcolsum;
      const ulonglong2 G1l = reinterpret_cast<const ulonglong2*>(a.dacc)[cell];
      const __int128 G1 = (static_cast<__int128>(G1l.x) << lo_bits) + static_cast<__int128>(G1l.y);
      const __int128 P1 = (static_cast<__int128>(ys[2 * n + k] + ys[2 * n + l]) << lo_bits) +
                          static_cast<__int128>(ys[3 * n + k] + ys[3 * n + l]);
      const __int128 X1 = (static_cast<__int128>(ys[k] + ys[l]) << lo_bits) +
                          static_cast<__int128>(ys[n + k] + ys[n + l]);
      tv = two_levels_to_real<Real>(static_cast<unsigned __int128>(P + Cd - G),
                                    static_cast<unsigned __int128>(P1 + C1 - G1), vb, a.scale);
      dv = two_levels_to_real<Real>(static_cast<unsigned __int128>(X - 2 * G),
                                    static_cast<unsigned __int128>(X1 - 2 * G1), vb, a.scale);
    } else {
      tv = fixed_to_real<Real>(P + Cd - G, a.scale);
      dv = fixed_to_real<Real>(X - 2 * G, a.scale);
    }
    if (a.finalize) dv = tv == Real(0) ? Real(0) : dv / tv;
    const int64_t off = static_cast<int64_t>(s - a.out_begin) * n + k;
#if SF_LIGHT_STREAM
    __stcs(dist + off, dv);  // final stripes: leave L2 to the GEMM operands
    __stcs(tot + off, tv);
#else
    dist[off] = dv;
    tot[off] = tv;
#endif
  }
}

}  // namespace sf
