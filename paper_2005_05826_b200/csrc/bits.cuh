// Small device helpers shared by the stripe kernels: bit scans, 0/1 factors
// and the exact fixed-point -> floating-point conversion.
#pragma once

#include <cstdint>

// Streaming (evict-first) loads/stores for the write-once / read-once slot
// arrays (light sums, final stripes), so they do not evict reused operands
// from L2. -DSF_LIGHT_STREAM=0 builds the plain-access A/B library.
#ifndef SF_LIGHT_STREAM
#define SF_LIGHT_STREAM 1
#endif

namespace sf {

// bfind: position of the most significant set bit (x != 0).
__device__ __forceinline__ int msb_pos(uint32_t x) {
  int b;
  asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(x));
  return b;
}

// (hit ? 1.0 : 0.0) built from its high word only: one SEL. acc = fma(L, f,
// acc) then adds L exactly (f = 1) or leaves acc unchanged (f = 0): one DFMA
// per limb and slot instead of the DADD + 2 FSEL ptxas emits for a
// conditional add (it if-converts predicated FP64 adds).
__device__ __forceinline__ double unit_if(uint32_t hit) {
  return __hiloint2double(hit ? 0x3ff00000 : 0, 0);
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Correctly rounded Real of (m + s) * 2^e, m < 2^128 an integer, s in {0, 1}
// a sticky flag for nonzero bits below m (only ever set when m >= 2^64, so
// the sticky bit lands far below the rounding position).
template <class Real>
__device__ __forceinline__ Real u128_to_real(unsigned __int128 m, bool sticky, int e) {
  const unsigned long long hi = static_cast<unsigned long long>(m >> 64);
  const unsigned long long lo = static_cast<unsigned long long>(m);
  unsigned long long top;
  int sh;
  if (hi == 0ull) {
    top = lo;
    sh = 0;
  } else {
    sh = 64 - __clzll(static_cast<long long>(hi));
    top = static_cast<unsigned long long>(m >> sh);
    const unsigned long long rest = sh == 64 ? lo : (lo & ((1ull << sh) - 1ull));
    if (rest != 0ull) sticky = true;
  }
  if (sticky) top |= 1ull;
  const int x = sh + e;
  if (sizeof(Real) == 8) {
    const double r = __ull2double_rn(top);
    // exact power-of-two scaling while 2^x and the result stay normal
    if (x >= -1022 && x <= 1023 && (top == 0ull || x + 64 <= 1023)) {
      const double r2 = r * __longlong_as_double(static_cast<long long>(1023 + x) << 52);
      if (top == 0ull || r2 >= 0x1p-1022) return static_cast<Real>(r2);
    }
    return static_cast<Real>(ldexp(r, x));
  }
  return static_cast<Real>(ldexpf(__ull2float_rn(top), x));
}

// Correctly rounded Real of (V0 2^vb + V1) 2^-(scale + vb): two fixed-point
// levels (V0, V1 >= 0 below 2^126, vb <= 63) as one exact value of up to
// 190 bits held in three 64-bit limbs, rounded once from its leading 64 bits
// with a sticky bit for the rest.
template <class Real>
__device__ __forceinline__ Real two_levels_to_real(unsigned __int128 V0, unsigned __int128 V1, int vb, int scale) {
  // w = V0 << vb as a 192-bit value w2:w1:w0 (low 128 bits from the shift,
  // the top from V0 >> (128 - vb)), then + V1
  const unsigned __int128 lo128 = V0 << vb;
  unsigned long long w0 = static_cast<unsigned long long>(lo128);
  unsigned long long w1 = static_cast<unsigned long long>(lo128 >> 64);
  unsigned long long w2 = vb ? static_cast<unsigned long long>(V0 >> (128 - vb)) : 0ull;
  // + V1
  const unsigned __int128 s0 = static_cast<unsigned __int128>(w0) + static_cast<unsigned long long>(V1);
  w0 = static_cast<unsigned long long>(s0);
  const unsigned __int128 s1 = static_cast<unsigned __int128>(w1) + static_cast<unsigned long long>(V1 >> 64) +
                               static_cast<unsigned long long>(s0 >> 64);
  w1 = static_cast<unsigned long long>(s1);
  w2 += static_cast<unsigned long long>(s1 >> 64);
  const int e = -(scale + vb);
  if (w2 == 0ull) return u128_to_real<Real>((static_cast<unsigned __int128>(w1) << 64) | w0, false, e);
  // leading 128 bits of the 192-bit value, sticky for what is shifted out
  const int sh = 64 - __clzll(static_cast<long long>(w2));  // 1..64
  const unsigned __int128 top = (static_cast<unsigned __int128>(w2) << (128 - sh)) |
                                (static_cast<unsigned __int128>(w1) << (64 - sh)) |
                                (sh == 64 ? 0 : static_cast<unsigned __int128>(w0 >> sh));
  const unsigned long long rest = sh == 64 ? w0 : (w0 & ((1ull << sh) - 1ull));
  return u128_to_real<Real>(top, rest != 0ull, e + sh);
}

// Exact value v * 2^-scale (v >= 0, a 128-bit integer), correctly rounded.
template <class Real>
__device__ __forceinline__ Real fixed_to_real(__int128 v, int scale) {
  return u128_to_real<Real>(static_cast<unsigned __int128>(v), false, -scale);
}

}  // namespace sf
