// Small device helpers shared by the stripe kernels: bit scans, 0/1 factors
// and the exact fixed-point -> floating-point conversion.
#pragma once

#include <cstdint>

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
  if (sizeof(Real) == 8) return static_cast<Real>(ldexp(__ull2double_rn(top), sh + e));
  return static_cast<Real>(ldexpf(__ull2float_rn(top), sh + e));
}

// Exact value v * 2^-scale (v >= 0, a 128-bit integer), correctly rounded.
template <class Real>
__device__ __forceinline__ Real fixed_to_real(__int128 v, int scale) {
  return u128_to_real<Real>(static_cast<unsigned __int128>(v), false, -scale);
}

}  // namespace sf
