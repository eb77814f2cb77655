// K2 (stripe update), K3 (finalize), K4 (condense) for sm_100a.
//
// K2 replaces run_naive / run_batched / run_tiled + update_entry
// (kernels.hpp:55-172). Every (stripe s, slot k) accumulator sums its rows in
// postorder with one fixed operation sequence, independent of tiling, chunk
// size, GPU count or stripe range -> results are deterministic and
// partition-independent, like the reference (README.md:36-44).
//
// Dense register-tiled kernel ("stripe_dense"):
//  - CTA tile = TK samples x TS stripes; warp tile = RK consecutive samples
//    (warp-uniform) x 32*RS stripes (lane l owns stripes sw + l*RS + i);
//  - a block of RB postorder rows is staged in shared memory per step: the
//    u window [k0, k0+TK) and the Hankel v window [k0+s0+1, k0+s0+TK+TS-1)
//    (wrapped mod n), the v window de-interleaved by residue mod RS so that
//    lane l's run (q + l*RS + m) hits consecutive words (no bank conflicts);
//  - each thread keeps RS x RK accumulators (x2 for ratio metrics) in
//    registers and reuses each staged v across the RS x RK anti-diagonal
//    (RK + RS - 1 loads for RK*RS updates), each u across RS stripes;
//  - a staged row whose whole CTA window is zero adds exactly +0.0 to every
//    accumulator in every metric, so it is skipped (bit-exact);
//  - unweighted rows arrive as presence bits and expand to 0/1 at staging.
#pragma once

#include <cstdint>

namespace sf {

enum : int { kUW = 1, kWU = 2, kWN = 3, kGen = 4 };  // kGen: generalized (not in the reference)
enum : int { kSrcBits = 0, kSrcF64 = 1, kSrcF32 = 2 };

template <class Real>
__device__ __forceinline__ Real fma_r(Real a, Real b, Real c);
template <>
__device__ __forceinline__ double fma_r<double>(double a, double b, double c) { return fma(a, b, c); }
template <>
__device__ __forceinline__ float fma_r<float>(float a, float b, float c) { return fmaf(a, b, c); }

template <class Real>
__device__ __forceinline__ Real mul_add_rn(Real a, Real b, Real c);  // c + a*b, two roundings
template <>
__device__ __forceinline__ double mul_add_rn<double>(double a, double b, double c) {
  return __dadd_rn(c, __dmul_rn(a, b));
}
template <>
__device__ __forceinline__ float mul_add_rn<float>(float a, float b, float c) {
  return __fadd_rn(c, __fmul_rn(a, b));
}

// update_entry (kernels.hpp:55-66). For unweighted 0/1 rows |u-v| and
// max(u,v) are 0 or 1, so the product is exact and fma == mul+add bitwise.
// Weighted metrics use one fma per accumulator unless EXACT (two roundings,
// bit-identical to the reference's no-FMA x86-64 build).
//
// The reference writes |u-v| as `diff < 0 ? -diff : diff` and max as
// `u > v ? u : v`; they differ from fabs/fmax only for NaN and signed zeros.
// Embedding values here are finite and >= +0 (validated counts, positive
// totals), and a -0 term cannot change an accumulator that starts at +0 and
// only grows, so fabs/fmax give identical sums — and map to the |x| operand
// modifier and DMNMX instead of DSETP+FSEL pairs (4 FP-pipe ops per update).
__device__ __forceinline__ double abs_r(double x) { return fabs(x); }
__device__ __forceinline__ float abs_r(float x) { return fabsf(x); }
__device__ __forceinline__ double max_r(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float max_r(float a, float b) { return fmaxf(a, b); }

template <int M, bool EXACT, class Real>
__device__ __forceinline__ void update_entry(Real u, Real v, Real len, Real& d, Real& t) {
  const Real diff = abs_r(u - v);
  if (EXACT && M != kUW)
    d = mul_add_rn(diff, len, d);
  else
    d = fma_r(diff, len, d);
  if constexpr (M == kUW) {
    t = fma_r(max_r(u, v), len, t);
  } else if constexpr (M == kWN) {
    if (EXACT)
      t = mul_add_rn(u + v, len, t);
    else
      t = fma_r(u + v, len, t);
  }
}

// Generalized UniFrac (alpha), per present row — not in the reference
// (parity unpinned; oracle/stripefrac_oracle.c states the published form):
//   s = u + v; if (s != 0) { w = s^alpha * L; d += w * (|u-v| / s); t += w; }
__device__ __forceinline__ double pow_r(double x, double a) { return pow(x, a); }
__device__ __forceinline__ float pow_r(float x, float a) { return powf(x, a); }

// x^alpha for x > 0 with the common exponents on their exact / correctly
// rounded forms (sqrt is correctly rounded, CUDA pow is within 2 ulp): the
// branch is warp-uniform (alpha is a launch argument).
template <class Real>
__device__ __forceinline__ Real pow_alpha(Real x, Real alpha) {
  if (alpha == Real(1)) return x;
  if (alpha == Real(0.5)) return sqrt(x);
  if (alpha == Real(0)) return Real(1);
  if (alpha == Real(2)) return x * x;
  return pow_r(x, alpha);
}

template <bool EXACT, class Real>
__device__ __forceinline__ void update_generalized(Real u, Real v, Real len, Real alpha, Real& d, Real& t) {
  const Real s = u + v;
  if (s != Real(0)) {
    const Real w = pow_alpha(s, alpha) * len;
    const Real q = abs_r(u - v) / s;
    d = EXACT ? mul_add_rn(w, q, d) : fma_r(w, q, d);
    t += w;
  }
}

struct StripeArgs {
  const void* emb;        // chunk rows: bits (uint32 words) / fp64 / fp32 values
  int64_t row_stride;     // in words or values
  const double* lens;     // [C] branch lengths of the chunk rows
  int32_t C;              // rows in the chunk
  int32_t n;              // samples
  int32_t s_begin;        // absolute first stripe held by dist/tot
  int32_t s_end;          // absolute end stripe
  void* dist;             // (s_end - s_begin) x n accumulators
  void* tot;              // same, or null for WU
  unsigned long long* exec_updates;  // executed node x slot updates (may be null)
};

template <int SRC, class Real>
__device__ __forceinline__ Real load_emb(const void* emb, int64_t row_off, int smp) {
  if constexpr (SRC == kSrcBits) {
    const uint32_t w = static_cast<const uint32_t*>(emb)[row_off + (smp >> 5)];
    return ((w >> (smp & 31)) & 1u) ? Real(1) : Real(0);
  } else if constexpr (SRC == kSrcF64) {
    return static_cast<Real>(static_cast<const double*>(emb)[row_off + smp]);
  } else {
    return static_cast<Real>(static_cast<const float*>(emb)[row_off + smp]);
  }
}

template <int M, class Real, int SRC, bool EXACT, int RK, int RS, int NWK, int NWS, int RB>
__global__ void __launch_bounds__(32 * NWK * NWS)
    stripe_dense_kernel(const StripeArgs a) {
  constexpr int NW = NWK * NWS;
  constexpr int TK = NWK * RK;
  constexpr int TS = NWS * 32 * RS;
  constexpr int VW = TK + TS - 1;
  constexpr int VSTR = (VW + RS - 1) / RS;
  constexpr bool kHasT = M != kWU;
  static_assert((RS & (RS - 1)) == 0, "RS must be a power of two");

  __shared__ Real sv[RB][RS][VSTR];
  __shared__ Real su[RB][TK];
  __shared__ Real sl[RB];
  __shared__ int sflag[RB];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wk = warp % NWK;
  const int ws = warp / NWK;
  const int n = a.n;
  const int k0 = blockIdx.x * TK;
  const int s0 = a.s_begin + blockIdx.y * TS;
  const int P0 = k0 + s0 + 1;  // first v position of the CTA window
  const int q = wk * RK + ws * 32 * RS;

  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);

  // accumulators: stripe s_i = s0 + ws*32*RS + lane*RS + i, sample k_j = k0 + wk*RK + j
  Real d[RS][RK];
  Real t[RS][RK];
  const int sbase = s0 + ws * 32 * RS + lane * RS;
  const int kbase = k0 + wk * RK;
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    const int s = sbase + i;
#pragma unroll
    for (int j = 0; j < RK; ++j) {
      const int k = kbase + j;
      const bool ok = s < a.s_end && k < n;
      const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
      d[i][j] = ok ? dist[off] : Real(0);
      if constexpr (kHasT) t[i][j] = ok ? tot[off] : Real(0);
    }
  }

  int active_rows = 0;
  for (int rb = 0; rb < a.C; rb += RB) {
    __syncthreads();
    // ---- stage RB rows: each warp stages whole rows
    for (int rr = warp; rr < RB; rr += NW) {
      const int r = rb + rr;
      bool nz = false;
      if (r < a.C) {
        const int64_t roff = static_cast<int64_t>(r) * a.row_stride;
        for (int e = lane; e < RS * VSTR; e += 32) {
          Real val = Real(0);
          if (e < VW) {
            int pos = P0 + e;
            while (pos >= n) pos -= n;  // stripe_pair wrap (stripes.cpp:23-28)
            val = load_emb<SRC, Real>(a.emb, roff, pos);
          }
          sv[rr][e % RS][e / RS] = val;
          nz |= val != Real(0);
        }
        for (int e = lane; e < TK; e += 32) {
          const int k = k0 + e;
          const Real val = k < n ? load_emb<SRC, Real>(a.emb, roff, k) : Real(0);
          su[rr][e] = val;
          nz |= val != Real(0);
        }
        if (lane == 0) sl[rr] = static_cast<Real>(a.lens[r]);
      }
      nz = __any_sync(0xffffffffu, nz);
      if (lane == 0) sflag[rr] = nz ? 1 : 0;
    }
    __syncthreads();
    // ---- accumulate the staged rows in postorder
    const int rows_here = min(RB, a.C - rb);
    for (int rr = 0; rr < rows_here; ++rr) {
      if (!sflag[rr]) continue;  // all-zero window: +0.0 everywhere
      ++active_rows;
      const Real len = sl[rr];
      Real u[RK];
#pragma unroll
      for (int j = 0; j < RK; ++j) u[j] = su[rr][wk * RK + j];
      const Real* vrow = &sv[rr][0][0];
#pragma unroll
      for (int m = 0; m < RK + RS - 1; ++m) {
        const int rel = q + m;
        const Real v = vrow[(rel & (RS - 1)) * VSTR + (rel / RS) + lane];
#pragma unroll
        for (int i = 0; i < RS; ++i) {
          const int j = m - i;
          if (j >= 0 && j < RK) update_entry<M, EXACT, Real>(u[j], v, len, d[i][j], t[i][j]);
        }
      }
    }
  }

  // ---- commit (one write per slot per chunk, like batched/tiled)
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    const int s = sbase + i;
#pragma unroll
    for (int j = 0; j < RK; ++j) {
      const int k = kbase + j;
      if (s < a.s_end && k < n) {
        const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
        dist[off] = d[i][j];
        if constexpr (kHasT) tot[off] = t[i][j];
      }
    }
  }
  if (a.exec_updates && tid == 0) {
    const int kk = min(TK, n - k0);
    const int ss = min(TS, a.s_end - s0);
    atomicAdd(a.exec_updates, static_cast<unsigned long long>(active_rows) *
                                  static_cast<unsigned long long>(kk) *
                                  static_cast<unsigned long long>(ss));
  }
}

// K3: finalize (kernels.hpp:251-259): d <- (t == 0) ? 0 : d / t, IEEE divide.
template <class Real>
__global__ void finalize_kernel(Real* __restrict__ dist, const Real* __restrict__ tot,
                                int64_t count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const Real t = tot[i];
    dist[i] = t == Real(0) ? Real(0) : dist[i] / t;
  }
}

// K4: condense one finalized stripe part into the n x n fp64 matrix
// (stripes.cpp:68-129). Slot (s,k) is pair (k, (k+s+1) mod n); for even n
// the second copies in the last stripe are compared with their first copy
// (slot k - n/2 of the same stripe) instead of written.
template <class Real>
__global__ void condense_kernel(const Real* __restrict__ dist, int32_t n, int32_t start,
                                int32_t stop, double* __restrict__ out,
                                int* __restrict__ bad) {
  const int S = n / 2;
  const bool even = (n % 2) == 0;
  const int64_t count = static_cast<int64_t>(stop - start) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = start + static_cast<int>(i / n);
    const int k = static_cast<int>(i % n);
    const Real v = dist[i];
    if (even && s == S - 1 && k >= n / 2) {
      const Real first = dist[i - n / 2];
      bool agree;
      if constexpr (sizeof(Real) == 8) {
        agree = first == v;
      } else {
        const float a = static_cast<float>(first), b = static_cast<float>(v);
        agree = fabsf(a - b) <= 1e-6f * fmaxf(fabsf(a), fabsf(b));
      }
      if (!agree) atomicExch(bad, 1);
      continue;
    }
    int l = k + s + 1;
    if (l >= n) l -= n;
    out[static_cast<int64_t>(k) * n + l] = static_cast<double>(v);
    out[static_cast<int64_t>(l) * n + k] = static_cast<double>(v);
  }
}

// Zero diagonal of the n x n matrix (condense writes every off-diagonal entry).
__global__ void diagonal_zero_kernel(double* __restrict__ out, int32_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i * n + i] = 0.0;
}

}  // namespace sf
