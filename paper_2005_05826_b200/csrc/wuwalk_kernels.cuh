// K2-W, u-walk form (kernel 12, the default for the weighted metrics and the
// generalized extension; kernel 11 remains the bitwise path).
//
// Kernel 11 walks, per slot, the union of both samples' present rows: lanes
// of a warp walk different rows (ncu: 9.5 of 32 lanes active). Here the walk
// is warp-uniform, like the unweighted split kernel: a warp owns one u column
// k and 32*RS slots (v columns l = k+s+1), walks the rows present in u in
// postorder, and every lane updates each of its slots:
//   v absent : d += fl(L*u)                  (the reference's term, |u-0| = u)
//   v present: d += |u - v| * L, and B += fl(L*v)   (B compensated)
// Rows present in v only add fl(L*v) each, i.e. sum_{v present} fl(L*v) -
// sum_{both} fl(L*v) = A_l - B: A_l is a per-column sum, B the per-slot sum
// of the same terms over the shared rows, both double-double (TwoSum), so
// the difference is accurate to ~1e-32 relative to A_l and identical samples
// give exactly 0. WN's total is separable: t = A_k + A_l.
// Generalized (alpha): absent rows add fl(L*u^a) to d and t (precomputed in a
// second pool), present rows w = (u+v)^a L, d += w |u-v|/(u+v), t += w, and
// the v-only rows add A^a_l - B^a to both — pow runs only on shared rows.
//
// Layout (whole problem resident; built chunk by chunk from the K1 rows):
//   nb[w][c], off[w][c]  32-row presence words and GLOBAL pool offsets
//                        (row 32w+r at bit 31-r), columns extended past n;
//   pool[], poola[]      present values (Real) and, generalized, fl(L*v^a).
// Results are within 1e-12 (fp64) of the reference's sequential sums: same
// terms, different (more accurate) summation.
#pragma once

#include <cstdint>

#include "bits.cuh"
#include "stripe_kernels.cuh"
#include "wsparse_kernels.cuh"

namespace sf {

// ---- double-double helpers (TwoSum: exact error of a + b)
__device__ __forceinline__ void dd_add(double& hi, double& lo, double b) {
  const double s = hi + b;
  const double bb = s - hi;
  const double e = (hi - (s - bb)) + (b - bb);
  hi = s;
  lo += e;
}

// (ah + al) - (bh + bl), rounded once to double.
__device__ __forceinline__ double dd_diff(double ah, double al, double bh, double bl) {
  const double s = ah - bh;
  const double bb = s - ah;
  const double e = (ah - (s - bb)) + (-bh - bb);
  return s + (e + (al - bl));
}

// Running pool base: chunk total (before the fill globalizes the offsets).
__global__ void wu_chunk_total_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                      int64_t last, unsigned long long* __restrict__ total) {
  *total = static_cast<unsigned long long>(off[last]) + cnt[last];
}
__global__ void wu_advance_base_kernel(unsigned long long* __restrict__ base,
                                       const unsigned long long* __restrict__ total) {
  *base += *total;
}

// Values of one chunk into the global pool; offsets made global in place.
template <class Real, bool GEN>
__global__ void wu_fill_kernel(const double* __restrict__ emb, int64_t stride, int32_t n, int32_t Wc,
                               int64_t n_ext, const uint32_t* __restrict__ nb, uint32_t* __restrict__ off,
                               const unsigned long long* __restrict__ base, const double* __restrict__ lens,
                               double alpha, Real* __restrict__ pool, Real* __restrict__ poola) {
  const int64_t total = static_cast<int64_t>(Wc) * n;
  const unsigned long long b0 = *base;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / n;
    const int64_t c = i - w * n;
    const int64_t cell = w * n_ext + c;
    const uint64_t at = b0 + off[cell];
    off[cell] = static_cast<uint32_t>(at);
    uint32_t bits = nb[cell];
    const double* col = emb + 32 * w * stride + c;
    uint64_t q = at;
    while (bits) {
      const int r = __clz(bits);
      bits ^= 0x80000000u >> r;
      const Real v = static_cast<Real>(col[static_cast<int64_t>(r) * stride]);
      pool[q] = v;
      if (GEN) {
        const Real L = static_cast<Real>(lens[32 * w + r]);
        poola[q] = pow_alpha(v, static_cast<Real>(alpha)) * L;
      }
      ++q;
    }
  }
}

// Per-column double-double sums A[c] = sum over present rows of fl(L*v)
// (generalized: of fl(L*v^a), the poola entries). Block = 32 columns x
// kColParts word ranges (loads coalesced across the columns); the parts'
// partial sums combine in a fixed order, so the result is deterministic.
constexpr int kColParts = 8;

template <class Real, bool GEN>
__global__ void __launch_bounds__(32 * kColParts) wu_colsum_kernel(const uint32_t* __restrict__ nb,
                                                                 const uint32_t* __restrict__ off, int64_t n_ext,
                                                                 int32_t n, int32_t W, const double* __restrict__ lens,
                                                                 const Real* __restrict__ pool,
                                                                 const Real* __restrict__ poola,
                                                                 double2* __restrict__ A) {
  __shared__ double2 part[kColParts][32];
  const int cl = threadIdx.x & 31, pi = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + cl;
  const int32_t per = (W + kColParts - 1) / kColParts;
  const int32_t w0 = pi * per, w1 = min(W, w0 + per);
  double hi = 0.0, lo = 0.0;
  if (c < n) {
    for (int32_t w = w0; w < w1; ++w) {
      uint32_t bits = __ldg(nb + w * n_ext + c);
      if (!bits) continue;
      uint32_t q = __ldg(off + w * n_ext + c);
      while (bits) {
        const int r = __clz(bits);
        bits ^= 0x80000000u >> r;
        double term;
        if (GEN)
          term = static_cast<double>(poola[q]);
        else
          term = static_cast<double>(static_cast<Real>(lens[32 * static_cast<int64_t>(w) + r]) * pool[q]);
        dd_add(hi, lo, term);
        ++q;
      }
    }
  }
  part[pi][cl] = make_double2(hi, lo);
  __syncthreads();
  if (pi == 0 && c < n) {
    for (int j = 1; j < kColParts; ++j) {
      const double2 o = part[j][cl];
      dd_add(hi, lo, o.x);
      lo += o.y;
    }
    A[c] = make_double2(hi, lo);
  }
}

// Nonzero presence words per column: bit j of nz[g][c] = (nb[32g + j][c] != 0).
__global__ void wu_nzmask_kernel(const uint32_t* __restrict__ nb, int64_t n_ext, int32_t n, int32_t W,
                                 uint32_t* __restrict__ nz) {
  const int64_t G = (static_cast<int64_t>(W) + 31) / 32;
  const int64_t total = G * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / n;
    const int64_t c = i - g * n;
    const int64_t left = W - 32 * g;
    const int jmax = left < 32 ? static_cast<int>(left) : 32;
    uint32_t m = 0u;
    for (int j = 0; j < jmax; ++j)
      if (__ldg(nb + (32 * g + j) * n_ext + c)) m |= 1u << j;
    nz[g * n + c] = m;
  }
}

__device__ __forceinline__ void wu_prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct WUWalkArgs {
  const uint32_t* nb;   // W x n_ext presence words (global)
  const uint32_t* off;  // W x n_ext global pool offsets
  const void* pool;     // Real
  const void* poola;    // Real, generalized only
  const double* lens;   // [32 W], zero past E
  const double2* A;     // [n] column sums (double-double)
  int64_t n_ext;
  int32_t W;
  int32_t n;
  int32_t s_begin, s_end;  // stripes of this launch (absolute)
  int32_t out_begin;       // stripe held by row 0 of dist / tot
  int32_t finalize;
  double alpha;
  void* dist;
  void* tot;  // null for WU
  unsigned long long* exec_updates;
  unsigned long long* fp64_ops;  // FP64-pipe lane-instructions issued (roofline), or null
  const uint32_t* nz;  // [ceil(W/32)][n] nonzero-word masks (null: scan every word)
  const unsigned long long* nbo;  // [W][n_ext] (offset << 32) | presence word, or null
};

// One 8-byte cell per (word, column): the presence word and its pool offset
// arrive in one load (and one sector) instead of two.
__global__ void wu_combine_kernel(const uint32_t* __restrict__ nb, const uint32_t* __restrict__ off,
                                  int64_t cells, unsigned long long* __restrict__ nbo) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    nbo[i] = (static_cast<unsigned long long>(off[i]) << 32) | nb[i];
}

template <int M, class Real, int RS, int NW>
__global__ void __launch_bounds__(32 * NW, 2) stripe_wuwalk_kernel(const WUWalkArgs a) {
  constexpr bool GEN = M == kGen;
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * NW + (threadIdx.x >> 5);
  const int n = a.n;
  if (k >= n) return;
  const int s0 = a.s_begin + blockIdx.y * 32 * RS;
  const int64_t n_ext = a.n_ext;
  const int64_t l0 = static_cast<int64_t>(k) + s0 + 1 + lane;
  const Real* __restrict__ pool = static_cast<const Real*>(a.pool);
  const Real* __restrict__ poola = static_cast<const Real*>(a.poola);
  const double alpha = a.alpha;
  int nvalid = 0;
#pragma unroll
  for (int i = 0; i < RS; ++i) nvalid += (s0 + lane + 32 * i < a.s_end) ? 1 : 0;
  const int wvalid = __reduce_add_sync(0xffffffffu, nvalid);

  double d[RS], bh[RS], bl[RS], t[GEN ? RS : 1];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    d[i] = 0.0;
    bh[i] = 0.0;
    bl[i] = 0.0;
    if (GEN) t[i] = 0.0;
  }
  unsigned long long ubits = 0;
  unsigned hits = 0;  // this lane's shared (u and v present) slot-rows
  // one nonzero presence word w of column k (u != 0)
  auto word = [&](int w, uint32_t u) {
      uint32_t ou;
      uint32_t vv[RS], vo[RS];
      if (a.nbo) {
        const unsigned long long* crow = a.nbo + static_cast<int64_t>(w) * n_ext;
        ou = static_cast<uint32_t>(__ldg(crow + k) >> 32);
#pragma unroll
        for (int i = 0; i < RS; ++i) {
          const unsigned long long c = __ldg(crow + l0 + 32 * i);
          vv[i] = static_cast<uint32_t>(c);
          vo[i] = static_cast<uint32_t>(c >> 32);
        }
      } else {
        ou = __ldg(a.off + static_cast<int64_t>(w) * n_ext + k);
        const uint32_t* vrow = a.nb + static_cast<int64_t>(w) * n_ext + l0;
        const uint32_t* orow = a.off + static_cast<int64_t>(w) * n_ext + l0;
#pragma unroll
        for (int i = 0; i < RS; ++i) vv[i] = __ldg(vrow + 32 * i);
#pragma unroll
        for (int i = 0; i < RS; ++i) vo[i] = (vv[i] & u) ? __ldg(orow + 32 * i) : 0u;
      }
      ubits += static_cast<unsigned>(__popc(u));
      const double* Lw = a.lens + 32 * static_cast<int64_t>(w);
      uint32_t hu = u;
      uint32_t q = ou;
      while (hu) {
        const int r = __clz(hu);
        const uint32_t m = 0x80000000u >> r;
        hu ^= m;
        const double L = static_cast<double>(static_cast<Real>(__ldg(Lw + r)));
        const double uval = static_cast<double>(pool[q]);
        // the v-absent term: fl(L*u) in the working precision (reference: |u-0|*L)
        const double Lu = GEN ? static_cast<double>(poola[q]) : static_cast<double>(static_cast<Real>(L) * pool[q]);
        ++q;
        const uint32_t below = ~(0xffffffffu >> r);  // rows 32w..32w+r-1 (r = 0: none)
#pragma unroll
        for (int i = 0; i < RS; ++i) {
          const uint32_t hit = vv[i] & m;
          const double f = unit_if(!hit);
          d[i] = fma(Lu, f, d[i]);
          if (GEN) t[i] = fma(Lu, f, t[i]);
          if (hit) {
            ++hits;
            const uint32_t qv = vo[i] + static_cast<uint32_t>(__popc(vv[i] & below));
            const double v = static_cast<double>(pool[qv]);
            if (GEN) {
              const double s = uval + v;
              const double wgt = pow_alpha(s, alpha) * L;
              d[i] = fma(wgt, fabs(uval - v) / s, d[i]);
              t[i] += wgt;
              dd_add(bh[i], bl[i], static_cast<double>(poola[qv]));
            } else {
              d[i] = fma(fabs(uval - v), L, d[i]);
              dd_add(bh[i], bl[i], static_cast<double>(static_cast<Real>(L) * pool[qv]));
            }
          }
        }
      }
  };
  if (a.nz) {
    // nonzero words only (per-column masks); the next word's u/v words and
    // offsets are pulled into L1 while this one is walked
    const int G = (a.W + 31) / 32;
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      uint32_t m = __ldg(a.nz + static_cast<int64_t>(g) * n + k);
      while (m) {
        const int w = 32 * g + (__ffs(m) - 1);
        m &= m - 1u;
        if (m) {
          const int64_t nrow = static_cast<int64_t>(32 * g + (__ffs(m) - 1)) * n_ext;
          if (a.nbo) {
            if (lane == 0) wu_prefetch_l1(a.nbo + nrow + k);
#pragma unroll
            for (int i = 0; i < RS; ++i) wu_prefetch_l1(a.nbo + nrow + l0 + 32 * i);
          } else {
            if (lane == 0) {
              wu_prefetch_l1(a.nb + nrow + k);
              wu_prefetch_l1(a.off + nrow + k);
            }
#pragma unroll
            for (int i = 0; i < RS; ++i) {
              wu_prefetch_l1(a.nb + nrow + l0 + 32 * i);
              wu_prefetch_l1(a.off + nrow + l0 + 32 * i);
            }
          }
        }
        word(w, a.nbo ? static_cast<uint32_t>(__ldg(a.nbo + static_cast<int64_t>(w) * n_ext + k))
                      : __ldg(a.nb + static_cast<int64_t>(w) * n_ext + k));
      }
    }
  } else {
#pragma unroll 1
    for (int w = 0; w < a.W; ++w) {
      const uint32_t u = __ldg(a.nb + static_cast<int64_t>(w) * n_ext + k);
      if (u) word(w, u);
    }
  }

  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);
  const double2 Ak = a.A[k];
#pragma unroll
  for (int i = 0; i < RS; ++i) {
    if (i >= nvalid) break;
    const int s = s0 + lane + 32 * i;
    const int64_t li = l0 + 32 * i;
    const int l = li >= n ? static_cast<int>(li - n) : static_cast<int>(li);
    const double2 Al = a.A[l];
    const double vonly = dd_diff(Al.x, Al.y, bh[i], bl[i]);  // rows present in v only
    const double dv = d[i] + vonly;
    const int64_t o = static_cast<int64_t>(s - a.out_begin) * n + k;
    if (M == kWU) {
      dist[o] = static_cast<Real>(dv);
      continue;
    }
    double tv;
    if (GEN) {
      tv = t[i] + vonly;
    } else {  // WN: t = A_k + A_l
      double hi = Ak.x, lo = Ak.y;
      dd_add(hi, lo, Al.x);
      tv = hi + (lo + Al.y);
    }
    const Real tr = static_cast<Real>(tv);
    Real dr = static_cast<Real>(dv);
    if (a.finalize) dr = tr == Real(0) ? Real(0) : dr / tr;
    dist[o] = dr;
    tot[o] = tr;
  }
  if (a.exec_updates && lane == 0)
    atomicAdd(a.exec_updates, ubits * static_cast<unsigned long long>(wvalid));
  if (a.fp64_ops) {
    // per (u row, live slot): the absent-term DFMA (+ t for generalized);
    // per shared row: WN/WU d DFMA + fl(L*v) DMUL + TwoSum (5 DADD) + lo DADD = 8,
    // generalized: d DFMA, t DADD, |u-v|, u+v, TwoSum = 9 (pow and the divide
    // not counted: a lower bound)
    const unsigned long long per_hit = GEN ? 9ull : 8ull;
    unsigned long long h = __reduce_add_sync(0xffffffffu, hits);
    if (lane == 0)
      atomicAdd(a.fp64_ops, ubits * static_cast<unsigned long long>(wvalid) * (GEN ? 2ull : 1ull) + h * per_hit);
  }
}

// Even n: the last stripe (s = n/2 - 1) holds every pair twice, (k, k+n/2)
// at k < n/2 and again at k + n/2. The reference computes both with a
// symmetric update and condense() checks they are bitwise equal
// (stripes.cpp:115-122); the u-walk sums the two copies in different orders,
// so the second copy is taken from the first.
template <class Real>
__global__ void wu_mirror_kernel(Real* __restrict__ dist, Real* __restrict__ tot, int32_t n,
                                 int64_t row_off) {
  const int half = n / 2;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < half; k += gridDim.x * blockDim.x) {
    dist[row_off + half + k] = dist[row_off + k];
    if (tot) tot[row_off + half + k] = tot[row_off + k];
  }
}

}  // namespace sf
