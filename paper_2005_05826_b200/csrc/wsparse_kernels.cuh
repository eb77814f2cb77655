// K2-W (sparse): weighted stripe update (normalized, unnormalized and the
// generalized-alpha extension, which the reference lacks) over
// node-packed presence bits plus a compacted value pool (kernel 11, the
// default for the weighted metrics).
//
// update_entry<Weighted*> (kernels.hpp:55-66) adds, for every postorder row
// e, d += |u-v|*L (and WN: t += (u+v)*L). A row where both samples are zero
// adds exactly +0.0 to an accumulator that is >= +0, so it can be skipped
// without changing a bit; at the EMP shape ~97% of the (row, slot) pairs are
// such rows. Each slot therefore walks only the rows present in either of its
// samples, in postorder, and applies the reference's update to them — the
// same operations in the same order, so EXACT (no FMA) is bitwise identical
// to the reference's x86-64 build and the FMA form is within 1e-12.
//
// Layout per embedding chunk (rows r0..r1 of the postorder, r0 % 32 == 0):
//   nb[w][c]   32 presence bits of chunk rows 32w..32w+31 for column c, row
//              32w+r at bit 31-r (FLO walks rows in ascending order); columns
//              extended past n so the shifted operand never wraps in a tile;
//   off[w][c]  first pool index of column c's values in word w (exclusive
//              scan of popc(nb) over [w][c]);
//   pool[]     the nonzero values, per (w, c) in row order, in the kernel's
//              precision (fp32: rounded once from the fp64 embedding, like
//              cast_batch, embed.hpp:71-84).
// The stripe kernel stages u/v words, offsets, occupancy and lengths of 32
// words (1024 rows) per step in shared memory (as the unweighted walk does,
// sparse_kernels.cuh); the present values are gathered from the pool (L1/L2).
// Accumulators are loaded from and stored to the stripes, so chunks chain.
#pragma once

#include <cstdint>

#include "stripe_kernels.cuh"

namespace sf {

// Presence words + popcounts of one chunk: thread per (word, column < n),
// coalesced over columns. Columns n..n_ext get count 0 (filled by extend).
__global__ void ws_pack_kernel(const double* __restrict__ emb, int64_t stride, int32_t C,
                               int32_t n, int32_t Wc, int64_t n_ext, uint32_t* __restrict__ nb,
                               uint32_t* __restrict__ cnt) {
  const int64_t total = static_cast<int64_t>(Wc) * n_ext;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / n_ext;
    const int64_t c = i - w * n_ext;
    uint32_t bits = 0u;
    if (c < n) {
      const int r_end = min(32, C - static_cast<int>(32 * w));
      const double* col = emb + 32 * w * stride + c;
      for (int r = 0; r < r_end; ++r)
        if (col[static_cast<int64_t>(r) * stride] != 0.0) bits |= 0x80000000u >> r;
    }
    nb[i] = bits;
    cnt[i] = static_cast<uint32_t>(__popc(bits));
  }
}

// Nonzero values of (w, c < n) into pool[off[w][c] ...], in row order.
template <class Real>
__global__ void ws_fill_kernel(const double* __restrict__ emb, int64_t stride, int32_t n,
                               int32_t Wc, int64_t n_ext, const uint32_t* __restrict__ nb,
                               const uint32_t* __restrict__ off, Real* __restrict__ pool) {
  const int64_t total = static_cast<int64_t>(Wc) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / n;
    const int64_t c = i - w * n;
    uint32_t bits = nb[w * n_ext + c];
    if (!bits) continue;
    Real* dst = pool + off[w * n_ext + c];
    const double* col = emb + 32 * w * stride + c;
    while (bits) {
      const int r = __clz(bits);
      bits ^= 0x80000000u >> r;
      *dst++ = static_cast<Real>(col[static_cast<int64_t>(r) * stride]);
    }
  }
}

// Wrap columns n..n_ext of both the words and the offsets.
__global__ void ws_extend_kernel(uint32_t* __restrict__ nb, uint32_t* __restrict__ off, int32_t n,
                                 int32_t Wc, int64_t n_ext) {
  const int64_t extra = n_ext - n;
  const int64_t total = static_cast<int64_t>(Wc) * extra;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / extra;
    const int64_t col = n + i % extra;
    nb[w * n_ext + col] = nb[w * n_ext + col % n];
    off[w * n_ext + col] = off[w * n_ext + col % n];
  }
}

struct WSparseArgs {
  const uint32_t* nb;    // Wc x n_ext presence words of the chunk
  const uint32_t* off;   // Wc x n_ext pool offsets
  const void* pool;      // Real values
  int64_t n_ext;
  const double* lens;    // [C] lengths of the chunk rows
  int32_t C;             // rows in the chunk
  int32_t Wc;            // words in the chunk
  int32_t n;
  int32_t s_begin, s_end;
  void* dist;
  void* tot;             // null for WU
  unsigned long long* exec_updates;
  double alpha;          // generalized UniFrac exponent (kGen only)
};

template <int RK, int RS, int NWK, int NWS>
struct WSparseTile {
  static constexpr int NW = NWK * NWS;
  static constexpr int NT = 32 * NW;
  static constexpr int TK = NWK * RK;
  static constexpr int TS = NWS * 32 * RS;
  static constexpr int VW = TK + TS;
  static constexpr int WC = 32;
  static constexpr int USTR = TK + 1;
  static constexpr int LSTR = 33;
  static constexpr int OFF_L = 0;
  static constexpr int OFF_U = OFF_L + WC * LSTR * 8;
  static constexpr int OFF_V = OFF_U + WC * USTR * 4;
  static constexpr int OFF_UO = OFF_V + WC * VW * 4;
  static constexpr int OFF_VO = OFF_UO + WC * USTR * 4;
  static constexpr int OFF_OU = OFF_VO + WC * VW * 4;
  static constexpr int OFF_OV = OFF_OU + TK * 4;
  static constexpr int BYTES = OFF_OV + VW * 4;
  static_assert(VW % 32 == 0, "v window must be a multiple of 32 columns (bank mapping)");
  static_assert(TK + VW <= NT, "one staging thread per column");
};

template <int M, class Real, bool EXACT, int RK, int RS, int NWK, int NWS>
__global__ void __launch_bounds__(32 * NWK * NWS, 2) stripe_wsparse_kernel(const WSparseArgs a) {
  using T = WSparseTile<RK, RS, NWK, NWS>;
  constexpr bool kHasT = M != kWU;
  extern __shared__ __align__(16) unsigned char smem[];
  const double* sL = reinterpret_cast<const double*>(smem + T::OFF_L);
  uint32_t* sU = reinterpret_cast<uint32_t*>(smem + T::OFF_U);
  uint32_t* sV = reinterpret_cast<uint32_t*>(smem + T::OFF_V);
  uint32_t* sUO = reinterpret_cast<uint32_t*>(smem + T::OFF_UO);
  uint32_t* sVO = reinterpret_cast<uint32_t*>(smem + T::OFF_VO);
  uint32_t* occU = reinterpret_cast<uint32_t*>(smem + T::OFF_OU);
  uint32_t* occV = reinterpret_cast<uint32_t*>(smem + T::OFF_OV);
  const Real* __restrict__ pool = static_cast<const Real*>(a.pool);
  const Real alpha = static_cast<Real>(a.alpha);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wk = warp % NWK;
  const int ws = warp / NWK;
  const int n = a.n;
  const int k0 = blockIdx.x * T::TK;
  const int s0 = a.s_begin + blockIdx.y * T::TS;
  const int64_t P0 = static_cast<int64_t>(k0) + s0 + 1;
  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);

  Real D[RK][RS], Tt[RK][RS];
  uint32_t valid = 0u;
#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      const bool ok = k < n && s < a.s_end;
      const int64_t o = static_cast<int64_t>(s - a.s_begin) * n + k;
      D[j][i] = ok ? dist[o] : Real(0);
      Tt[j][i] = (ok && kHasT) ? tot[o] : Real(0);
      valid |= (ok ? 1u : 0u) << (j * RS + i);
    }
  unsigned long long executed = 0;

  for (int w0 = 0; w0 < a.Wc; w0 += T::WC) {
    const int wc = min(T::WC, a.Wc - w0);
    __syncthreads();
    if (tid < T::TK + T::VW) {
      const bool is_u = tid < T::TK;
      const int col = is_u ? tid : tid - T::TK;
      const int64_t gcol = is_u ? static_cast<int64_t>(k0) + col : P0 + col;
      const int64_t base = static_cast<int64_t>(w0) * a.n_ext + gcol;
      uint32_t occ = 0u;
#pragma unroll 8
      for (int w = 0; w < T::WC; ++w) {
        const int64_t idx = base + static_cast<int64_t>(w) * a.n_ext;
        const uint32_t v = w < wc ? __ldg(a.nb + idx) : 0u;
        const uint32_t o = v ? __ldg(a.off + idx) : 0u;
        occ |= (v != 0u ? 0x80000000u : 0u) >> w;
        if (is_u) {
          sU[w * T::USTR + col] = v;
          sUO[w * T::USTR + col] = o;
        } else {
          sV[w * T::VW + col] = v;
          sVO[w * T::VW + col] = o;
        }
      }
      if (is_u)
        occU[col] = occ;
      else
        occV[col] = occ;
    } else {
      double* sLw = reinterpret_cast<double*>(smem + T::OFF_L);
      for (int e = tid - (T::TK + T::VW); e < T::WC * 32; e += T::NT - (T::TK + T::VW)) {
        const int w = e >> 5, r = e & 31;
        const int row = (w0 + w) * 32 + r;
        sLw[w * T::LSTR + r] = (w < wc && row < a.C) ? a.lens[row] : 0.0;
      }
    }
    __syncthreads();

#pragma unroll
    for (int j = 0; j < RK; ++j) {
      const int cu = wk * RK + j;
      const uint32_t ou = occU[cu];
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        if (!(valid & (1u << (j * RS + i)))) continue;
        const int cv = cu + ws * 32 * RS + lane + 32 * i;
        uint32_t occ = ou | occV[cv];
        Real d = D[j][i], t = Tt[j][i];
        while (occ) {
          const int w = __clz(occ);
          occ ^= 0x80000000u >> w;
          const uint32_t u = sU[w * T::USTR + cu];
          const uint32_t v = sV[w * T::VW + cv];
          const Real* pu = pool + sUO[w * T::USTR + cu];
          const Real* pv = pool + sVO[w * T::VW + cv];
          uint32_t o = u | v;
          const double* Lw = sL + w * T::LSTR;
          executed += __popc(o);
          do {  // present rows in ascending order
            const int r = __clz(o);
            const uint32_t m = 0x80000000u >> r;
            o ^= m;
            Real uv = Real(0), vv = Real(0);
            if (u & m) uv = __ldg(pu++);
            if (v & m) vv = __ldg(pv++);
            if constexpr (M == kGen)
              update_generalized<EXACT, Real>(uv, vv, static_cast<Real>(Lw[r]), alpha, d, t);
            else
              update_entry<M, EXACT, Real>(uv, vv, static_cast<Real>(Lw[r]), d, t);
          } while (o);
        }
        D[j][i] = d;
        Tt[j][i] = t;
      }
    }
  }

#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      if (!(valid & (1u << (j * RS + i)))) continue;
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      const int64_t o = static_cast<int64_t>(s - a.s_begin) * n + k;
      dist[o] = D[j][i];
      if (kHasT) tot[o] = Tt[j][i];
    }
  if (a.exec_updates) {
    for (int sh = 16; sh > 0; sh >>= 1) executed += __shfl_down_sync(0xffffffffu, executed, sh);
    if (lane == 0) atomicAdd(a.exec_updates, executed);
  }
}

}  // namespace sf
