// K2-UW (sparse): unweighted stripe update over node-packed presence bits.
//
// Same result, bit for bit, as update_entry<Unweighted> (kernels.hpp:55-66)
// summed over rows in postorder: for a slot (k, l = (k+s+1) mod n),
//   d = sum_{e in postorder, u_e(k) xor u_e(l)} L_e,
//   t = sum_{e in postorder, u_e(k) or  u_e(l)} L_e,
// because a 0/1 row adds exactly L_e or +0.0 and the adds happen in the same
// order (ascending row). The dense formulation spends 4 FP64 ops on every
// (row, slot) although ~98% of them are 0/0 at the EMP shape;
// here each slot walks only the rows present in either of its samples:
//
//   NB[w][c]  = 32 presence bits of rows 32w..32w+31 for sample column c
//               (word-major, sample columns extended past n so the shifted
//               operand k+s+1 never wraps inside a tile);
//   per CTA   = TK samples x TS stripes; rows are streamed in chunks of 32
//               words (1024 rows): u words [k0, k0+TK), v words
//               [k0+s0+1, k0+s0+TK+TS), per-column occupancy masks of the
//               chunk's nonzero words, and the rows' lengths;
//   per slot  = for each nonzero word of (u | v) (occupancy mask), for each
//               set bit of o = u | v in ascending order: t += L, and
//               d += L when the bit is set in x = u ^ v.
// Lanes run along stripes (same k, consecutive l), so the u side is shared by
// the warp and shared-memory accesses stay conflict-free although lanes walk
// different words.
#pragma once

#include <cstdint>

namespace sf {

// Sample-packed rows (row r: word c holds samples 32c..32c+31) -> node-packed
// columns NB[w][col] for col < n (rows >= E are zero). One warp per 32x32
// bit block, transposed with ballots.
__global__ void transpose_bits_kernel(const uint32_t* __restrict__ rows, int64_t row_words,
                                      int32_t E, int32_t n, uint32_t* __restrict__ nb,
                                      int64_t n_ext, int32_t W) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t ncw = row_words;  // sample words per row
  const int64_t blocks = static_cast<int64_t>(W) * ncw;
  for (int64_t bidx = warp; bidx < blocks; bidx += nwarps) {
    const int64_t w = bidx / ncw;
    const int64_t c = bidx % ncw;
    const int64_t r = w * 32 + lane;
    const uint32_t mine = r < E ? rows[r * row_words + c] : 0u;
    uint32_t out = 0u;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const uint32_t col = __ballot_sync(0xffffffffu, (mine >> b) & 1u);
      if (b == lane) out = col;
    }
    const int64_t smp = c * 32 + lane;
    if (smp < n) nb[w * n_ext + smp] = out;
  }
}

// Wrap columns: NB[w][col] = NB[w][col mod n] for n <= col < n_ext.
__global__ void extend_columns_kernel(uint32_t* __restrict__ nb, int64_t n_ext, int32_t n,
                                      int32_t W) {
  const int64_t extra = n_ext - n;
  const int64_t total = static_cast<int64_t>(W) * extra;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = i / extra;
    const int64_t col = n + i % extra;
    nb[w * n_ext + col] = nb[w * n_ext + col % n];
  }
}

struct SparseArgs {
  const uint32_t* nb;     // W x n_ext node-packed presence words
  int64_t n_ext;          // columns per word row
  const double* lens;     // [W*32] lengths, zero past E
  int32_t W;              // row words
  int32_t n;
  int32_t s_begin, s_end;
  void* dist;             // (s_end - s_begin) x n
  void* tot;
  unsigned long long* exec_updates;
};

template <class Real, int RK, int RS, int NWK, int NWS>
__global__ void __launch_bounds__(32 * NWK * NWS, 2) stripe_sparse_kernel(const SparseArgs a) {
  constexpr int NT = 32 * NWK * NWS;
  constexpr int TK = NWK * RK;          // samples per CTA
  constexpr int TS = NWS * 32 * RS;     // stripes per CTA
  constexpr int VW = TK + TS;           // v columns staged (one spare)
  constexpr int WC = 32;                // words per chunk (1024 rows)
  constexpr int USTR = TK + 1;          // padded: lanes on different words hit different banks
  constexpr int LSTR = 33;
  static_assert(VW % 32 == 0, "v window must be a multiple of 32 columns (bank mapping)");
  static_assert(TK + VW <= NT, "one staging thread per column");

  __shared__ uint32_t sU[WC * USTR];
  __shared__ uint32_t sV[WC * VW];
  __shared__ uint32_t occU[TK];
  __shared__ uint32_t occV[VW];
  __shared__ double sL[WC * LSTR];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wk = warp % NWK;
  const int ws = warp / NWK;
  const int n = a.n;
  const int k0 = blockIdx.x * TK;
  const int s0 = a.s_begin + blockIdx.y * TS;
  const int64_t P0 = static_cast<int64_t>(k0) + s0 + 1;

  Real* dist = static_cast<Real*>(a.dist);
  Real* tot = static_cast<Real*>(a.tot);

  Real D[RK][RS], T[RK][RS];
#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      const bool ok = k < n && s < a.s_end;
      const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
      D[j][i] = ok ? dist[off] : Real(0);
      T[j][i] = ok ? tot[off] : Real(0);
    }
  unsigned long long executed = 0;

  for (int w0 = 0; w0 < a.W; w0 += WC) {
    const int wc = min(WC, a.W - w0);
    __syncthreads();
    // ---- stage: one thread per column for the words + occupancy mask,
    //      the rest load lengths
    if (tid < TK + VW) {
      const bool is_u = tid < TK;
      const int col = is_u ? tid : tid - TK;
      const int64_t gcol = is_u ? static_cast<int64_t>(k0) + col : P0 + col;
      const uint32_t* src = a.nb + static_cast<int64_t>(w0) * a.n_ext + gcol;
      uint32_t occ = 0u;
      for (int w = 0; w < WC; ++w) {
        const uint32_t v = w < wc ? __ldg(src + static_cast<int64_t>(w) * a.n_ext) : 0u;
        occ |= (v != 0u ? 1u : 0u) << w;
        if (is_u)
          sU[w * USTR + col] = v;
        else
          sV[w * VW + col] = v;
      }
      if (is_u)
        occU[col] = occ;
      else
        occV[col] = occ;
    } else {
      for (int e = tid - (TK + VW); e < WC * 32; e += NT - (TK + VW)) {
        const int w = e >> 5, j = e & 31;
        sL[w * LSTR + j] = w < wc ? a.lens[static_cast<int64_t>(w0 + w) * 32 + j] : 0.0;
      }
    }
    __syncthreads();
    // ---- walk the present rows of every slot, in postorder
#pragma unroll
    for (int j = 0; j < RK; ++j) {
      const int cu = wk * RK + j;
      const uint32_t ou = occU[cu];
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        const int cv = cu + ws * 32 * RS + lane + 32 * i;
        uint32_t occ = ou | occV[cv];
        Real d = D[j][i], t = T[j][i];
        while (occ) {
          const int w = __ffs(occ) - 1;
          occ &= occ - 1u;
          const uint32_t u = sU[w * USTR + cu];
          const uint32_t v = sV[w * VW + cv];
          uint32_t o = u | v;
          const uint32_t x = u ^ v;
          const double* Lw = sL + w * LSTR;
          executed += __popc(o);
          do {
            const uint32_t b = o & (0u - o);
            o ^= b;
            const Real L = static_cast<Real>(Lw[31 - __clz(b)]);
            t += L;
            if (x & b) d += L;
          } while (o);
        }
        D[j][i] = d;
        T[j][i] = t;
      }
    }
  }

#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      if (k < n && s < a.s_end) {
        const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
        dist[off] = D[j][i];
        tot[off] = T[j][i];
      }
    }
  if (a.exec_updates) {
    // count only valid slots' work would need per-slot masks; tails are
    // small, so the CTA's executed (row, slot) visits are reported as is
    for (int off = 16; off > 0; off >>= 1) executed += __shfl_down_sync(0xffffffffu, executed, off);
    if (lane == 0) atomicAdd(a.exec_updates, executed);
  }
}

}  // namespace sf
