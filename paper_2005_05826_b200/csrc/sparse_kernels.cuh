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
//   NB[w][c]  = 32 presence bits of rows 32w..32w+31 for sample column c,
//               row 32w+r at bit (31-r) so FLO yields rows in ascending
//               order; word-major, sample columns extended past n so the
//               shifted operand k+s+1 never wraps inside a tile;
//   per CTA   = TK samples x TS stripes; rows stream in chunks of 32 words
//               (1024 rows): u words [k0, k0+TK), v words [k0+s0+1, ...),
//               per-column occupancy masks of the chunk's nonzero words, and
//               the rows' lengths, staged in shared memory;
//   per lane  = RK x RS slots (lanes run along stripes, so the u side is
//               shared by the warp), accumulators in registers; for each slot
//               the lane walks the nonzero words of u|v (occupancy mask) and
//               their set bits in ascending row order: t += L for every bit of
//               u|v, d += L when the bit is also in u^v.
// (A per-warp work queue with shared-memory accumulators was tried to even
//  out the very uneven per-slot work; its divergent claim path cost more than
//  the divergence it removed — see profiles/.)
#pragma once

#include <cstdint>

namespace sf {

// Sample-packed rows (row r: word c holds samples 32c..32c+31) -> node-packed
// bit-reversed columns NB[w][col] for col < n (rows >= E are zero). One warp
// per 32x32 bit block, transposed with ballots.
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
      if (b == lane) out = __brev(col);  // row 32w+i -> bit 31-i
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

template <int RK, int RS, int NWK, int NWS>
struct SparseTile {
  static constexpr int NW = NWK * NWS;
  static constexpr int NT = 32 * NW;
  static constexpr int TK = NWK * RK;       // samples per CTA
  static constexpr int TS = NWS * 32 * RS;  // stripes per CTA
  static constexpr int VW = TK + TS;        // v columns staged (one spare)
  static constexpr int WC = 32;             // words per chunk (1024 rows)
  static constexpr int USTR = TK + 1;       // padded: different words -> different banks
  static constexpr int LSTR = 33;
  // dynamic shared memory layout (bytes)
  static constexpr int OFF_L = 0;
  static constexpr int OFF_U = OFF_L + WC * LSTR * 8;
  static constexpr int OFF_V = OFF_U + WC * USTR * 4;
  static constexpr int OFF_OU = OFF_V + WC * VW * 4;
  static constexpr int OFF_OV = OFF_OU + TK * 4;
  static constexpr int BYTES = OFF_OV + VW * 4;
  static_assert(VW % 32 == 0, "v window must be a multiple of 32 columns (bank mapping)");
  static_assert(TK + VW <= NT, "one staging thread per column");
};

template <class Real, int RK, int RS, int NWK, int NWS>
__global__ void __launch_bounds__(32 * NWK * NWS, 2) stripe_sparse_kernel(const SparseArgs a) {
  using T = SparseTile<RK, RS, NWK, NWS>;
  extern __shared__ __align__(16) unsigned char smem[];
  const double* sL = reinterpret_cast<const double*>(smem + T::OFF_L);
  uint32_t* sU = reinterpret_cast<uint32_t*>(smem + T::OFF_U);
  uint32_t* sV = reinterpret_cast<uint32_t*>(smem + T::OFF_V);
  uint32_t* occU = reinterpret_cast<uint32_t*>(smem + T::OFF_OU);
  uint32_t* occV = reinterpret_cast<uint32_t*>(smem + T::OFF_OV);

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

  // slot (j, i): sample k0 + wk*RK + j, stripe s0 + ws*32*RS + lane + 32*i
  Real D[RK][RS], Tt[RK][RS];
  uint32_t valid = 0u;
#pragma unroll
  for (int j = 0; j < RK; ++j)
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const int k = k0 + wk * RK + j;
      const int s = s0 + ws * 32 * RS + lane + 32 * i;
      const bool ok = k < n && s < a.s_end;
      const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
      D[j][i] = ok ? dist[off] : Real(0);
      Tt[j][i] = ok ? tot[off] : Real(0);
      valid |= (ok ? 1u : 0u) << (j * RS + i);
    }
  unsigned long long executed = 0;

  for (int w0 = 0; w0 < a.W; w0 += T::WC) {
    const int wc = min(T::WC, a.W - w0);
    __syncthreads();
    // ---- stage: one thread per column for its words + occupancy mask
    //      (word w at bit 31-w); the remaining threads stage the lengths
    if (tid < T::TK + T::VW) {
      const bool is_u = tid < T::TK;
      const int col = is_u ? tid : tid - T::TK;
      const int64_t gcol = is_u ? static_cast<int64_t>(k0) + col : P0 + col;
      const uint32_t* src = a.nb + static_cast<int64_t>(w0) * a.n_ext + gcol;
      uint32_t occ = 0u;
#pragma unroll 8
      for (int w = 0; w < T::WC; ++w) {
        const uint32_t v = w < wc ? __ldg(src + static_cast<int64_t>(w) * a.n_ext) : 0u;
        occ |= (v != 0u ? 0x80000000u : 0u) >> w;
        if (is_u)
          sU[w * T::USTR + col] = v;
        else
          sV[w * T::VW + col] = v;
      }
      if (is_u)
        occU[col] = occ;
      else
        occV[col] = occ;
    } else {
      double* sLw = reinterpret_cast<double*>(smem + T::OFF_L);
      for (int e = tid - (T::TK + T::VW); e < T::WC * 32; e += T::NT - (T::TK + T::VW)) {
        const int w = e >> 5, r = e & 31;
        sLw[w * T::LSTR + r] = w < wc ? a.lens[static_cast<int64_t>(w0 + w) * 32 + r] : 0.0;
      }
    }
    __syncthreads();

    // ---- walk the present rows of every slot, in postorder
#pragma unroll
    for (int j = 0; j < RK; ++j) {
      const int cu = wk * RK + j;
      const uint32_t ou = occU[cu];
      const uint32_t* pu = sU + cu;
#pragma unroll
      for (int i = 0; i < RS; ++i) {
        if (!(valid & (1u << (j * RS + i)))) continue;
        const int cv = cu + ws * 32 * RS + lane + 32 * i;
        const uint32_t* pv = sV + cv;
        uint32_t occ = ou | occV[cv];
        Real d = D[j][i], t = Tt[j][i];
        while (occ) {
          const int w = __clz(occ);  // next nonzero word (word w at bit 31-w)
          occ ^= 0x80000000u >> w;
          const uint32_t u = pu[w * T::USTR];
          const uint32_t v = pv[w * T::VW];
          uint32_t o = u | v;
          const uint32_t x = u ^ v;
          const double* Lw = sL + w * T::LSTR;
          executed += __popc(o);
          do {  // present rows in ascending order: row 32w+r sits at bit 31-r
            const int r = __clz(o);
            const uint32_t m = 0x80000000u >> r;
            o ^= m;
            const Real L = static_cast<Real>(Lw[r]);
            t += L;
            if (x & m) d += L;
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
      const int64_t off = static_cast<int64_t>(s - a.s_begin) * n + k;
      dist[off] = D[j][i];
      tot[off] = Tt[j][i];
    }
  if (a.exec_updates) {
    for (int off = 16; off > 0; off >>= 1) executed += __shfl_down_sync(0xffffffffu, executed, off);
    if (lane == 0) atomicAdd(a.exec_updates, executed);
  }
}


}  // namespace sf
