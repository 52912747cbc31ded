// SELL-32/G-sigma row kernels: the solve-phase layout of every matrix the
// V-cycle streams.
//
// Rows are sorted by length (descending, ties by row index) inside windows of
// kSellWindow rows and cut into slices of 32/G consecutive sorted rows; each
// row gets G lanes of a warp (G = 1, 2, 4 or 8, chosen per matrix from its
// mean row length). Entry k of a row lives in chunk k/G at lane
// (row_in_slice * G + k % G): one chunk of a slice is 32 contiguous slots, so
// every index/value load of the warp is a single contiguous transaction.
// The G lanes of a row load and multiply their entries in parallel (G times
// the memory-level parallelism of a thread-per-row loop on long rows); the
// row's leader lane then adds the products one by one in column order,
// fetched with warp shuffles -- the reference's sequential, separately
// rounded sum (sparse.cpp:193-198), hence bit-identical results. Padding
// slots are skipped, never added.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace airg {

constexpr int kSellWindow = 256;
constexpr int kSellBatch = 2;  // chunks in flight per lane

struct SellView {
  const int32_t* off;   // nslices + 1 slot offsets
  const int32_t* len;   // row length per sorted row
  const int32_t* perm;  // sorted row -> original row
  const int32_t* ci;    // interleaved slice data (bit 31 may flag C columns)
  const double* v;
  int n;
  int nslices;
  int g;                // lanes per row (1, 2, 4, 8)
};

// lanes-per-row from the mean row length (AIRG_SELL_G overrides)
inline int sell_lanes_for(double mean_len) {
  if (mean_len <= 6.0) return 1;
  if (mean_len <= 12.0) return 2;
  if (mean_len <= 28.0) return 4;
  return 8;
}

template <int G, bool kFC>
__device__ __forceinline__ void sell_row_g(const SellView& m, int slice, int lane, int len,
                                           const double* __restrict__ x, double& sf, double& sc) {
  sf = 0.0;
  sc = 0.0;
  const int g = lane % G;
  const int lead = lane - g;
  const int chunks = (len + G - 1) / G;
  const int wchunks = __reduce_max_sync(0xffffffffu, chunks);  // warp-uniform trip count
  const int base = __ldg(m.off + slice) + lane;
  for (int ch0 = 0; ch0 < wchunks; ch0 += kSellBatch) {
    int c[kSellBatch];
    double a[kSellBatch], p[kSellBatch];
#pragma unroll
    for (int j = 0; j < kSellBatch; ++j) {
      const bool ok = (ch0 + j) * G + g < len;
      const int idx = base + (ch0 + j) * 32;
      c[j] = ok ? __ldg(m.ci + idx) : 0;
      a[j] = ok ? __ldg(m.v + idx) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kSellBatch; ++j) {
      const bool ok = (ch0 + j) * G + g < len;
      p[j] = ok ? __dmul_rn(a[j], __ldg(x + (kFC ? (c[j] & 0x7fffffff) : c[j]))) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kSellBatch; ++j) {
      if (ch0 + j >= wchunks) break;  // warp-uniform
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const double pq = G == 1 ? p[j] : __shfl_sync(0xffffffffu, p[j], lead + q);
        const int cq = kFC ? (G == 1 ? c[j] : __shfl_sync(0xffffffffu, c[j], lead + q)) : 0;
        if (g == 0 && (ch0 + j) * G + q < len) {
          if (kFC && cq < 0)
            sc = __dadd_rn(sc, pq);
          else
            sf = __dadd_rn(sf, pq);
        }
      }
    }
  }
}

template <int G, class Epi>
__device__ __forceinline__ void sell_body(const SellView& m, const double* __restrict__ x,
                                          Epi& epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int slice = t >> 5, lane = t & 31;
  const int row = slice * (32 / G) + lane / G;  // sorted row index
  const bool has = slice < m.nslices && row < m.n;
  const int len = has ? __ldg(m.len + row) : 0;
  const int orig = has ? __ldg(m.perm + row) : 0;
  pdl_wait();
  pdl_trigger();
  if (slice < m.nslices) {  // warp-uniform
    double s, unused;
    sell_row_g<G, false>(m, slice, lane, len, x, s, unused);
    if (has && lane % G == 0) epi.row(orig, s);
  }
}

template <int G, class Epi>
__device__ __forceinline__ void sell_body_fc(const SellView& m, const double* __restrict__ x,
                                             Epi& epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int slice = t >> 5, lane = t & 31;
  const int row = slice * (32 / G) + lane / G;
  const bool has = slice < m.nslices && row < m.n;
  const int len = has ? __ldg(m.len + row) : 0;
  const int orig = has ? __ldg(m.perm + row) : 0;
  pdl_wait();
  pdl_trigger();
  if (slice < m.nslices) {
    double sf, sc;
    sell_row_g<G, true>(m, slice, lane, len, x, sf, sc);
    if (has && lane % G == 0) epi.row2(orig, sf, sc);
  }
}

// Epi::row(original_row, acc); Epi::finish() once per thread (block reductions)
template <class Epi>
__global__ void __launch_bounds__(256) sell_rows(SellView m, const double* __restrict__ x, Epi epi) {
  switch (m.g) {
    case 1: sell_body<1>(m, x, epi); break;
    case 2: sell_body<2>(m, x, epi); break;
    case 4: sell_body<4>(m, x, epi); break;
    default: sell_body<8>(m, x, epi); break;
  }
  epi.finish();
}

// F-row variant (columns with bit 31 set are C columns): Epi::row2(orig, sf, sc)
template <class Epi>
__global__ void __launch_bounds__(256) sell_rows_fc(SellView m, const double* __restrict__ x, Epi epi) {
  switch (m.g) {
    case 1: sell_body_fc<1>(m, x, epi); break;
    case 2: sell_body_fc<2>(m, x, epi); break;
    case 4: sell_body_fc<4>(m, x, epi); break;
    default: sell_body_fc<8>(m, x, epi); break;
  }
}

inline unsigned sell_grid(const SellView& m) {
  const int64_t threads = (int64_t)m.nslices * 32;
  return (unsigned)(threads > 0 ? (threads + 255) / 256 : 1);
}

}  // namespace airg
