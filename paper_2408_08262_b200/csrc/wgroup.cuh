// Long-row kernels with G lanes per row and B entries per lane in flight
// (AIRG_WG=G, rows of at least AIRG_WG_ROWS entries on average).
//
// Thread-per-row kernels on the 20-30 entry rows of the Galerkin levels are
// bound by L1 wavefronts: a warp instruction that loads one entry of 32
// different rows touches 32 different lines, for the column, the value AND
// the x gather. Here the G lanes of a row read G consecutive entries per
// instruction (one line for the group's columns, one or two for its values,
// and x gathers from one row's sorted column run), and each lane issues all
// B loads of a chunk of G*B entries before using any (the next chunk's
// column/value loads are issued with this chunk's x gathers; the first
// chunk before the PDL wait -- the matrix is static). The ordered sum stays
// the reference's: every lane of the group adds the chunk's products in
// column order (entry k0 + j*G + l is product j of lane l, fetched by a
// shuffle), each product rounded as a separate multiply (sparse.cpp:193-198;
// the F/C split of solve.cpp:72-80 by the sign bit of the column).
#pragma once

// included by tiled.cuh before its launch macros

namespace airg {

#ifndef AIRG_WG_B
#define AIRG_WG_B 4
#endif
constexpr int kWgB = AIRG_WG_B;

template <int G, int B>
struct WgChunk {
  int c[B];
  double a[B];
  __device__ __forceinline__ void load(int k0, int e, int lane, const int32_t* __restrict__ ci,
                                       const double* __restrict__ v) {
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int k = k0 + j * G + lane;
      c[j] = k < e ? __ldg(ci + k) : 0;
      a[j] = k < e ? __ldg(v + k) : 0.0;
    }
  }
};

template <int G, int B, bool FC, class Epi>
__global__ void __launch_bounds__(kTileThreads) rows_wgroup(TileView m, const double* __restrict__ x, Epi epi) {
  const int r = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G);
  const int lane = threadIdx.x & (G - 1);
  const int base = (threadIdx.x & 31) & ~(G - 1);
  const unsigned mask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << base;
  const bool live = r < m.nrows;
  int s = 0, e = 0;
  WgChunk<G, B> ch;
  if (live) {
    s = __ldg(m.rp + r);
    e = __ldg(m.rp + r + 1);
    ch.load(s, e, lane, m.ci, m.v);
  }
  typename pre_of<Epi>::type pre{};
  if constexpr (has_pre<Epi>::value) {
    if (live && lane == 0) pre = epi.pre(r);
  }
  pdl_wait();
  pdl_trigger();
  double sf = 0.0, sc = 0.0;
  for (int k0 = s; k0 < e; k0 += G * B) {  // trip count uniform over the group
    unsigned isc[B];
#pragma unroll
    for (int j = 0; j < B; ++j) isc[j] = FC ? (__ballot_sync(mask, ch.c[j] < 0) >> base) : 0u;
    double xv[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int k = k0 + j * G + lane;
      xv[j] = k < e ? __ldg(x + (FC ? (ch.c[j] & 0x7fffffff) : ch.c[j])) : 0.0;
    }
    WgChunk<G, B> nx;
    if (k0 + G * B < e) nx.load(k0 + G * B, e, lane, m.ci, m.v);
    double p[B];
#pragma unroll
    for (int j = 0; j < B; ++j) p[j] = __dmul_rn(ch.a[j], xv[j]);
    ch = nx;
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int cnt = min(G, e - (k0 + j * G));
      for (int l = 0; l < cnt; ++l) {
        const double q = __shfl_sync(mask, p[j], l, G);
        if (FC && ((isc[j] >> l) & 1u))
          sc = __dadd_rn(sc, q);
        else
          sf = __dadd_rn(sf, q);
      }
    }
  }
  if (live && lane == 0) {
    if constexpr (FC) {
      if constexpr (has_pre<Epi>::value)
        epi.row2_pre(r, sf, sc, pre);
      else
        epi.row2(r, sf, sc);
    } else {
      if constexpr (has_pre<Epi>::value)
        epi.row_pre(r, sf, pre);
      else
        epi.row(r, sf);
    }
  }
  if constexpr (!FC) epi.finish();
}

}  // namespace airg
