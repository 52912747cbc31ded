// Bit-exact CSR row kernels with two work decompositions, chosen per matrix
// by its mean row length (Csr::ntiles / tiles are built once, build_tiles()).
//
// * short rows (mean <= kShortRow): thread per row, batched loads
//   (rowdot.cuh). A warp's 32 consecutive rows are contiguous in memory,
//   so the warp still touches whole cache lines.
// * long rows: WARP TILES. A tile = the rows whose first nonzero falls in one
//   kWarpNnz-entry chunk of the nnz arrays. Each warp owns one tile:
//   phase 1 streams the tile's column indices and values with unit stride
//   (fully coalesced), gathers x and stores every product a_ij * x_j --
//   rounded exactly as the reference rounds it -- in the warp's slice of
//   shared memory; phase 2 (after __syncwarp, no block barrier) has one lane
//   per row add its products in column order (the reference's sequential
//   order, sparse.cpp:193-198) and run the epilogue.
// Both give the reference's bits. Tiles longer than the shared slice (rows
// of more than ~kWarpCap - kWarpNnz entries) fall back to the batched
// per-lane loop for that tile.
#pragma once

#include <type_traits>

#include "rowdot.cuh"

namespace airg {

#ifndef AIRG_TILE_THREADS
#define AIRG_TILE_THREADS 128
#endif
constexpr int kTileThreads = AIRG_TILE_THREADS;  // 4 warps per block (re-measured with pipelined batches: 0.891 ms/iteration vs 0.92 at 64 and 256)
constexpr int kWarpsPerBlock = kTileThreads / 32;
constexpr int kWarpNnz = 256;               // chunk size that cuts tiles
constexpr int kWarpCap = 384;               // shared products per warp
constexpr int kShortRow = 6;                // mean nnz/row below which rows win

struct TileView {
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
  const int32_t* tiles;  // nullptr => thread-per-row (group <= 1) or group-per-row mode
  int ntiles;
  int nrows;
  int group = 1;         // lanes per row of the group kernels (1, 2, 4, 8, 16, 32)
  int nnz = 0;           // > 0: thread-per-row kernels use aligned vector loads (rowdot.cuh)
  int vec = 0;           // entries per vector batch (4 or 8), 0 = scalar loop
  const int32_t* perm = nullptr;  // thread -> row (rows sorted by length per block), null = identity
  const uint16_t* c16 = nullptr;  // 16-bit column deltas (rowdot.cuh dot16), null = int32 columns
  const int32_t* cbase = nullptr;
  int stage = 0;         // > 0: staged row kernels (staged.cuh), shared slice capacity in entries
  int wg = 0;            // > 0: lanes per row of the long-row group kernels (wgroup.cuh)
  int w32 = 0;           // 1: warp-staged product kernels (w32.cuh)
};

// ---- thread per row -----------------------------------------------------------
// Row bounds and the first batch of the row are loaded before the PDL wait
// (static matrix data, rowdot.cuh RowBatch); m.vec selects aligned vector
// batches for long-row matrices.
// Epilogues may expose `Pre pre(int row)`: operands the epilogue reads that
// were produced two or more kernels earlier (when this kernel launches under
// PDL its predecessor has passed its own dependency wait, so everything
// before the predecessor is complete). They are loaded with the row's
// static data, before the wait, and handed to row_pre / row2_pre.
template <class E, class = void>
struct has_pre : std::false_type {};
template <class E>
struct has_pre<E, std::void_t<typename E::Pre>> : std::true_type {};

template <int VB, bool VEC, class Epi>
__device__ __forceinline__ void thread_row(const TileView& m, const double* __restrict__ x, Epi& epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < m.nrows;
  const int i = live && m.perm ? __ldg(m.perm + t) : t;
  int s = 0, e = 0;
  RowBatch<VB, VEC> b;
  if (live) {
    s = __ldg(m.rp + i);
    e = __ldg(m.rp + i + 1);
    if (s < e) b.load(batch_start<VB, VEC>(s), e, m.nnz, m.ci, m.v);
  }
  if constexpr (has_pre<Epi>::value) {
    typename Epi::Pre pre{};
    if (live) pre = epi.pre(i);
    pdl_wait();
    pdl_trigger();
    if (live) epi.row_pre(i, dot_prefetched<VB, VEC>(s, e, m.nnz, m.ci, m.v, x, b), pre);
  } else {
    pdl_wait();
    pdl_trigger();
    if (live) epi.row(i, dot_prefetched<VB, VEC>(s, e, m.nnz, m.ci, m.v, x, b));
  }
}

// VEC (a separate instantiation per batch kind keeps each kernel's register
// count at what its own loop needs)
// batch kinds (TileView::vec): 0 = 8-entry scalar batches, 8 = aligned 8-entry
// vector batches (long rows), 4 = 4-entry scalar batches (short rows)
// minimum resident blocks per SM of the row kernels (build knob; 1 = the
// compiler's register choice)
#ifndef AIRG_ROWS_MIN_BLOCKS
#define AIRG_ROWS_MIN_BLOCKS 1
#endif
template <class Epi, bool VEC = false, int VB = kRowBatch>
__global__ void __launch_bounds__(kTileThreads, AIRG_ROWS_MIN_BLOCKS) rows_thread(TileView m, const double* __restrict__ x,
                                                            Epi epi) {
  thread_row<VB, VEC>(m, x, epi);
  epi.finish();
}

// the same row kernel over 16-bit column deltas
template <class Epi>
__global__ void __launch_bounds__(kTileThreads) rows_thread16(TileView m, const double* __restrict__ x, Epi epi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < m.nrows;
  int s = 0, e = 0, base = 0;
  RowBatch16 b;
  if (live) {
    s = __ldg(m.rp + i);
    e = __ldg(m.rp + i + 1);
    base = __ldg(m.cbase + i);
    if (s < e) b.load(s & ~7, e, m.nnz, m.c16, m.v);
  }
  if constexpr (has_pre<Epi>::value) {
    typename Epi::Pre pre{};
    if (live) pre = epi.pre(i);
    pdl_wait();
    pdl_trigger();
    if (live) epi.row_pre(i, dot16(s, e, base, m.nnz, m.c16, m.v, x, b), pre);
  } else {
    pdl_wait();
    pdl_trigger();
    if (live) epi.row(i, dot16(s, e, base, m.nnz, m.c16, m.v, x, b));
  }
  epi.finish();
}

template <int VB, bool VEC, class Epi>
__device__ __forceinline__ void thread_row_fc(const TileView& m, const double* __restrict__ x, Epi& epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < m.nrows;
  const int i = live && m.perm ? __ldg(m.perm + t) : t;
  int s = 0, e = 0;
  RowBatch<VB, VEC> b;
  if (live) {
    s = __ldg(m.rp + i);
    e = __ldg(m.rp + i + 1);
    if (s < e) b.load(batch_start<VB, VEC>(s), e, m.nnz, m.ci, m.v);
  }
  if constexpr (has_pre<Epi>::value) {
    typename Epi::Pre pre{};
    if (live) pre = epi.pre(i);
    pdl_wait();
    pdl_trigger();
    if (!live) return;
    double sf, sc;
    dot_fc_prefetched<VB, VEC>(s, e, m.nnz, m.ci, m.v, x, b, sf, sc);
    epi.row2_pre(i, sf, sc, pre);
  } else {
    pdl_wait();
    pdl_trigger();
    if (!live) return;
    double sf, sc;
    dot_fc_prefetched<VB, VEC>(s, e, m.nnz, m.ci, m.v, x, b, sf, sc);
    epi.row2(i, sf, sc);
  }
}

// AIRG_FC_MIN_BLOCKS=5 (<= 48 registers, one wave on the big levels) spills
// and measured slower (18.56 vs 18.2 ms per C2 solve); kept as a build knob
#ifndef AIRG_FC_MIN_BLOCKS
#define AIRG_FC_MIN_BLOCKS 1
#endif
constexpr int kFcMinBlocks = AIRG_FC_MIN_BLOCKS;
// entries per aligned vector batch of the long-row first F residual
#ifndef AIRG_FC_VEC_BATCH
#define AIRG_FC_VEC_BATCH 8
#endif
constexpr int kFcVecBatch = AIRG_FC_VEC_BATCH;
// entries per batch of the other long-row kernels (aligned vector batches)
// and of the mid-length scalar kernels
#ifndef AIRG_VEC_BATCH
#define AIRG_VEC_BATCH 8
#endif
#ifndef AIRG_SCALAR_BATCH
#define AIRG_SCALAR_BATCH 8
#endif
constexpr int kVecBatch = AIRG_VEC_BATCH;
constexpr int kScalarBatch = AIRG_SCALAR_BATCH;
template <class Epi, bool VEC = false, int VB = kRowBatch>
__global__ void __launch_bounds__(kTileThreads, kFcMinBlocks) rows_thread_fc(TileView m, const double* __restrict__ x,
                                                               Epi epi) {
  thread_row_fc<VB, VEC>(m, x, epi);
}

// First F residual computed from data complete before its predecessor
// started: with XS = the prolongation of the coarse correction (solve.cu
// XProlong), its inputs come from two kernels back, so it runs concurrently
// with the prolongation kernel and waits for it only at its end (keeping the
// completion order the following kernels rely on).
template <class Epi, class XS, bool VEC = false, int VB = kRowBatch>
__global__ void __launch_bounds__(kTileThreads, kFcMinBlocks) rows_thread_fc_early(TileView m, XS xs, Epi epi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m.nrows) {
    const int s = __ldg(m.rp + i), e = __ldg(m.rp + i + 1);
    RowBatch<VB, VEC> b;
    if (s < e) b.load(batch_start<VB, VEC>(s), e, m.nnz, m.ci, m.v);
    const typename Epi::Pre pre = epi.pre(i);
    double sf, sc;
    dot_fc_src<VB, VEC>(s, e, m.nnz, m.ci, m.v, xs, b, sf, sc);
    epi.row2_pre(i, sf, sc, pre);
  }
  pdl_wait();
  pdl_trigger();
}

// First F residual as two ordered row dots over A_FF (global fine columns)
// and A_FC (coarse columns): the C part reads x_C = e_c, the coarse
// correction, which is complete before this kernel launches (two kernels
// back), so A_FC x_C is computed BEFORE the dependency wait -- overlapping
// the prolongation kernel -- and only A_FF x_F waits for it. Each partial
// sum keeps its column order, so (b_F - A_FF x_F) - A_FC x_C has the same
// bits as the single-pass kernel (x_C = 0 + 1.0 * (0 + 1.0 * e_c) equals e_c
// up to the sign of a zero, which cannot change a sum that starts at +0.0).
template <class Epi, bool VEC = false, int VB = kRowBatch>
__global__ void __launch_bounds__(kTileThreads, kFcMinBlocks)
rows_fres_split(TileView ff, TileView fc, const double* __restrict__ x, const double* __restrict__ ec, Epi epi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < ff.nrows;
  int s = 0, e = 0;
  double sc = 0.0;
  RowBatch<VB, VEC> b;
  typename Epi::Pre pre{};
  if (live) {
    const int cs = __ldg(fc.rp + i), ce = __ldg(fc.rp + i + 1);
    RowBatch<VB, VEC> bc;
    if (cs < ce) bc.load(batch_start<VB, VEC>(cs), ce, fc.nnz, fc.ci, fc.v);
    sc = dot_prefetched<VB, VEC>(cs, ce, fc.nnz, fc.ci, fc.v, ec, bc);
    s = __ldg(ff.rp + i);
    e = __ldg(ff.rp + i + 1);
    if (s < e) b.load(batch_start<VB, VEC>(s), e, ff.nnz, ff.ci, ff.v);
    pre = epi.pre(i);
  }
  pdl_wait();
  pdl_trigger();
  if (live) epi.row2_pre(i, dot_prefetched<VB, VEC>(s, e, ff.nnz, ff.ci, ff.v, x, b), sc, pre);
}

// ---- warp tiles -----------------------------------------------------------------
template <class Epi>
__global__ void __launch_bounds__(kTileThreads) rows_warp_tiles(TileView m,
                                                                const double* __restrict__ x,
                                                                Epi epi) {
  __shared__ double prod_all[kWarpsPerBlock][kWarpCap];
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * kWarpsPerBlock + w;
  if (t < m.ntiles) {
    double* prod = prod_all[w];
    const int r0 = __ldg(m.tiles + t), r1 = __ldg(m.tiles + t + 1);
    const int k0 = __ldg(m.rp + r0), k1 = __ldg(m.rp + r1);
    const int cnt = k1 - k0;
    if (cnt > kWarpCap) {
      for (int r = r0 + lane; r < r1; r += 32)
        epi.row(r, dot_ordered(__ldg(m.rp + r), __ldg(m.rp + r + 1), m.ci, m.v, x));
    } else {
#pragma unroll 4
      for (int j = lane; j < cnt; j += 32) {
        const int k = k0 + j;
        prod[j] = __dmul_rn(__ldg(m.v + k), __ldg(x + __ldg(m.ci + k)));
      }
      __syncwarp();
      for (int r = r0 + lane; r < r1; r += 32) {
        const int s = __ldg(m.rp + r) - k0, e = __ldg(m.rp + r + 1) - k0;
        double acc = 0.0;
        for (int q = s; q < e; ++q) acc = __dadd_rn(acc, prod[q]);
        epi.row(r, acc);
      }
    }
  }
  epi.finish();
}

// F-row variant: columns with bit 31 set are C columns; the F and C partial
// sums are kept apart (solve.cpp:72-80). Epi::row2(r, sf, sc).
template <class Epi>
__global__ void __launch_bounds__(kTileThreads) rows_warp_tiles_fc(TileView m,
                                                                   const double* __restrict__ x,
                                                                   Epi epi) {
  __shared__ double prod_all[kWarpsPerBlock][kWarpCap];
  __shared__ uint8_t isc_all[kWarpsPerBlock][kWarpCap];
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * kWarpsPerBlock + w;
  if (t >= m.ntiles) return;
  double* prod = prod_all[w];
  uint8_t* isc = isc_all[w];
  const int r0 = __ldg(m.tiles + t), r1 = __ldg(m.tiles + t + 1);
  const int k0 = __ldg(m.rp + r0), k1 = __ldg(m.rp + r1);
  const int cnt = k1 - k0;
  if (cnt > kWarpCap) {
    for (int r = r0 + lane; r < r1; r += 32) {
      double sf, sc;
      dot_ordered_fc(__ldg(m.rp + r), __ldg(m.rp + r + 1), m.ci, m.v, x, sf, sc);
      epi.row2(r, sf, sc);
    }
    return;
  }
#pragma unroll 4
  for (int j = lane; j < cnt; j += 32) {
    const int k = k0 + j;
    const int c = __ldg(m.ci + k);
    prod[j] = __dmul_rn(__ldg(m.v + k), __ldg(x + (c & 0x7fffffff)));
    isc[j] = c < 0;
  }
  __syncwarp();
  for (int r = r0 + lane; r < r1; r += 32) {
    const int s = __ldg(m.rp + r) - k0, e = __ldg(m.rp + r + 1) - k0;
    double sf = 0.0, sc = 0.0;
    for (int q = s; q < e; ++q) {
      if (isc[q])
        sc = __dadd_rn(sc, prod[q]);
      else
        sf = __dadd_rn(sf, prod[q]);
    }
    epi.row2(r, sf, sc);
  }
}

// ---- lane groups: G lanes per row ------------------------------------------------
// The G lanes of a row load G consecutive (column, value) pairs at a time
// (unit stride across the group), gather x and form the products -- each
// rounded exactly as the reference rounds it -- and lane 0 of the group adds
// them in column order from the group's registers (G shuffles). Same bits as
// thread per row; G times the memory parallelism per row, which is what the
// long rows of the mid/coarse Galerkin levels need.
template <int G>
__device__ __forceinline__ unsigned group_mask() {
  return G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
}

template <int G, class Epi>
__global__ void __launch_bounds__(kTileThreads) rows_group(TileView m, const double* __restrict__ x,
                                                           Epi epi) {
  pdl_wait();
  pdl_trigger();
  const int r = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G);
  const int lane = threadIdx.x & (G - 1);
  if (r < m.nrows) {
    const unsigned mask = group_mask<G>();
    const int s = __ldg(m.rp + r), e = __ldg(m.rp + r + 1);
    double acc = 0.0;
    for (int k0 = s; k0 < e; k0 += 2 * G) {
      const int ka = k0 + lane, kb = ka + G;
      const int ca = ka < e ? __ldg(m.ci + ka) : 0, cb = kb < e ? __ldg(m.ci + kb) : 0;
      const double va = ka < e ? __ldg(m.v + ka) : 0.0, vb = kb < e ? __ldg(m.v + kb) : 0.0;
      const double pa = ka < e ? __dmul_rn(va, __ldg(x + ca)) : 0.0;
      const double pb = kb < e ? __dmul_rn(vb, __ldg(x + cb)) : 0.0;
      const int cnt = e - k0;
      const int na = cnt < G ? cnt : G;
      for (int j = 0; j < na; ++j) acc = __dadd_rn(acc, __shfl_sync(mask, pa, j, G));
      const int nb = cnt - G < G ? cnt - G : G;
      for (int j = 0; j < nb; ++j) acc = __dadd_rn(acc, __shfl_sync(mask, pb, j, G));
    }
    if (lane == 0) epi.row(r, acc);
  }
  epi.finish();
}

template <int G, class Epi>
__global__ void __launch_bounds__(kTileThreads) rows_group_fc(TileView m, const double* __restrict__ x,
                                                              Epi epi) {
  pdl_wait();
  pdl_trigger();
  const int r = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G);
  const int lane = threadIdx.x & (G - 1);
  if (r >= m.nrows) return;
  const unsigned mask = group_mask<G>();
  const int shift = (threadIdx.x & 31) & ~(G - 1);
  const int s = __ldg(m.rp + r), e = __ldg(m.rp + r + 1);
  double sf = 0.0, sc = 0.0;
  for (int k0 = s; k0 < e; k0 += G) {
    const int k = k0 + lane;
    const int c = k < e ? __ldg(m.ci + k) : 0;
    const double p = k < e ? __dmul_rn(__ldg(m.v + k), __ldg(x + (c & 0x7fffffff))) : 0.0;
    const unsigned isc = __ballot_sync(mask, c < 0) >> shift;
    const int cnt = e - k0 < G ? e - k0 : G;
    for (int j = 0; j < cnt; ++j) {
      const double q = __shfl_sync(mask, p, j, G);
      if ((isc >> j) & 1u)
        sc = __dadd_rn(sc, q);
      else
        sf = __dadd_rn(sf, q);
    }
  }
  if (lane == 0) epi.row2(r, sf, sc);
}

}  // namespace airg
#include "staged.cuh"
#include "wgroup.cuh"
#include "w32.cuh"
namespace airg {

// grid size for either mode
inline unsigned rows_grid(const TileView& m) {
  if (m.tiles) return (unsigned)((m.ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock > 0
                                     ? (m.ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock
                                     : 1);
  const int64_t threads = (int64_t)m.nrows * (m.wg > 0 ? m.wg : m.group > 1 ? m.group : 1);
  const int64_t blocks = (threads + kTileThreads - 1) / kTileThreads;
  return (unsigned)(blocks > 0 ? blocks : 1);
}

// dispatch a group kernel on the runtime lane count (G in {2,4,8,16,32}); the
// kernel is bound to a pointer first so the template commas stay out of the
// launch macros
#define ROWS_GROUP_CASE(LAUNCHER, ctx, KERNEL, G, Epi, view, x, epi)             \
  case G: {                                                                     \
    auto* kfn__ = &KERNEL<G, Epi>;                                              \
    LAUNCHER(ctx, kfn__, rows_grid(view), kTileThreads, 0, view, x, epi);       \
  } break;
#define ROWS_GROUP_SWITCH(LAUNCHER, ctx, KERNEL, Epi, view, x, epi) \
  switch ((view).group) {                                          \
    ROWS_GROUP_CASE(LAUNCHER, ctx, KERNEL, 2, Epi, view, x, epi)    \
    ROWS_GROUP_CASE(LAUNCHER, ctx, KERNEL, 4, Epi, view, x, epi)    \
    ROWS_GROUP_CASE(LAUNCHER, ctx, KERNEL, 8, Epi, view, x, epi)    \
    ROWS_GROUP_CASE(LAUNCHER, ctx, KERNEL, 16, Epi, view, x, epi)   \
    default:                                                       \
    ROWS_GROUP_CASE(LAUNCHER, ctx, KERNEL, 32, Epi, view, x, epi)   \
  }

// long-row group kernels on the view's lane count (wgroup.cuh)
#define WG_SWITCH(ctx, FC, Epi, view, x, epi)                                                   \
  switch ((view).wg) {                                                                          \
    case 4:                                                                                     \
      LAUNCH_PDL(ctx, (rows_wgroup<4, kWgB * 2, FC, Epi>), rows_grid(view), kTileThreads, 0, view, x, epi); \
      break;                                                                                    \
    case 16:                                                                                    \
      LAUNCH_PDL(ctx, (rows_wgroup<16, 2, FC, Epi>), rows_grid(view), kTileThreads, 0, view, x, epi); \
      break;                                                                                    \
    default:                                                                                    \
      LAUNCH_PDL(ctx, (rows_wgroup<8, kWgB, FC, Epi>), rows_grid(view), kTileThreads, 0, view, x, epi); \
  }

// Launch helpers (used inside LAUNCH-counted wrappers).
#define LAUNCH_ROWS(ctx, Epi, view, x, epi)                                          \
  do {                                                                               \
    if ((view).tiles)                                                                \
      LAUNCH(ctx, rows_warp_tiles<Epi>, rows_grid(view), kTileThreads, 0, view, x, epi); \
    else if ((view).group > 1)                                                              \
      ROWS_GROUP_SWITCH(LAUNCH, ctx, rows_group, Epi, view, x, epi)                                  \
    else {                                                                           \
      auto* kfn__ = (view).c16 ? &rows_thread16<Epi> : (view).vec == 8 ? &rows_thread<Epi, true, kVecBatch> : (view).vec == 4 ? &rows_thread<Epi, false, 4> : &rows_thread<Epi, false, kScalarBatch>;   \
      LAUNCH(ctx, kfn__, rows_grid(view), kTileThreads, 0, view, x, epi);              \
    }                                                                                \
  } while (0)
// programmatic-dependent-launch variants (used inside the captured V-cycle)
#define LAUNCH_ROWS_P(ctx, Epi, view, x, epi)                                                   \
  do {                                                                                          \
    if ((view).tiles)                                                                           \
      LAUNCH_PDL(ctx, rows_warp_tiles<Epi>, rows_grid(view), kTileThreads, 0, view, x, epi);    \
    else if ((view).group > 1)                                                              \
      ROWS_GROUP_SWITCH(LAUNCH_PDL, ctx, rows_group, Epi, view, x, epi)                                  \
    else if ((view).w32)                                                                        \
      LAUNCH_PDL(ctx, (rows_w32<Epi, false>), rows_grid(view), kTileThreads, (w32_smem_checked<Epi, false>()), view, x, epi); \
    else if ((view).wg > 0)                                                                     \
      WG_SWITCH(ctx, false, Epi, view, x, epi)                                                  \
    else if ((view).stage > 0)                                                                  \
      LAUNCH_PDL(ctx, (rows_staged<Epi, false>), rows_grid(view), kTileThreads, stage_smem(view), view, x, epi); \
    else {                                                                                      \
      auto* kfn__ = (view).c16 ? &rows_thread16<Epi> : (view).vec == 8 ? &rows_thread<Epi, true, kVecBatch> : (view).vec == 4 ? &rows_thread<Epi, false, 4> : &rows_thread<Epi, false, kScalarBatch>;              \
      LAUNCH_PDL(ctx, kfn__, rows_grid(view), kTileThreads, 0, view, x, epi);                     \
    }                                                                                           \
  } while (0)
#define LAUNCH_ROWS_FC_P(ctx, Epi, view, x, epi)                                                \
  do {                                                                                          \
    if ((view).tiles)                                                                           \
      LAUNCH_PDL(ctx, rows_warp_tiles_fc<Epi>, rows_grid(view), kTileThreads, 0, view, x, epi); \
    else if ((view).group > 1)                                                              \
      ROWS_GROUP_SWITCH(LAUNCH_PDL, ctx, rows_group_fc, Epi, view, x, epi)                                  \
    else if ((view).w32)                                                                        \
      LAUNCH_PDL(ctx, (rows_w32<Epi, true>), rows_grid(view), kTileThreads, (w32_smem_checked<Epi, true>()), view, x, epi); \
    else if ((view).wg > 0)                                                                     \
      WG_SWITCH(ctx, true, Epi, view, x, epi)                                                   \
    else if ((view).stage > 0)                                                                  \
      LAUNCH_PDL(ctx, (rows_staged<Epi, true>), rows_grid(view), kTileThreads, stage_smem(view), view, x, epi); \
    else {                                                                                      \
      auto* kfn__ = (view).vec == 8 ? &rows_thread_fc<Epi, true, kFcVecBatch> : (view).vec == 4 ? &rows_thread_fc<Epi, false, 4> : &rows_thread_fc<Epi, false, kScalarBatch>;        \
      LAUNCH_PDL(ctx, kfn__, rows_grid(view), kTileThreads, 0, view, x, epi);                     \
    }                                                                                           \
  } while (0)
#define LAUNCH_ROWS_FC(ctx, Epi, view, x, epi)                                          \
  do {                                                                                  \
    if ((view).tiles)                                                                   \
      LAUNCH(ctx, rows_warp_tiles_fc<Epi>, rows_grid(view), kTileThreads, 0, view, x, epi); \
    else if ((view).group > 1)                                                              \
      ROWS_GROUP_SWITCH(LAUNCH, ctx, rows_group_fc, Epi, view, x, epi)                                  \
    else {                                                                              \
      auto* kfn__ = (view).vec == 8 ? &rows_thread_fc<Epi, true, kFcVecBatch> : (view).vec == 4 ? &rows_thread_fc<Epi, false, 4> : &rows_thread_fc<Epi, false, kScalarBatch>;  \
      LAUNCH(ctx, kfn__, rows_grid(view), kTileThreads, 0, view, x, epi);                   \
    }                                                                                   \
  } while (0)

// ---- epilogues ---------------------------------------------------------------
struct EpiStore {  // y = A x
  double* y;
  __device__ void row(int r, double acc) const { y[r] = acc; }
  __device__ void finish() const {}
};

}  // namespace airg
