// CSR row kernels of the solve: one CSR row traversal + an epilogue functor
// (the vector ops the reference runs after each SpMV, fused into it).
//
// Two arithmetic modes (airg_solve_config::fast):
//
// * EXACT (default; the reference's bits): thread per row, every row summed
//   left to right in column order with separately rounded products
//   (sparse.cpp:193-198, rowdot.cuh), batched and software-pipelined loads,
//   row bounds and the first batch loaded before the PDL dependency wait.
//   A warp's 32 consecutive rows are contiguous, so the warp still touches
//   whole cache lines on the short rows of the fine levels.
//
// * FAST: G lanes per row (G = row_lanes(): about four entries per lane),
//   each lane streaming a strided share of the row with coalesced (column,
//   value) loads across the group, fused multiply-adds, and a butterfly
//   (xor-shuffle) tree reduction. A row is then one round of independent
//   loads instead of a dependent chain: this is what the long A_F / R rows of
//   the Galerkin levels (20-40 entries, few thousand rows: latency bound under
//   thread-per-row) need. Results differ from the reference by rounding only
//   (the parity tests bound the solve: rtol 1e-10, +-1 iteration, 1e-8 in x).
#pragma once

#include <type_traits>

#include "rowdot.cuh"
#include "sparse.cuh"

namespace airg {

constexpr int kTileThreads = 128;  // 4 warps per block (measured: 64 and 256 slower; fast mode C4: 517 / 440 vs 435 us per iteration)

struct TileView {
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
  int nrows;
  int nnz;   // bounds the aligned vector loads
  int vec;   // exact mode: entries per vector batch (8), 4-entry scalar (4), 8-entry scalar (0)
  int lanes; // fast mode: lanes per row (1, 2, 4, 8, 16, 32)
  int olanes; // exact mode: lanes of the ordered-lane kernel (0: thread per row)
};

// Epilogues may expose `Pre pre(int row)`: operands the epilogue reads that
// were produced two or more kernels earlier (when this kernel launches under
// PDL its predecessor has passed its own dependency wait, so everything
// before the predecessor is complete). They are loaded with the row's
// static data, before the wait, and handed to row_pre / row2_pre.
template <class E, class = void>
struct has_pre : std::false_type {};
template <class E>
struct has_pre<E, std::void_t<typename E::Pre>> : std::true_type {};

// ---- exact: thread per row ----------------------------------------------------
template <class Epi, bool VEC, int VB>
__global__ void __launch_bounds__(kTileThreads) rows_thread(TileView m, const double* __restrict__ x, Epi epi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < m.nrows;
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
  epi.finish();
}

// F rows of A with C columns flagged by bit 31: the F and C partial sums are
// kept apart (solve.cpp:72-80); Epi::row2(r, sf, sc).
template <class Epi, bool VEC, int VB>
__global__ void __launch_bounds__(kTileThreads) rows_thread_fc(TileView m, const double* __restrict__ x, Epi epi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < m.nrows;
  int s = 0, e = 0;
  RowBatch<VB, VEC> b;
  if (live) {
    s = __ldg(m.rp + i);
    e = __ldg(m.rp + i + 1);
    if (s < e) b.load(batch_start<VB, VEC>(s), e, m.nnz, m.ci, m.v);
  }
  typename Epi::Pre pre{};
  if (live) pre = epi.pre(i);
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  double sf, sc;
  dot_fc_prefetched<VB, VEC>(s, e, m.nnz, m.ci, m.v, x, b, sf, sc);
  epi.row2_pre(i, sf, sc, pre);
}

// ---- fast: G lanes per row -------------------------------------------------------
// kLaneBatch entries per lane are loaded before the dependency wait (the
// matrix is static); longer rows continue in a strided loop.
constexpr int kLaneBatch = 4;

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}

template <int G, bool FC>
struct LaneRow {
  int s = 0, e = 0;
  int c[kLaneBatch];
  double a[kLaneBatch];
  __device__ __forceinline__ void load(const TileView& m, int r, int lane) {
    s = __ldg(m.rp + r);
    e = __ldg(m.rp + r + 1);
#pragma unroll
    for (int q = 0; q < kLaneBatch; ++q) {
      const int k = s + lane + q * G;
      c[q] = k < e ? __ldg(m.ci + k) : 0;
      a[q] = k < e ? __ldg(m.v + k) : 0.0;
    }
  }
  // sum over this lane's share of the row; FC: C-column products into sc
  __device__ __forceinline__ void dot(const TileView& m, const double* __restrict__ x, int lane, double& sf,
                                      double& sc) const {
    sf = 0.0;
    sc = 0.0;
    double xv[kLaneBatch];
#pragma unroll
    for (int q = 0; q < kLaneBatch; ++q)
      xv[q] = s + lane + q * G < e ? __ldg(x + (FC ? (c[q] & 0x7fffffff) : c[q])) : 0.0;
#pragma unroll
    for (int q = 0; q < kLaneBatch; ++q) {
      if (FC && c[q] < 0)
        sc = fma(a[q], xv[q], sc);
      else
        sf = fma(a[q], xv[q], sf);
    }
    for (int k0 = s + lane + kLaneBatch * G; k0 < e; k0 += kLaneBatch * G) {
      int cc[kLaneBatch];
      double aa[kLaneBatch], xx[kLaneBatch];
#pragma unroll
      for (int q = 0; q < kLaneBatch; ++q) {
        const int k = k0 + q * G;
        cc[q] = k < e ? __ldg(m.ci + k) : 0;
        aa[q] = k < e ? __ldg(m.v + k) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kLaneBatch; ++q)
        xx[q] = k0 + q * G < e ? __ldg(x + (FC ? (cc[q] & 0x7fffffff) : cc[q])) : 0.0;
#pragma unroll
      for (int q = 0; q < kLaneBatch; ++q) {
        if (FC && cc[q] < 0)
          sc = fma(aa[q], xx[q], sc);
        else
          sf = fma(aa[q], xx[q], sf);
      }
    }
  }
};

template <class Epi, int G>
__global__ void __launch_bounds__(kTileThreads) rows_lanes(TileView m, const double* __restrict__ x, Epi epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = t / G, lane = t & (G - 1);
  const bool live = r < m.nrows;
  LaneRow<G, false> row;
  if (live) row.load(m, r, lane);
  if constexpr (has_pre<Epi>::value) {
    typename Epi::Pre pre{};
    if (live && lane == 0) pre = epi.pre(r);
    pdl_wait();
    pdl_trigger();
    double sf = 0.0, sc;
    if (live) row.dot(m, x, lane, sf, sc);
    sf = group_sum<G>(sf);
    if (live && lane == 0) epi.row_pre(r, sf, pre);
  } else {
    pdl_wait();
    pdl_trigger();
    double sf = 0.0, sc;
    if (live) row.dot(m, x, lane, sf, sc);
    sf = group_sum<G>(sf);
    if (live && lane == 0) epi.row(r, sf);
  }
  epi.finish();
}

template <class Epi, int G>
__global__ void __launch_bounds__(kTileThreads) rows_lanes_fc(TileView m, const double* __restrict__ x, Epi epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = t / G, lane = t & (G - 1);
  const bool live = r < m.nrows;
  LaneRow<G, true> row;
  if (live) row.load(m, r, lane);
  typename Epi::Pre pre{};
  if (live && lane == 0) pre = epi.pre(r);
  pdl_wait();
  pdl_trigger();
  double sf = 0.0, sc = 0.0;
  if (live) row.dot(m, x, lane, sf, sc);
  sf = group_sum<G>(sf);
  sc = group_sum<G>(sc);
  if (live && lane == 0) epi.row2_pre(r, sf, sc, pre);
}

// ---- exact, long rows: G lanes load, one ordered sum ---------------------------
// A row of the exact mode is one sequential chain of separately rounded
// products and sums in column order (the reference's bits). With thread per
// row, a 30-entry row is four dependent batches of loads; here G lanes load
// Q = 4 entries each in one round (coalesced), form the products, and lane 0
// adds them in column order from the lanes' registers by shuffles -- the same
// chain of roundings, one round of loads per 4 G entries. FC: F and C columns
// into two sums (bit 31 of the column), as rows_thread_fc.
constexpr int kOQ = 4;
template <class E, bool = has_pre<E>::value>
struct PreOf {
  struct type {};
};
template <class E>
struct PreOf<E, true> {
  using type = typename E::Pre;
};
template <class Epi, int G, bool FC>
__global__ void __launch_bounds__(kTileThreads) rows_olanes(TileView m, const double* __restrict__ x, Epi epi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = t / G, lane = t & (G - 1);
  const bool live = r < m.nrows;
  int s = 0, len = 0;
  int c[kOQ];
  double a[kOQ];
  if (live) {
    s = __ldg(m.rp + r);
    len = __ldg(m.rp + r + 1) - s;
  }
#pragma unroll
  for (int q = 0; q < kOQ; ++q) {
    const int k = lane + q * G;
    c[q] = k < len ? __ldg(m.ci + s + k) : 0;
    a[q] = k < len ? __ldg(m.v + s + k) : 0.0;
  }
  typename PreOf<Epi>::type pre{};
  if constexpr (has_pre<Epi>::value)
    if (live && lane == 0) pre = epi.pre(r);
  pdl_wait();
  pdl_trigger();
  int maxlen = len;
#pragma unroll
  for (int o = 16; o; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
  double sf = 0.0, sc = 0.0;
  for (int base = 0; base < maxlen; base += kOQ * G) {
    if (base > 0) {
#pragma unroll
      for (int q = 0; q < kOQ; ++q) {
        const int k = base + lane + q * G;
        c[q] = k < len ? __ldg(m.ci + s + k) : 0;
        a[q] = k < len ? __ldg(m.v + s + k) : 0.0;
      }
    }
    double p[kOQ];
#pragma unroll
    for (int q = 0; q < kOQ; ++q) {
      const int k = base + lane + q * G;
      p[q] = k < len ? __dmul_rn(a[q], __ldg(x + (FC ? (c[q] & 0x7fffffff) : c[q]))) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kOQ; ++q) {
#pragma unroll
      for (int src = 0; src < G; ++src) {
        const double v = __shfl_sync(0xffffffffu, p[q], src, G);
        const int cf = FC ? __shfl_sync(0xffffffffu, c[q], src, G) : 0;
        if (lane == 0 && base + q * G + src < len) {
          if (FC && cf < 0)
            sc = __dadd_rn(sc, v);
          else
            sf = __dadd_rn(sf, v);
        }
      }
    }
  }
  if (live && lane == 0) {
    if constexpr (FC)
      epi.row2_pre(r, sf, sc, pre);
    else if constexpr (has_pre<Epi>::value)
      epi.row_pre(r, sf, pre);
    else
      epi.row(r, sf);
  }
  if constexpr (!FC) epi.finish();
}

// ---- launch ------------------------------------------------------------------------
inline TileView tview(const Csr& m) {
  return TileView{m.rp.p, m.ci.p, m.v.p, m.n, (int)m.nnz, row_vec(m.n, m.nnz), row_lanes(m.n, m.nnz, m.max_row),
                  row_olanes(m.n, m.nnz)};
}

inline unsigned rows_grid(const TileView& m, bool fast) {
  const int64_t threads = (int64_t)m.nrows * (fast ? m.lanes : (m.olanes > 1 ? m.olanes : 1));
  const int64_t blocks = (threads + kTileThreads - 1) / kTileThreads;
  return (unsigned)(blocks > 0 ? blocks : 1);
}

// the kernel for a view: exact batch kind by m.vec, fast lane count by m.lanes
template <class Epi>
inline auto rows_kernel(const TileView& m, bool fast) -> void (*)(TileView, const double*, Epi) {
  if (fast) {
    switch (m.lanes) {
      case 1: return &rows_lanes<Epi, 1>;
      case 2: return &rows_lanes<Epi, 2>;
      case 4: return &rows_lanes<Epi, 4>;
      case 8: return &rows_lanes<Epi, 8>;
      case 16: return &rows_lanes<Epi, 16>;
      default: return &rows_lanes<Epi, 32>;
    }
  }
  if (m.olanes == 4) return &rows_olanes<Epi, 4, false>;
  if (m.olanes == 8) return &rows_olanes<Epi, 8, false>;
  return m.vec == 8 ? &rows_thread<Epi, true, 8> : m.vec == 4 ? &rows_thread<Epi, false, 4>
                                                              : &rows_thread<Epi, false, 8>;
}
template <class Epi>
inline auto rows_kernel_fc(const TileView& m, bool fast) -> void (*)(TileView, const double*, Epi) {
  if (fast) {
    switch (m.lanes) {
      case 1: return &rows_lanes_fc<Epi, 1>;
      case 2: return &rows_lanes_fc<Epi, 2>;
      case 4: return &rows_lanes_fc<Epi, 4>;
      case 8: return &rows_lanes_fc<Epi, 8>;
      case 16: return &rows_lanes_fc<Epi, 16>;
      default: return &rows_lanes_fc<Epi, 32>;
    }
  }
  if (m.olanes == 4) return &rows_olanes<Epi, 4, true>;
  if (m.olanes == 8) return &rows_olanes<Epi, 8, true>;
  return m.vec == 8 ? &rows_thread_fc<Epi, true, 8> : m.vec == 4 ? &rows_thread_fc<Epi, false, 4>
                                                                 : &rows_thread_fc<Epi, false, 8>;
}

// Launch helpers (LAUNCH / LAUNCH_PDL count the launch in the context).
#define LAUNCH_ROWS_MODE(ctx, Epi, view, x, epi, fast)                                          \
  do {                                                                                          \
    auto* kfn__ = rows_kernel<Epi>((view), (fast));                                             \
    LAUNCH_PDL(ctx, kfn__, rows_grid((view), (fast)), kTileThreads, 0, (view), (x), (epi));     \
  } while (0)
#define LAUNCH_ROWS_FC_MODE(ctx, Epi, view, x, epi, fast)                                       \
  do {                                                                                          \
    auto* kfn__ = rows_kernel_fc<Epi>((view), (fast));                                          \
    LAUNCH_PDL(ctx, kfn__, rows_grid((view), (fast)), kTileThreads, 0, (view), (x), (epi));     \
  } while (0)
#define LAUNCH_ROWS(ctx, Epi, view, x, epi) LAUNCH_ROWS_MODE(ctx, Epi, view, x, epi, false)

// ---- epilogues ---------------------------------------------------------------
struct EpiStore {  // y = A x
  double* y;
  __device__ void row(int r, double acc) const { y[r] = acc; }
  __device__ void finish() const {}
};

}  // namespace airg
