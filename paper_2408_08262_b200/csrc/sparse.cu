// L0 sparse kernels: CSR upload/validation, SpMV, with_full_diagonal and
// drop_entries (reference: proj/src/sparse.cpp).
#include "sparse.cuh"
#include "sell.cuh"
#include "tiled.cuh"

namespace airg {

namespace {

// ---- upload: int64 reference layout -> int32 device CSR with the checks of
// the SparseMatrix constructor (sparse.cpp:27-45). err[0] collects the
// smallest offending row per error class.
__global__ void convert_validate(int64_t n, int64_t m, const int64_t* __restrict__ rp64,
                                 const int64_t* __restrict__ ci64, const double* __restrict__ v,
                                 int32_t* __restrict__ rp, int32_t* __restrict__ ci,
                                 unsigned long long* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  rp[i] = (int32_t)rp64[i];
  if (i == n) return;
  const int64_t s = rp64[i], e = rp64[i + 1];
  if (s > e) {
    atomicMin(&err[0], (unsigned long long)i);  // not monotone
    return;
  }
  for (int64_t k = s; k < e; ++k) {
    const int64_t c = ci64[k];
    if (c < 0 || c >= m) atomicMin(&err[1], (unsigned long long)i);
    if (k > s && !(ci64[k - 1] < c)) atomicMin(&err[2], (unsigned long long)i);
    if (isnan(v[k])) atomicMin(&err[3], (unsigned long long)i);
    ci[k] = (int32_t)c;
  }
}

__global__ void widen_rows(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           int64_t* __restrict__ rp64, int64_t* __restrict__ ci64) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  rp64[i] = rp[i];
  if (i == n) return;
  for (int k = rp[i]; k < rp[i + 1]; ++k) ci64[k] = ci[k];
}

// ---- SpMV, sparse.cpp:185-201: thread per row, sequential in column order,
// every product and sum rounded separately (no FMA) -> bit-identical.
__global__ void spmv_rows(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, const double* __restrict__ x,
                          double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  y[i] = dot_ordered(__ldg(rp + i), __ldg(rp + i + 1), ci, v, x);
}

// ---- with_full_diagonal, sparse.cpp:132-160
// rows r of a slab starting at global row rb: the diagonal is column rb + r
__global__ void fulldiag_count(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               int32_t* __restrict__ cnt, int rb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  bool seen = false;
  for (int k = rp[r]; k < rp[r + 1]; ++k) seen |= ci[k] == i;
  cnt[r] = rp[r + 1] - rp[r] + (seen ? 0 : 1);
}
__global__ void fulldiag_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ v, const int32_t* __restrict__ orp,
                              int32_t* __restrict__ oci, double* __restrict__ ov, int rb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  int o = orp[r];
  bool seen = false;
  for (int k = rp[r]; k < rp[r + 1]; ++k) {
    const int c = ci[k];
    if (!seen && c > i) {
      oci[o] = i;
      ov[o++] = 0.0;
      seen = true;
    }
    if (c == i) seen = true;
    oci[o] = c;
    ov[o++] = v[k];
  }
  if (!seen) {
    oci[o] = i;
    ov[o] = 0.0;
  }
}

// ---- drop_entries, sparse.cpp:244-268
__device__ __forceinline__ bool keep_entry(double mag, double threshold, double row_max, bool diag) {
  return diag || !(mag < threshold && mag < row_max);
}
__global__ void drop_count(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, double tol, int square,
                           int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double row_max = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) row_max = fmax(row_max, fabs(v[k]));
  const double threshold = __dmul_rn(tol, row_max);
  int c = 0;
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    c += keep_entry(fabs(v[k]), threshold, row_max, square && ci[k] == i);
  cnt[i] = c;
}
__global__ void drop_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, double tol, int square,
                          const int32_t* __restrict__ orp, int32_t* __restrict__ oci,
                          double* __restrict__ ov) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double row_max = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) row_max = fmax(row_max, fabs(v[k]));
  const double threshold = __dmul_rn(tol, row_max);
  int o = orp[i];
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (keep_entry(fabs(v[k]), threshold, row_max, square && ci[k] == i)) {
      oci[o] = ci[k];
      ov[o++] = v[k];
    }
}

// ---- 16-bit column deltas: span of every row, then the deltas
__global__ void k_row_span(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           unsigned long long* __restrict__ out) {  // [0] max span, [1] any negative column
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long span = 0, neg = 0;
  if (i < n && rp[i + 1] > rp[i]) {
    const int lo = ci[rp[i]], hi = ci[rp[i + 1] - 1];  // columns sorted ascending
    span = (unsigned long long)(hi - lo);
    neg = lo < 0 || hi < 0;
  }
  block_max(out, span);
  block_max(out + 1, neg);
}
__global__ void k_make_c16(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           uint16_t* __restrict__ c16, int32_t* __restrict__ cbase) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int base = rp[i + 1] > rp[i] ? ci[rp[i]] : 0;
  cbase[i] = base;
  for (int k = rp[i]; k < rp[i + 1]; ++k) c16[k] = (uint16_t)(ci[k] - base);
}

// ---- per-block row order: rows of one kTileThreads window sorted by length
// (descending, ties by index) so a warp's rows have similar lengths
__global__ void k_window_sort(int n, const int32_t* __restrict__ rp, int32_t* __restrict__ perm) {
  __shared__ int len[kTileThreads], idx[kTileThreads];
  const int base = blockIdx.x * kTileThreads, t = threadIdx.x;
  const int i = base + t;
  len[t] = i < n ? rp[i + 1] - rp[i] : -1;
  idx[t] = i;
  __syncthreads();
  for (int size = 2; size <= kTileThreads; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int p = t ^ stride;
      if (p > t) {
        const bool desc = (t & size) == 0;
        const bool t_first = len[t] != len[p] ? len[t] > len[p] : idx[t] < idx[p];
        if (t_first != desc) {
          const int l0 = len[t], i0 = idx[t];
          len[t] = len[p];
          idx[t] = idx[p];
          len[p] = l0;
          idx[p] = i0;
        }
      }
      __syncthreads();
    }
  if (i < n) perm[i] = idx[t];
}

// ---- tiles (tiled.cuh): a row starts a tile when its first nonzero lies in a
// different kWarpNnz chunk than its predecessor's.
__global__ void tile_flags(int n, const int32_t* __restrict__ rp, int32_t* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0) || (rp[i] / kWarpNnz != rp[i - 1] / kWarpNnz);
}
__global__ void tile_fill(int n, const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                          int32_t* __restrict__ tiles, int ntiles) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) tiles[pos[i]] = i;
  if (i == 0) tiles[ntiles] = n;
}

// ---- SELL-32-sigma build (sell.cuh)
// sort (len desc, row asc) inside each 256-row window with a bitonic sort
__global__ void __launch_bounds__(kSellWindow) sell_sort(int n, const int32_t* __restrict__ rp,
                                                         int32_t* __restrict__ perm,
                                                         int32_t* __restrict__ slen) {
  __shared__ int32_t klen[kSellWindow], kidx[kSellWindow];
  const int t = threadIdx.x, r = blockIdx.x * kSellWindow + t;
  klen[t] = r < n ? rp[r + 1] - rp[r] : -1;
  kidx[t] = r;
  __syncthreads();
  for (int size = 2; size <= kSellWindow; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int p = t ^ stride;
      if (p > t) {
        // "a before b" in the target order: longer first, then lower row
        const bool dir = (t & size) == 0;
        const bool t_after_p = (klen[t] < klen[p]) || (klen[t] == klen[p] && kidx[t] > kidx[p]);
        if (t_after_p == dir) {
          int a = klen[t]; klen[t] = klen[p]; klen[p] = a;
          a = kidx[t]; kidx[t] = kidx[p]; kidx[p] = a;
        }
      }
      __syncthreads();
    }
  }
  if (r < n) {
    perm[r] = kidx[t];
    slen[r] = klen[t];
  }
}
// slice width in slots: chunks of its longest (first) row x 32
__global__ void sell_width(int nslices, int rows_per_slice, int g, const int32_t* __restrict__ slen,
                           int32_t* __restrict__ w) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nslices) w[s] = ((slen[s * rows_per_slice] + g - 1) / g) * 32;
}
__global__ void sell_fill(int n, int rows_per_slice, int g, const int32_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const double* __restrict__ v,
                          const int32_t* __restrict__ perm, const int32_t* __restrict__ slen,
                          const int32_t* __restrict__ off, int32_t* __restrict__ sci,
                          double* __restrict__ sv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int o = perm[r], len = slen[r];
  const int s = r / rows_per_slice, rl = r % rows_per_slice;
  const int base = off[s] + rl * g;
  for (int k = 0; k < len; ++k) {
    const int slot = base + (k / g) * 32 + (k % g);
    sci[slot] = ci[rp[o] + k];
    sv[slot] = v[rp[o] + k];
  }
}

__global__ void map_cols_kernel(int64_t nnz, const int32_t* __restrict__ ci,
                                const int32_t* __restrict__ map, int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) out[k] = map[ci[k]];
}

}  // namespace

// Row-kernel decomposition for this matrix (tiled.cuh):
//   default (AIRG_ROWS unset or =thread): thread per row everywhere;
//   AIRG_ROWS=group: G lanes per row, G from the mean row length
//     (AIRG_GROUP=G forces G);
//   AIRG_ROWS=tiles: warp tiles everywhere; =auto: warp tiles for long rows.
static int rows_override() {
  static int v = [] {
    const char* e = getenv("AIRG_ROWS");
    if (!e || !strcmp(e, "thread")) return 1;
    if (!strcmp(e, "group")) return 3;
    if (!strcmp(e, "tiles")) return 2;
    return 0;  // auto
  }();
  return v;
}

// Aligned 8-entry vector batches pay off on long rows (the A_F rows of the
// Galerkin levels, ~25-30 entries); rows of <= 5 entries on average (the
// fine levels' A, R, A_FF, Aff^-1) use 4-entry batches; the rest the 8-entry
// scalar loop. AIRG_VEC=0|4|8 forces one choice for every matrix.
int row_vec(int64_t n, int64_t nnz) {
  // mean row length from which vector batches pay (AIRG_VEC_ROWS overrides)
  static const int64_t kVecRows = [] {
    const char* e = getenv("AIRG_VEC_ROWS");
    return e ? (int64_t)atoi(e) : (int64_t)12;
  }();
  static const int64_t kShortRows = [] {
    const char* e = getenv("AIRG_SHORT_ROWS");
    return e ? (int64_t)atoi(e) : (int64_t)5;
  }();
  static const int forced = [] {
    const char* e = getenv("AIRG_VEC");
    return e ? atoi(e) : -1;
  }();
  if (forced >= 0) return forced == 8 || forced == 4 ? forced : 0;
  if (n <= 0) return 0;
  if (nnz >= kVecRows * n) return 8;  // long rows: aligned vector batches
  if (nnz <= kShortRows * n) return 4;  // short rows: 4-entry scalar batches
  return 0;
}

static int forced_group() {
  static const int forced = [] {
    const char* e = getenv("AIRG_GROUP");
    const int g = e ? atoi(e) : 0;
    return g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32 ? g : 0;
  }();
  return forced;
}

// lanes per row for a matrix of n rows and nnz entries
int row_group_for(int64_t n, int64_t nnz) {
  const int forced = forced_group();
  if (forced) return forced;
  if (n <= 0) return 1;
  const double mean = (double)nnz / (double)n;
  int g = 1;
  while (g < 16 && mean >= 4.0 * g * 2) g *= 2;  // about 4+ entries per lane
  return g;
}

bool solve_layout_sell() {
  static const bool v = [] {
    const char* e = getenv("AIRG_LAYOUT");
    return e && !strcmp(e, "sell");
  }();
  return v;
}

// widest 128-row block slice [rp[r0] & ~3, rp[r1]) of a matrix (staged.cuh)
__global__ void k_block_span(int n, const int32_t* __restrict__ rp, unsigned* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int r0 = b * kTileThreads;
  if (r0 >= n) return;
  const int r1 = min(r0 + kTileThreads, n);
  atomicMax(out, (unsigned)(rp[r1] - (rp[r0] & ~3)));
}

// AIRG_STAGE=1: row kernels of the captured V-cycle stage each block's
// (column, value) slice in shared memory by bulk copies (staged.cuh) for
// every matrix that is not short-row; capacity = the widest block slice,
// capped at AIRG_STAGE_CAP entries (default 4000: 48 KB; wider blocks walk
// global memory)
static bool stage_enabled() {
  static const bool v = [] {
    const char* e = getenv("AIRG_STAGE");
#if defined(AIRG_STAGE_DEFAULT) && AIRG_STAGE_DEFAULT
    return !(e && e[0] == '0');
#else
    return e && e[0] == '1';
#endif
  }();
  return v;
}

static void build_stage(Ctx& c, Csr& a) {
  static const int cap = [] {
    const char* e = getenv("AIRG_STAGE_CAP");
    const int v = e ? atoi(e) : 4000;
    return v < 4 ? 4 : v > 4000 ? 4000 : v;
  }();
  a.stage = 0;
  if (!stage_enabled() || a.n <= 0 || a.group > 1 || a.perm.p || a.c16.p) return;
  if (row_vec(a.n, a.nnz) == 4) return;  // short rows: per-thread loads already touch whole lines
  if (((uintptr_t)a.ci.p & 15) || ((uintptr_t)a.v.p & 15)) return;
  DBuf<unsigned> sp(c, 1);
  sp.zero(c);
  const int nb = (a.n + kTileThreads - 1) / kTileThreads;
  LAUNCH(c, k_block_span, blocks_for(nb, 256), 256, 0, a.n, a.rp.p, sp.p);
  unsigned h = 0;
  to_host(c, &h, sp.p, 1);
  const int need = ((int)h + 3) & ~3;
  a.stage = need < cap ? need : (cap & ~3);
}

void build_tiles(Ctx& c, Csr& a) {
  if (a.row_mode != 0) return;
  const int ov = rows_override();
  if (ov == 3 || ov == 1 || forced_group()) {
    a.row_mode = 1;
    a.ntiles = 0;
    a.group = (int8_t)(ov == 3 || forced_group() ? row_group_for(a.n, a.nnz) : 1);
    // AIRG_SORT=1: rows of a block sorted by length (less divergence in a
    // warp) -- bit-identical, measured 11 % slower on C2 (row locality lost)
    static const bool sort_rows = [] {
      const char* e = getenv("AIRG_SORT");
      return e && e[0] == '1';
    }();
    if (sort_rows && a.group <= 1 && a.n > 0) {  // rows of a block sorted by length
      a.perm.alloc(c, (size_t)a.n);
      LAUNCH(c, k_window_sort, blocks_for(a.n, kTileThreads), kTileThreads, 0, a.n, a.rp.p, a.perm.p);
    }
    // AIRG_C16=1: 16-bit column deltas for long-row matrices (10 instead of
    // 12 B per entry) -- bit-identical, measured slower (0.997 vs 0.958 ms
    // per C2 iteration): the row kernels are latency / L1 bound, not byte bound
    static const bool c16 = [] {
      const char* e = getenv("AIRG_C16");
      return e && e[0] == '1';
    }();
    if (c16 && a.group <= 1 && a.n > 0 && a.nnz >= 8 * (int64_t)a.n && !sort_rows) {
      DBuf<unsigned long long> sp(c, 2);
      sp.zero(c);
      LAUNCH(c, k_row_span, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, sp.p);
      unsigned long long h[2];
      to_host(c, h, sp.p, 2);
      if (h[0] < 65536 && h[1] == 0) {  // every row fits 16-bit deltas; no flagged columns
        a.c16.alloc(c, (size_t)a.nnz + 8);
        a.cbase.alloc(c, (size_t)a.n);
        LAUNCH(c, k_make_c16, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, a.c16.p, a.cbase.p);
      }
    }
    build_stage(c, a);
    return;
  }
  const bool short_rows = ov ? ov == 1 : (a.n == 0 || a.nnz <= (int64_t)kShortRow * a.n);
  if (short_rows) {
    a.row_mode = 1;
    a.ntiles = 0;
    return;
  }
  a.row_mode = 2;
  DBuf<int32_t> flag(c, (size_t)a.n), pos(c, (size_t)a.n + 1);
  LAUNCH(c, tile_flags, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, flag.p);
  const int64_t nt = exclusive_scan(c, flag.p, pos.p, a.n);
  a.tiles.alloc(c, (size_t)nt + 1);
  LAUNCH(c, tile_fill, blocks_for(a.n, 256), 256, 0, a.n, flag.p, pos.p, a.tiles.p, (int)nt);
  a.ntiles = (int32_t)nt;
}

void build_sell(Ctx& c, Csr& a) {
  if (a.s_nslices >= 0) return;
  const int n = a.n;
  static const int g_override = [] {
    const char* e = getenv("AIRG_SELL_G");
    return e ? atoi(e) : 0;
  }();
  int g = g_override > 0 ? g_override : sell_lanes_for(n ? (double)a.nnz / n : 0.0);
  if (g != 1 && g != 2 && g != 4 && g != 8) g = 1;
  const int rps = 32 / g;
  const int nslices = (n + rps - 1) / rps;
  a.s_g = g;
  a.s_perm.alloc(c, (size_t)std::max(1, n));
  a.s_len.alloc(c, (size_t)std::max(1, n + kSellWindow));
  a.s_len.zero(c);
  a.s_off.alloc(c, (size_t)nslices + 1);
  if (n == 0) {
    a.s_off.zero(c);
    a.s_nslices = 0;
    return;
  }
  LAUNCH(c, sell_sort, (n + kSellWindow - 1) / kSellWindow, kSellWindow, 0, n, a.rp.p, a.s_perm.p,
         a.s_len.p);
  DBuf<int32_t> w(c, (size_t)nslices);
  LAUNCH(c, sell_width, blocks_for(nslices, 256), 256, 0, nslices, rps, g, a.s_len.p, w.p);
  const int64_t slots = exclusive_scan(c, w.p, a.s_off.p, nslices);
  a.s_ci.alloc(c, (size_t)slots);
  a.s_v.alloc(c, (size_t)slots);
  a.s_ci.zero(c);
  a.s_v.zero(c);
  LAUNCH(c, sell_fill, blocks_for(n, 256), 256, 0, n, rps, g, a.rp.p, a.ci.p, a.v.p, a.s_perm.p,
         a.s_len.p, a.s_off.p, a.s_ci.p, a.s_v.p);
  a.s_nslices = nslices;
}

void map_columns(Ctx& c, const Csr& a, const int32_t* d_map, int32_t new_ncols, Csr& out) {
  out.alloc(c, a.n, new_ncols, a.nnz);
  CUDA_CHECK(cudaMemcpyAsync(out.rp.p, a.rp.p, sizeof(int32_t) * (a.n + 1), cudaMemcpyDeviceToDevice, c.stream));
  if (a.nnz) {
    CUDA_CHECK(cudaMemcpyAsync(out.v.p, a.v.p, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice, c.stream));
    LAUNCH(c, map_cols_kernel, blocks_for(a.nnz, 256), 256, 0, a.nnz, a.ci.p, d_map, out.ci.p);
  }
}

void csr_upload(Ctx& c, int64_t n, int64_t m, const int64_t* h_rp, const int64_t* h_ci,
                const double* h_v, Csr& out) {
  if (n < 0 || m < 0) throw InvalidArgument("SparseMatrix: negative dimension");
  if (!h_rp) throw InvalidArgument("SparseMatrix: row_offsets length must be nrows+1");
  if (h_rp[0] != 0) throw InvalidArgument("SparseMatrix: row_offsets[0] must be 0");
  const int64_t nnz = h_rp[n];
  if (nnz < 0) throw InvalidArgument("SparseMatrix: row_offsets not monotone");
  out.alloc(c, n, m, nnz);
  DBuf<int64_t> rp64(c, (size_t)n + 1), ci64(c, (size_t)nnz);
  DBuf<double> v(c, 0);
  to_device(c, rp64.p, h_rp, (size_t)n + 1);
  to_device(c, ci64.p, h_ci, (size_t)nnz);
  to_device(c, out.v.p, h_v, (size_t)nnz);
  DBuf<unsigned long long> err(c, 4);
  CUDA_CHECK(cudaMemsetAsync(err.p, 0xff, 4 * sizeof(unsigned long long), c.stream));
  LAUNCH(c, convert_validate, blocks_for(n + 1, 256), 256, 0, n, m, rp64.p, ci64.p, out.v.p,
         out.rp.p, out.ci.p, err.p);
  unsigned long long e[4];
  to_host(c, e, err.p, 4);
  static const char* msg[4] = {"SparseMatrix: row_offsets not monotone",
                               "SparseMatrix: column index out of range",
                               "SparseMatrix: column indices not strictly increasing within row",
                               "SparseMatrix: stored NaN value"};
  for (int k = 0; k < 4; ++k)
    if (e[k] != ~0ull) throw InvalidArgument(msg[k]);
}

void csr_download(Ctx& c, const Csr& a, int64_t* h_rp, int64_t* h_ci, double* h_v) {
  DBuf<int64_t> rp64(c, (size_t)a.n + 1), ci64(c, (size_t)a.nnz);
  LAUNCH(c, widen_rows, blocks_for((int64_t)a.n + 1, 256), 256, 0, (int64_t)a.n, a.rp.p, a.ci.p,
         rp64.p, ci64.p);
  if (h_rp) CUDA_CHECK(cudaMemcpyAsync(h_rp, rp64.p, sizeof(int64_t) * (a.n + 1), cudaMemcpyDeviceToHost, c.stream));
  if (h_ci && a.nnz) CUDA_CHECK(cudaMemcpyAsync(h_ci, ci64.p, sizeof(int64_t) * a.nnz, cudaMemcpyDeviceToHost, c.stream));
  if (h_v && a.nnz) CUDA_CHECK(cudaMemcpyAsync(h_v, a.v.p, sizeof(double) * a.nnz, cudaMemcpyDeviceToHost, c.stream));
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// y = A x: the tiled coalesced kernel (tiled.cuh); tiles are a per-matrix
// cache built on first use (outside graph capture).
void spmv(Ctx& c, const Csr& a, const double* x, double* y) {
  if (a.n == 0) return;
  Csr& m = const_cast<Csr&>(a);
  if (m.s_nslices >= 0) {  // solve matrices carry a SELL copy (sell.cuh)
    SellView sv{m.s_off.p, m.s_len.p, m.s_perm.p, m.s_ci.p, m.s_v.p, m.n, m.s_nslices, m.s_g};
    LAUNCH(c, sell_rows<EpiStore>, sell_grid(sv), 256, 0, sv, x, EpiStore{y});
    return;
  }
  build_tiles(c, m);
  TileView tv{m.rp.p, m.ci.p, m.v.p, m.row_mode == 2 ? m.tiles.p : nullptr, m.ntiles, m.n, m.group, (int)m.nnz, row_vec(m.n, m.nnz), m.perm.p, m.c16.p, m.cbase.p};
  LAUNCH_ROWS(c, EpiStore, tv, x, EpiStore{y});
}

// reference-order thread-per-row SpMV (kept for A/B checks of the tiled path)
void spmv_thread_rows(Ctx& c, const Csr& a, const double* x, double* y) {
  if (a.n == 0) return;
  LAUNCH(c, spmv_rows, blocks_for(a.n, 128), 128, 0, a.n, a.rp.p, a.ci.p, a.v.p, x, y);
}

void with_full_diagonal(Ctx& c, const Csr& a, Csr& out, int row_base) {
  if (row_base == 0 && a.n != a.m)
    throw InvalidArgument("SparseMatrix: with_full_diagonal requires a square matrix");
  DBuf<int32_t> cnt(c, (size_t)a.n);
  Csr r;
  if (a.n) LAUNCH(c, fulldiag_count, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, cnt.p, row_base);
  r.rp.alloc(c, (size_t)a.n + 1);
  const int64_t nnz = exclusive_scan(c, cnt.p, r.rp.p, a.n);
  r.n = a.n;
  r.m = a.m;
  r.nnz = nnz;
  r.ci.alloc(c, (size_t)nnz);
  r.v.alloc(c, (size_t)nnz);
  if (a.n)
    LAUNCH(c, fulldiag_fill, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, a.v.p, r.rp.p,
           r.ci.p, r.v.p, row_base);
  out = std::move(r);
}

void drop_entries(Ctx& c, const Csr& a, double tol, bool keep_diagonal, Csr& out) {
  if (tol < 0.0) throw InvalidArgument("drop_entries: tol must be >= 0");
  const int square = keep_diagonal && a.n == a.m;
  DBuf<int32_t> cnt(c, (size_t)a.n);
  Csr r;
  if (a.n) LAUNCH(c, drop_count, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, a.v.p, tol, square, cnt.p);
  r.rp.alloc(c, (size_t)a.n + 1);
  const int64_t nnz = exclusive_scan(c, cnt.p, r.rp.p, a.n);
  r.n = a.n;
  r.m = a.m;
  r.nnz = nnz;
  r.ci.alloc(c, (size_t)nnz);
  r.v.alloc(c, (size_t)nnz);
  if (a.n)
    LAUNCH(c, drop_fill, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, a.v.p, tol, square,
           r.rp.p, r.ci.p, r.v.p);
  out = std::move(r);
}

}  // namespace airg
