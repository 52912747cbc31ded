// L0 sparse kernels: CSR upload/validation, SpMV, with_full_diagonal and
// drop_entries (reference: proj/src/sparse.cpp).
#include "sparse.cuh"
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

__global__ void map_cols_kernel(int64_t nnz, const int32_t* __restrict__ ci,
                                const int32_t* __restrict__ map, int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) out[k] = map[ci[k]];
}

}  // namespace

// Batch kind of the exact thread-per-row kernels (rowdot.cuh): aligned
// 8-entry vector batches pay off on long rows (the A_F rows of the Galerkin
// levels, ~25-30 entries); rows of <= 5 entries on average (the fine levels'
// A, R, A_FF, Aff^-1) use 4-entry batches; the rest the 8-entry scalar loop
// (thresholds measured on the C2 hierarchy, round 1).
constexpr int kOQLanesSwitch = 4;  // 4 lanes x 4 entries cover rows up to 16; longer -> 8 lanes
// Exact mode, long rows on small operators (latency bound): AIRG_OLANES_MEAN
// entries per row and above (default 12; 0 = off) on at most AIRG_OLANES_N
// rows (default 20 k). C4 exact GMRES 645 -> 633 us per iteration (the first
// F residuals of levels 9-18: 7.6-9.5 -> 4.6-6.3 us); on 46 k-row operators
// the ordered-lane kernel is slower (8.6 -> 13.8 us).
int row_olanes(int64_t n, int64_t nnz) {
  static const double mean_min = [] {
    const char* e = getenv("AIRG_OLANES_MEAN");
    return (e && e[0]) ? atof(e) : 12.0;
  }();
  static const int64_t n_max = [] {
    const char* e = getenv("AIRG_OLANES_N");
    return (e && e[0]) ? atoll(e) : (int64_t)20000;
  }();
  if (mean_min <= 0.0 || n <= 0 || n > n_max) return 0;
  const double mean = (double)nnz / (double)n;
  if (mean < mean_min) return 0;
  return mean > 4.0 * kOQLanesSwitch ? 8 : 4;
}

int row_vec(int64_t n, int64_t nnz) {
  if (n <= 0) return 0;
  if (nnz >= 12 * n) return 8;
  if (nnz <= 5 * n) return 4;
  return 0;
}

// Lanes per row of the fast-mode kernels: the fewest lanes (a power of two,
// at most 16) whose first batch (kLaneBatch = 4 entries per lane, loaded
// before the dependency wait) covers a mean row, so a typical row is one
// round of coalesced loads (1 = thread per row).
//
// Small operators (the coarse levels) are latency bound, not bandwidth
// bound: a row longer than the first batch costs a further dependent round
// of (column, value) then x loads after the wait. When the longest row is
// known and the rows x lanes stay within AIRG_LANE_WAVE threads (default
// 150 k, about half a wave of 148 SMs x 2048: measured best on C4 against
// 75 k and 300 k), the lanes grow (up to a warp) until the first batch
// covers the longest row.
int row_lanes(int64_t n, int64_t nnz, int32_t max_row) {
  if (n <= 0) return 1;
  // (2, 3 and 6 entries per lane measured 9 %, 2 % and 4 % slower on the
  // C4 GMRES solve)
  const double mean = (double)nnz / (double)n;
  int g = 1;
  while (g < 16 && mean > 4.0 * g) g *= 2;
  static const int64_t wave = [] {
    const char* e = getenv("AIRG_LANE_WAVE");
    return (e && e[0]) ? atoll(e) : (int64_t)150000;
  }();
  if (max_row > 0)
    while (g < 32 && max_row > 4 * g && n * 2 * g <= wave) g *= 2;
  return g;
}

namespace {
__global__ void k_row_max(int n, const int32_t* __restrict__ rp, int* __restrict__ out) {
  int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = max(m, rp[i + 1] - rp[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out, m);
}
}  // namespace

void row_max(Ctx& c, const std::vector<Csr*>& ms) {
  if (ms.empty()) return;
  DBuf<int> d(c, ms.size());
  CUDA_CHECK(cudaMemsetAsync(d.p, 0, sizeof(int) * ms.size(), c.stream));
  for (size_t k = 0; k < ms.size(); ++k)
    if (ms[k]->n > 0)
      LAUNCH(c, k_row_max, (unsigned)std::min<int64_t>(blocks_for(ms[k]->n, 256), 1184), 256, 0, ms[k]->n,
             ms[k]->rp.p, d.p + k);
  std::vector<int> h(ms.size());
  to_host(c, h.data(), d.p, ms.size());
  for (size_t k = 0; k < ms.size(); ++k) ms[k]->max_row = h[k];
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

// y = A x (sparse.cpp:185-201): the exact thread-per-row kernel.
void spmv(Ctx& c, const Csr& a, const double* x, double* y) {
  if (a.n == 0) return;
  LAUNCH_ROWS(c, EpiStore, tview(a), x, EpiStore{y});
}

// reference-order thread-per-row SpMV (kept for A/B checks of the tiled path)
void spmv_thread_rows(Ctx& c, const Csr& a, const double* x, double* y) {
  if (a.n == 0) return;
  LAUNCH(c, spmv_rows, blocks_for(a.n, 128), 128, 0, a.n, a.rp.p, a.ci.p, a.v.p, x, y);
}

void with_full_diagonal(Ctx& c, const Csr& a, Csr& out, int row_base, bool slab) {
  if (!slab && row_base == 0 && a.n != a.m)
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
