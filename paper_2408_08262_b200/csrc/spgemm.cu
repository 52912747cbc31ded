// Row-wise SpGEMM C = A B with the reference's exact per-entry accumulation
// order (sparse.cpp:203-242): for each output entry the products a_ij b_jc
// are added in A-row order then B-row order, each rounded separately
// (--fmad=false), starting from 0.0; cancellation zeros stay stored.
//
// Phase 1 bounds each row's product count; phase 2 (thread per row)
// accumulates into a sorted, de-duplicated list in that row's scratch
// segment, which preserves the order of contributions to every column
// whatever the lookup structure; phase 3 scans the kept counts and
// compacts, optionally fusing drop_entries (sparse.cpp:244-268).
#include "sparse.cuh"

namespace airg {

namespace {

__global__ void spgemm_bound(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                             const int32_t* __restrict__ brp, int64_t* __restrict__ ub) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t s = 0;
  for (int k = arp[i]; k < arp[i + 1]; ++k) {
    const int j = aci[k];
    s += brp[j + 1] - brp[j];
  }
  ub[i] = s;
}

__global__ void spgemm_accumulate(int n, const int32_t* __restrict__ arp,
                                  const int32_t* __restrict__ aci, const double* __restrict__ av,
                                  const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                  const double* __restrict__ bv, const int64_t* __restrict__ off,
                                  int32_t* __restrict__ scol, double* __restrict__ sval,
                                  int32_t* __restrict__ len, int32_t* __restrict__ kept,
                                  double drop_tol, int square_keep_diag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t* cols = scol + off[i];
  double* vals = sval + off[i];
  int L = 0;
  for (int k = arp[i]; k < arp[i + 1]; ++k) {
    const double a = av[k];
    const int j = aci[k];
    for (int t = brp[j]; t < brp[j + 1]; ++t) {
      const int cc = bci[t];
      const double p = __dmul_rn(a, bv[t]);
      // binary search for cc in cols[0, L)
      int lo = 0, hi = L;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < cc)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < L && cols[lo] == cc) {
        vals[lo] = __dadd_rn(vals[lo], p);
      } else {
        for (int q = L; q > lo; --q) {
          cols[q] = cols[q - 1];
          vals[q] = vals[q - 1];
        }
        cols[lo] = cc;
        vals[lo] = __dadd_rn(0.0, p);
        ++L;
      }
    }
  }
  len[i] = L;
  if (drop_tol < 0.0) {
    kept[i] = L;
    return;
  }
  double row_max = 0.0;
  for (int q = 0; q < L; ++q) row_max = fmax(row_max, fabs(vals[q]));
  const double thr = __dmul_rn(drop_tol, row_max);
  int kc = 0;
  for (int q = 0; q < L; ++q) {
    const double mag = fabs(vals[q]);
    const bool diag = square_keep_diag && cols[q] == i;
    kc += diag || !(mag < thr && mag < row_max);
  }
  kept[i] = kc;
}

__global__ void spgemm_compact(int n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ scol, const double* __restrict__ sval,
                               const int32_t* __restrict__ len, const int32_t* __restrict__ orp,
                               int32_t* __restrict__ oci, double* __restrict__ ov, double drop_tol,
                               int square_keep_diag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t* cols = scol + off[i];
  const double* vals = sval + off[i];
  const int L = len[i];
  int o = orp[i];
  if (drop_tol < 0.0) {
    for (int q = 0; q < L; ++q) {
      oci[o + q] = cols[q];
      ov[o + q] = vals[q];
    }
    return;
  }
  double row_max = 0.0;
  for (int q = 0; q < L; ++q) row_max = fmax(row_max, fabs(vals[q]));
  const double thr = __dmul_rn(drop_tol, row_max);
  for (int q = 0; q < L; ++q) {
    const double mag = fabs(vals[q]);
    const bool diag = square_keep_diag && cols[q] == i;
    if (diag || !(mag < thr && mag < row_max)) {
      oci[o] = cols[q];
      ov[o++] = vals[q];
    }
  }
}

}  // namespace

void spgemm(Ctx& c, const Csr& a, const Csr& b, Csr& out, double drop_tol, bool keep_diag) {
  if (a.m != b.n) throw InvalidArgument("spgemm: dimension mismatch");
  const int n = a.n;
  Csr r;
  r.n = a.n;
  r.m = b.m;
  r.rp.alloc(c, (size_t)n + 1);
  if (n == 0) {
    CUDA_CHECK(cudaMemsetAsync(r.rp.p, 0, sizeof(int32_t), c.stream));
    out = std::move(r);
    return;
  }
  DBuf<int64_t> ub(c, (size_t)n), off(c, (size_t)n + 1);
  LAUNCH(c, spgemm_bound, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, b.rp.p, ub.p);
  const int64_t total = exclusive_scan64(c, ub.p, off.p, n);
  DBuf<int32_t> scol(c, (size_t)total), len(c, (size_t)n), kept(c, (size_t)n);
  DBuf<double> sval(c, (size_t)total);
  const int sq = (keep_diag && a.n == b.m) ? 1 : 0;
  LAUNCH(c, spgemm_accumulate, blocks_for(n, 128), 128, 0, n, a.rp.p, a.ci.p, a.v.p, b.rp.p,
         b.ci.p, b.v.p, off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq);
  const int64_t nnz = exclusive_scan(c, kept.p, r.rp.p, n);
  r.nnz = nnz;
  r.ci.alloc(c, (size_t)nnz);
  r.v.alloc(c, (size_t)nnz);
  LAUNCH(c, spgemm_compact, blocks_for(n, 256), 256, 0, n, off.p, scol.p, sval.p, len.p, r.rp.p,
         r.ci.p, r.v.p, drop_tol, sq);
  out = std::move(r);
}

}  // namespace airg
