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

// ---- warp-per-row accumulation with a shared-memory hash table ---------------
// Products are taken 32 at a time in traversal order (A-row entry, then B-row
// entry). Lanes holding the same column form a group (__match_any_sync); the
// group's lowest lane adds the members' products to the column's slot one by
// one in lane order, so every entry still sees its contributions in the
// reference's order, starting from 0.0. Occupied slots are then compacted,
// bitonic-sorted by column and written to the row's scratch segment. Rows
// with more than kWarpA A-entries or kHashCap distinct columns are flagged
// and left to the thread-per-row kernel below.
constexpr int kWarpA = 64;

// kHashCap distinct columns per row, kSpgWarps rows per block; `only`
// (nullable) restricts the kernel to rows flagged by a previous pass.
template <int kHashCap, int kSpgWarps>
__global__ void __launch_bounds__(kSpgWarps * 32)
spgemm_warp_rows(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                 const double* __restrict__ av, const int32_t* __restrict__ brp,
                 const int32_t* __restrict__ bci, const double* __restrict__ bv,
                 const int64_t* __restrict__ off, int32_t* __restrict__ scol,
                 double* __restrict__ sval, int32_t* __restrict__ len, int32_t* __restrict__ kept,
                 int32_t* __restrict__ fallback, double drop_tol, int square_keep_diag,
                 const int32_t* __restrict__ only) {
  __shared__ int32_t keys_all[kSpgWarps][kHashCap];
  __shared__ double vals_all[kSpgWarps][kHashCap];
  __shared__ int32_t pref_all[kSpgWarps][kWarpA + 1];
  __shared__ double pbuf_all[kSpgWarps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSpgWarps + w;
  if (i >= n) return;
  if (only && !only[i]) return;
  int32_t* keys = keys_all[w];
  double* vals = vals_all[w];
  int32_t* pref = pref_all[w];
  double* pbuf = pbuf_all[w];
  const int s = arp[i], na = arp[i + 1] - s;
  if (na > kWarpA) {
    if (lane == 0) fallback[i] = 1;
    return;
  }
  // prefix of the B-row lengths of this A row (warp scan); empty A rows
  // (e.g. a C point without F neighbours in A_cf) give total = 0
  if (lane == 0) pref[0] = 0;
  __syncwarp();
  for (int k0 = 0; k0 < na; k0 += 32) {
    const int k = k0 + lane;
    int l = 0;
    if (k < na) {
      const int j = aci[s + k];
      l = brp[j + 1] - brp[j];
    }
    int incl = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int base = k0 == 0 ? 0 : pref[k0];
    if (k < na) pref[k + 1] = base + incl;
    __syncwarp();
  }
  const int total = pref[na];
  for (int q = lane; q < kHashCap; q += 32) keys[q] = -1;
  __syncwarp();
  bool overflow = false;
  for (int q0 = 0; q0 < total; q0 += 32) {
    const int q = q0 + lane;
    const bool valid = q < total;
    int col = -1;
    double p = 0.0;
    if (valid) {
      int lo = 0, hi = na;  // largest k with pref[k] <= q
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pref[mid] <= q)
          lo = mid;
        else
          hi = mid - 1;
      }
      const int j = aci[s + lo];
      const int t = brp[j] + (q - pref[lo]);
      col = bci[t];
      p = __dmul_rn(av[s + lo], bv[t]);
    }
    pbuf[lane] = p;
    const unsigned grp = __match_any_sync(0xffffffffu, valid ? col : -2 - lane);
    __syncwarp();
    if (valid && lane == __ffs(grp) - 1) {
      unsigned h = ((unsigned)col * 2654435761u) & (kHashCap - 1);
      int probes = 0;
      for (;;) {
        const int k = keys[h];
        if (k == col) break;
        if (k == -1) {
          const int prev = atomicCAS(&keys[h], -1, col);
          if (prev == -1) {
            vals[h] = 0.0;
            break;
          }
          if (prev == col) break;
        }
        h = (h + 1) & (kHashCap - 1);
        if (++probes >= kHashCap) {
          overflow = true;
          break;
        }
      }
      if (!overflow) {
        double v = vals[h];
        for (unsigned m = grp; m; m &= m - 1) v = __dadd_rn(v, pbuf[__ffs(m) - 1]);
        vals[h] = v;
      }
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, overflow)) {
      if (lane == 0) fallback[i] = 1;
      return;
    }
  }
  // compact occupied slots to the front (keys/vals), then bitonic sort by column
  int cnt = 0;
  for (int q0 = 0; q0 < kHashCap; q0 += 32) {
    const int k = keys[q0 + lane];
    const double v = vals[q0 + lane];
    const unsigned occ = __ballot_sync(0xffffffffu, k >= 0);
    __syncwarp();  // the whole chunk is read before any compacted write
    if (k >= 0) {  // destinations are distinct and never beyond this chunk
      const int dst = cnt + __popc(occ & ((1u << lane) - 1));
      keys[dst] = k;
      vals[dst] = v;
    }
    __syncwarp();
    cnt += __popc(occ);
  }
  int S = 1;
  while (S < cnt) S <<= 1;
  for (int q = cnt + lane; q < S; q += 32) keys[q] = 0x7fffffff;
  __syncwarp();
  for (int size = 2; size <= S; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < S; t += 32) {
        const int p2 = t ^ stride;
        if (p2 > t) {
          const bool asc = (t & size) == 0;
          const int kt = keys[t], kp = keys[p2];
          if ((kt > kp) == asc) {
            keys[t] = kp;
            keys[p2] = kt;
            const double vt = vals[t];
            vals[t] = vals[p2];
            vals[p2] = vt;
          }
        }
      }
      __syncwarp();
    }
  // write the row, drop count (sparse.cpp:244-268 rule)
  int32_t* oc = scol + off[i];
  double* ov = sval + off[i];
  double rmax = 0.0;
  for (int q = lane; q < cnt; q += 32) {
    oc[q] = keys[q];
    ov[q] = vals[q];
    rmax = fmax(rmax, fabs(vals[q]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  int kc = 0;
  if (drop_tol < 0.0) {
    kc = cnt;
  } else {
    const double thr = __dmul_rn(drop_tol, rmax);
    for (int q = lane; q < cnt; q += 32) {
      const double mag = fabs(vals[q]);
      const bool diag = square_keep_diag && keys[q] == i;
      kc += diag || !(mag < thr && mag < rmax);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) kc += __shfl_xor_sync(0xffffffffu, kc, o);
  }
  if (lane == 0) {
    len[i] = cnt;
    kept[i] = kc;
    fallback[i] = 0;
  }
}

__global__ void spgemm_accumulate(int n, const int32_t* __restrict__ arp,
                                  const int32_t* __restrict__ aci, const double* __restrict__ av,
                                  const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                  const double* __restrict__ bv, const int64_t* __restrict__ off,
                                  int32_t* __restrict__ scol, double* __restrict__ sval,
                                  int32_t* __restrict__ len, int32_t* __restrict__ kept,
                                  double drop_tol, int square_keep_diag,
                                  const int32_t* __restrict__ only) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (only && !only[i]) return;  // rows the warp kernel already produced
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
  static const bool thread_only = [] {
    const char* e = getenv("AIRG_SPGEMM");
    return e && !strcmp(e, "thread");
  }();
  if (thread_only) {
    LAUNCH(c, spgemm_accumulate, blocks_for(n, 128), 128, 0, n, a.rp.p, a.ci.p, a.v.p, b.rp.p,
           b.ci.p, b.v.p, off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, (const int32_t*)nullptr);
  } else {
    // 256-slot tables, 8 rows per block; overflowing rows retry with
    // 2048-slot tables (one row per block), then the thread-per-row kernel
    DBuf<int32_t> fb(c, (size_t)n), fb2(c, (size_t)n);
    fb.zero(c);
    fb2.zero(c);
    LAUNCH(c, (spgemm_warp_rows<256, 8>), (n + 7) / 8, 256, 0, n, a.rp.p, a.ci.p, a.v.p, b.rp.p,
           b.ci.p, b.v.p, off.p, scol.p, sval.p, len.p, kept.p, fb.p, drop_tol, sq,
           (const int32_t*)nullptr);
    LAUNCH(c, (spgemm_warp_rows<2048, 1>), n, 32, 0, n, a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p,
           off.p, scol.p, sval.p, len.p, kept.p, fb2.p, drop_tol, sq, (const int32_t*)fb.p);
    LAUNCH(c, spgemm_accumulate, blocks_for(n, 128), 128, 0, n, a.rp.p, a.ci.p, a.v.p, b.rp.p,
           b.ci.p, b.v.p, off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, (const int32_t*)fb2.p);
  }
  const int64_t nnz = exclusive_scan(c, kept.p, r.rp.p, n);
  r.nnz = nnz;
  r.ci.alloc(c, (size_t)nnz);
  r.v.alloc(c, (size_t)nnz);
  LAUNCH(c, spgemm_compact, blocks_for(n, 256), 256, 0, n, off.p, scol.p, sval.p, len.p, r.rp.p,
         r.ci.p, r.v.p, drop_tol, sq);
  out = std::move(r);
}

}  // namespace airg
