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

// warp-aggregated append of row i to list `cls` (one atomic per warp and class)
__device__ __forceinline__ void append_row(int i, int cls, bool live, int32_t* __restrict__ lists,
                                           int32_t* __restrict__ counts, int64_t stride) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned m = __ballot_sync(0xffffffffu, live && cls == k);
    if (!m) continue;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if ((int)lane == leader) base = atomicAdd(counts + k, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (live && cls == k) lists[k * stride + base + __popc(m & ((1u << lane) - 1))] = i;
  }
}

// products per row (upper bound of the row's length) and the row's class:
// 0 thread per row (few products or more A entries than the warp prefix
// holds), 1 warp hash. Lists: [0 | 1 | 2 | 3] x n, counts[4].
constexpr int kThreadProducts = 32;
constexpr int kWarpA = 64;
// bmap (nullable): B row of each A column (B holds gathered rows of a
// distributed operator); identity when null
__device__ __forceinline__ int brow(const int32_t* __restrict__ bmap, int j) { return bmap ? bmap[j] : j; }

__global__ void spgemm_bound(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                             const int32_t* __restrict__ brp, const int32_t* __restrict__ bmap,
                             int64_t* __restrict__ ub, int32_t* __restrict__ lists, int32_t* __restrict__ counts,
                             int classify) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n;
  int64_t s = 0;
  int cls = 0;
  if (live) {
    for (int k = arp[i]; k < arp[i + 1]; ++k) {
      const int j = brow(bmap, aci[k]);
      s += brp[j + 1] - brp[j];
    }
    ub[i] = s;
    cls = (s <= kThreadProducts || arp[i + 1] - arp[i] > kWarpA) ? 0 : 1;
  }
  if (classify) append_row(i, cls, live, lists, counts, n);
}

// ---- warp-per-row accumulation with a shared-memory hash table ---------------
// Products are taken 32 at a time in traversal order (A-row entry, then B-row
// entry). Lanes holding the same column form a group (__match_any_sync); the
// group's lowest lane adds the members' products to the column's slot one by
// one in lane order, so every entry still sees its contributions in the
// reference's order, starting from 0.0. Occupied slots are then compacted,
// bitonic-sorted by column and written to the row's scratch segment. Rows
// with more than kHashCap distinct columns go to the next list (a bigger
// table, then the thread-per-row kernel). Rows are taken from a device list
// by a persistent grid (the list length never crosses to the host).

// ---- sorted write-out of a warp's accumulated row ------------------------------
// The drop rule (sparse.cpp:244-268) on the sorted row: keep the diagonal
// (square products), else keep unless |v| < tol * rowmax and |v| < rowmax.
__device__ __forceinline__ void row_counts(int cnt, double drop_tol, int lane, int32_t* __restrict__ len,
                                           int32_t* __restrict__ kept, int i, int kc_lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) kc_lane += __shfl_xor_sync(0xffffffffu, kc_lane, o);
  if (lane == 0) {
    len[i] = cnt;
    kept[i] = drop_tol < 0.0 ? cnt : kc_lane;
  }
}

// Bitonic sort of the compacted (column, value) pairs in registers: element
// t = e * 32 + lane; strides >= 32 swap registers, smaller ones exchange with
// __shfl_xor. Padding keys (INT_MAX) sort last. Replaces the shared-memory
// sort (the bulk of the warp kernel's instructions) for rows of <= 256.
template <int E>
__device__ __forceinline__ void finish_reg(const int32_t* __restrict__ keys, const double* __restrict__ vals,
                                           int cnt, int lane, int i, int gi, int32_t* __restrict__ oc,
                                           double* __restrict__ ov, double drop_tol, int square_keep_diag,
                                           int32_t* __restrict__ len, int32_t* __restrict__ kept) {
  constexpr int S = 32 * E;
  int k[E];
  double v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int t = e * 32 + lane;
    k[e] = t < cnt ? keys[t] : 0x7fffffff;
    v[e] = t < cnt ? vals[t] : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int size = 2; size <= S; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int es = stride >> 5;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int e2 = e ^ es;
          if (e2 > e) {
            const bool asc = ((e * 32 + lane) & size) == 0;
            if ((k[e] > k[e2]) == asc) {
              const int tk = k[e];
              k[e] = k[e2];
              k[e2] = tk;
              const double tv = v[e];
              v[e] = v[e2];
              v[e2] = tv;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int kp = __shfl_xor_sync(0xffffffffu, k[e], stride);
          const double vp = __shfl_xor_sync(0xffffffffu, v[e], stride);
          const bool asc = ((e * 32 + lane) & size) == 0;
          const bool lower = (lane & stride) == 0;
          const bool take = (lower == asc) ? (kp < k[e]) : (kp > k[e]);
          if (take) {
            k[e] = kp;
            v[e] = vp;
          }
        }
      }
    }
  }
  double rmax = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int t = e * 32 + lane;
    if (t < cnt) {
      oc[t] = k[e];
      ov[t] = v[e];
      rmax = fmax(rmax, fabs(v[e]));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  int kc = 0;
  if (drop_tol >= 0.0) {
    const double thr = __dmul_rn(drop_tol, rmax);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int t = e * 32 + lane;
      if (t < cnt) {
        const double mag = fabs(v[e]);
        const bool diag = square_keep_diag && k[e] == gi;
        kc += diag || !(mag < thr && mag < rmax);
      }
    }
  }
  row_counts(cnt, drop_tol, lane, len, kept, i, kc);
}

// Rank placement instead of a sort network: the keys are distinct, so each
// compacted entry's position in the sorted row is the number of smaller
// keys, counted against 16-byte broadcast reads of the compacted keys
// (padded with INT_MAX). ~cnt/4 shared loads per lane instead of the
// bitonic network's log^2 shuffle stages (40% of the warp kernel's issue
// slots on the C2 Galerkin products). keys must be 16-byte aligned with
// room for cnt + 4 entries.
template <int E>
__device__ __forceinline__ void finish_rank(int32_t* __restrict__ keys, const double* __restrict__ vals, int cnt,
                                            int lane, int i, int gi, int32_t* __restrict__ oc,
                                            double* __restrict__ ov, double drop_tol, int square_keep_diag,
                                            int32_t* __restrict__ len, int32_t* __restrict__ kept) {
  int k[E];
  double v[E];
  int r[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int t = e * 32 + lane;
    k[e] = t < cnt ? keys[t] : 0x7fffffff;
    v[e] = t < cnt ? vals[t] : 0.0;
    r[e] = 0;
  }
  if (lane < 4) keys[cnt + lane] = 0x7fffffff;
  __syncwarp();
  const int4* k4 = reinterpret_cast<const int4*>(keys);
  for (int t = 0; t < cnt; t += 4) {
    const int4 q = k4[t >> 2];
#pragma unroll
    for (int e = 0; e < E; ++e) r[e] += (q.x < k[e]) + (q.y < k[e]) + (q.z < k[e]) + (q.w < k[e]);
  }
  double rmax = 0.0;
  int kc = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int t = e * 32 + lane;
    if (t < cnt) {
      oc[r[e]] = k[e];
      ov[r[e]] = v[e];
      rmax = fmax(rmax, fabs(v[e]));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (drop_tol >= 0.0) {
    const double thr = __dmul_rn(drop_tol, rmax);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int t = e * 32 + lane;
      if (t < cnt) {
        const double mag = fabs(v[e]);
        const bool diag = square_keep_diag && k[e] == gi;
        kc += diag || !(mag < thr && mag < rmax);
      }
    }
  }
  __syncwarp();  // the keys are read before the table is reused
  row_counts(cnt, drop_tol, lane, len, kept, i, kc);
}

// rows of more than 256 distinct columns (2048-slot tables): shared-memory sort
__device__ __forceinline__ void finish_smem(int32_t* __restrict__ keys, double* __restrict__ vals, int cnt,
                                            int lane, int i, int gi, int32_t* __restrict__ oc, double* __restrict__ ov,
                                            double drop_tol, int square_keep_diag, int32_t* __restrict__ len,
                                            int32_t* __restrict__ kept) {
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
  double rmax = 0.0;
  for (int q = lane; q < cnt; q += 32) {
    oc[q] = keys[q];
    ov[q] = vals[q];
    rmax = fmax(rmax, fabs(vals[q]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  int kc = 0;
  if (drop_tol >= 0.0) {
    const double thr = __dmul_rn(drop_tol, rmax);
    for (int q = lane; q < cnt; q += 32) {
      const double mag = fabs(vals[q]);
      const bool diag = square_keep_diag && keys[q] == gi;
      kc += diag || !(mag < thr && mag < rmax);
    }
  }
  row_counts(cnt, drop_tol, lane, len, kept, i, kc);
}

template <int kHashCap, bool RANK>
__device__ __forceinline__ bool warp_row(int i, int lane, int32_t* __restrict__ keys, double* __restrict__ vals,
                                         int32_t* __restrict__ pref, double* __restrict__ pbuf,
                                         const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                         const double* __restrict__ av, const int32_t* __restrict__ brp,
                                         const int32_t* __restrict__ bci, const double* __restrict__ bv,
                                         const int64_t* __restrict__ off, int32_t* __restrict__ scol,
                                         double* __restrict__ sval, int32_t* __restrict__ len,
                                         int32_t* __restrict__ kept, double drop_tol, int square_keep_diag,
                                         const int32_t* __restrict__ bmap, int rb) {
  const int s = arp[i], na = arp[i + 1] - s;
  if (na > kWarpA) return true;
  // prefix of the B-row lengths of this A row (warp scan); empty A rows
  // (e.g. a C point without F neighbours in A_cf) give total = 0
  if (lane == 0) pref[0] = 0;
  __syncwarp();
  for (int k0 = 0; k0 < na; k0 += 32) {
    const int k = k0 + lane;
    int l = 0;
    if (k < na) {
      const int j = brow(bmap, aci[s + k]);
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
      const int j = brow(bmap, aci[s + lo]);
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
    if (__any_sync(0xffffffffu, overflow)) return true;
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
  int32_t* oc = scol + off[i];
  double* ov = sval + off[i];
  if (RANK && cnt <= 32) {
    finish_rank<1>(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  } else if (RANK && cnt <= 64) {
    finish_rank<2>(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  } else if (RANK && cnt <= 128) {
    finish_rank<4>(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  } else if (cnt <= 32) {
    finish_reg<1>(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  } else if (cnt <= 64) {
    finish_reg<2>(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  } else if (cnt <= 128) {
    finish_reg<4>(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  } else {
    finish_smem(keys, vals, cnt, lane, i, rb + i, oc, ov, drop_tol, square_keep_diag, len, kept);
  }
  return false;
}

// kSpgWarps warps per block, one list row per warp at a time; rows that
// overflow the table are appended to next_list
template <int kHashCap, int kSpgWarps, bool RANK>
__global__ void __launch_bounds__(kSpgWarps * 32, kSpgWarps == 8 ? 7 : 1)
spgemm_warp_list(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                 int32_t* __restrict__ next_list, int32_t* __restrict__ next_count,
                 const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                 const double* __restrict__ av, const int32_t* __restrict__ brp,
                 const int32_t* __restrict__ bci, const double* __restrict__ bv,
                 const int64_t* __restrict__ off, int32_t* __restrict__ scol, double* __restrict__ sval,
                 int32_t* __restrict__ len, int32_t* __restrict__ kept, double drop_tol,
                 int square_keep_diag, const int32_t* __restrict__ bmap, int rb) {
  __shared__ __align__(16) int32_t keys_all[kSpgWarps][kHashCap];
  __shared__ double vals_all[kSpgWarps][kHashCap];
  __shared__ int32_t pref_all[kSpgWarps][kWarpA + 1];
  __shared__ double pbuf_all[kSpgWarps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nrows = *count;
  for (int q = blockIdx.x * kSpgWarps + w; q < nrows; q += gridDim.x * kSpgWarps) {
    const int i = list[q];
    const bool ovf = warp_row<kHashCap, RANK>(i, lane, keys_all[w], vals_all[w], pref_all[w], pbuf_all[w], arp,
                                        aci, av, brp, bci, bv, off, scol, sval, len, kept, drop_tol,
                                        square_keep_diag, bmap, rb);
    if (ovf && lane == 0) next_list[atomicAdd(next_count, 1)] = i;
    __syncwarp();
  }
}

// thread per row: sorted insertion into the row's scratch segment
__device__ __forceinline__ void thread_row(int i, const int32_t* __restrict__ arp,
                                           const int32_t* __restrict__ aci, const double* __restrict__ av,
                                           const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                           const double* __restrict__ bv, const int64_t* __restrict__ off,
                                           int32_t* __restrict__ scol, double* __restrict__ sval,
                                           int32_t* __restrict__ len, int32_t* __restrict__ kept,
                                           double drop_tol, int square_keep_diag,
                                           const int32_t* __restrict__ bmap, int rb) {
  int32_t* cols = scol + off[i];
  double* vals = sval + off[i];
  int L = 0;
  for (int k = arp[i]; k < arp[i + 1]; ++k) {
    const double a = av[k];
    const int j = brow(bmap, aci[k]);
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
    const bool diag = square_keep_diag && cols[q] == rb + i;
    kc += diag || !(mag < thr && mag < row_max);
  }
  kept[i] = kc;
}

// rows of `list` (or every row when list == nullptr), grid-stride
__global__ void spgemm_accumulate(int n, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                                  const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                  const double* __restrict__ av, const int32_t* __restrict__ brp,
                                  const int32_t* __restrict__ bci, const double* __restrict__ bv,
                                  const int64_t* __restrict__ off, int32_t* __restrict__ scol,
                                  double* __restrict__ sval, int32_t* __restrict__ len,
                                  int32_t* __restrict__ kept, double drop_tol, int square_keep_diag,
                                  const int32_t* __restrict__ bmap, int rb) {
  const int rows = list ? *count : n;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < rows; q += gridDim.x * blockDim.x)
    thread_row(list ? list[q] : q, arp, aci, av, brp, bci, bv, off, scol, sval, len, kept, drop_tol,
               square_keep_diag, bmap, rb);
}

__global__ void spgemm_compact(int n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ scol, const double* __restrict__ sval,
                               const int32_t* __restrict__ len, const int32_t* __restrict__ orp,
                               int32_t* __restrict__ oci, double* __restrict__ ov, double drop_tol,
                               int square_keep_diag, int rb) {
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
    const bool diag = square_keep_diag && cols[q] == rb + i;
    if (diag || !(mag < thr && mag < row_max)) {
      oci[o] = cols[q];
      ov[o++] = vals[q];
    }
  }
}

}  // namespace

void spgemm(Ctx& c, const Csr& a, const Csr& b, Csr& out, double drop_tol, bool keep_diag,
            const int32_t* bmap, int row_base, int64_t square_n) {
  if (!bmap && a.m != b.n) throw InvalidArgument("spgemm: dimension mismatch");
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
  static const bool thread_only = [] {
    const char* e = getenv("AIRG_SPGEMM");
    return e && !strcmp(e, "thread");
  }();
  DBuf<int64_t> ub(c, (size_t)n), off(c, (size_t)n + 1);
  DBuf<int32_t> lists(c, thread_only ? 1 : 4 * (size_t)n), counts(c, 4);
  counts.zero(c);
  LAUNCH(c, spgemm_bound, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, b.rp.p, bmap, ub.p, lists.p,
         counts.p, thread_only ? 0 : 1);
  const int64_t total = exclusive_scan64(c, ub.p, off.p, n);
  DBuf<int32_t> scol(c, (size_t)total), len(c, (size_t)n), kept(c, (size_t)n);
  DBuf<double> sval(c, (size_t)total);
  // square rule (keep the diagonal): the product is square -- for a row slab,
  // square_n is the global row count
  const int sq = (keep_diag && (square_n >= 0 ? square_n : (int64_t)a.n) == b.m) ? 1 : 0;
  const unsigned tgrid = (unsigned)std::min<int64_t>(blocks_for(n, 128), 16 * c.num_sms);
  if (thread_only) {
    LAUNCH(c, spgemm_accumulate, tgrid, 128, 0, n, (const int32_t*)nullptr, (const int32_t*)nullptr,
           a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p,
           off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, bmap, row_base);
  } else {
    // list 0: few products -> thread per row; list 1: warp + 256-slot table,
    // overflow -> list 2: one warp per block + 2048-slot table, overflow ->
    // list 3: thread per row. Persistent grids read the list lengths on device.
    const int64_t N = n;
    // AIRG_SPGEMM_SORT=bitonic: the register sort network instead of rank placement
    static const bool rank = [] {
      const char* e = getenv("AIRG_SPGEMM_SORT");
      return !(e && !strcmp(e, "bitonic"));
    }();
    auto* k256 = rank ? spgemm_warp_list<256, 8, true> : spgemm_warp_list<256, 8, false>;
    auto* k2048 = rank ? spgemm_warp_list<2048, 1, true> : spgemm_warp_list<2048, 1, false>;
    // the persistent grid is ONE wave: more CTAs than fit would run their
    // statically assigned rows after the first wave drains
    static int per_sm = 0;
    if (!per_sm) {
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k256, 256, 0));
      per_sm = std::max(per_sm, 1);
    }
    LAUNCH(c, spgemm_accumulate, tgrid, 128, 0, n, (const int32_t*)lists.p, (const int32_t*)counts.p,
           a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p,
           off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, bmap, row_base);
    LAUNCH(c, k256, (unsigned)std::min<int64_t>((N + 7) / 8, (int64_t)per_sm * c.num_sms), 256, 0,
           (const int32_t*)(lists.p + N), (const int32_t*)(counts.p + 1), lists.p + 2 * N, counts.p + 2,
           a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p,
           off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, bmap, row_base);
    LAUNCH(c, k2048, (unsigned)std::min<int64_t>(N, 8 * c.num_sms), 32, 0,
           (const int32_t*)(lists.p + 2 * N), (const int32_t*)(counts.p + 2), lists.p + 3 * N, counts.p + 3,
           a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p,
           off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, bmap, row_base);
    LAUNCH(c, spgemm_accumulate, tgrid, 128, 0, n, (const int32_t*)(lists.p + 3 * N),
           (const int32_t*)(counts.p + 3), a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p,
           off.p, scol.p, sval.p, len.p, kept.p, drop_tol, sq, bmap, row_base);
  }
  const int64_t nnz = exclusive_scan(c, kept.p, r.rp.p, n);
  r.nnz = nnz;
  r.ci.alloc(c, (size_t)nnz);
  r.v.alloc(c, (size_t)nnz);
  LAUNCH(c, spgemm_compact, blocks_for(n, 256), 256, 0, n, off.p, scol.p, sval.p, len.p, r.rp.p,
         r.ci.p, r.v.p, drop_tol, sq, row_base);
  out = std::move(r);
}

}  // namespace airg
