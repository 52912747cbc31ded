// Ordered (bit-exact) row dot products with batched loads.
//
// The reference sums a row left to right in column order with separately
// rounded products (sparse.cpp:193-198). A thread keeps exactly that order,
// but issues the index/value loads of B entries, then the B gathers of x,
// before the B dependent adds: B independent memory requests in flight per
// thread instead of one, which turns the latency-bound serial loop into a
// bandwidth-bound one on the long coarse-level rows.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace airg {

constexpr int kRowBatch = 8;

__device__ __forceinline__ double dot_ordered(int s, int e, const int32_t* __restrict__ ci,
                                              const double* __restrict__ v,
                                              const double* __restrict__ x) {
  double acc = 0.0;
  for (int k0 = s; k0 < e; k0 += kRowBatch) {
    int c[kRowBatch];
    double a[kRowBatch], xv[kRowBatch];
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) {
      const int k = k0 + j;
      c[j] = k < e ? __ldg(ci + k) : 0;
      a[j] = k < e ? __ldg(v + k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) xv[j] = (k0 + j < e) ? __ldg(x + c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j)
      if (k0 + j < e) acc = __dadd_rn(acc, __dmul_rn(a[j], xv[j]));
  }
  return acc;
}

// F-row residual variant: columns with bit 31 set are C columns; the F and C
// partial sums are kept apart (solve.cpp:72-80).
__device__ __forceinline__ void dot_ordered_fc(int s, int e, const int32_t* __restrict__ ci,
                                               const double* __restrict__ v,
                                               const double* __restrict__ x, double& sf,
                                               double& sc) {
  sf = 0.0;
  sc = 0.0;
  for (int k0 = s; k0 < e; k0 += kRowBatch) {
    int c[kRowBatch];
    double a[kRowBatch], xv[kRowBatch];
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) {
      const int k = k0 + j;
      c[j] = k < e ? __ldg(ci + k) : 0;
      a[j] = k < e ? __ldg(v + k) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) xv[j] = (k0 + j < e) ? __ldg(x + (c[j] & 0x7fffffff)) : 0.0;
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) {
      if (k0 + j < e) {
        const double p = __dmul_rn(a[j], xv[j]);
        if (c[j] >= 0)
          sf = __dadd_rn(sf, p);
        else
          sc = __dadd_rn(sc, p);
      }
    }
  }
}

// Aligned-vector variants: the row is walked in 4-entry groups aligned to 16
// bytes (one int4 of columns, two double2 of values per group; entries of
// the group outside [s, e) are loaded but not used), so a thread issues a
// quarter of the column and half of the value requests of the scalar loop.
// The products and the left-to-right sum are the same as above. VB = entries
// per batch (4 or 8). nnz bounds the vector loads (tail groups go scalar).
template <int VB>
__device__ __forceinline__ void load_group(int k4, int nnz, const int32_t* __restrict__ ci,
                                           const double* __restrict__ v, int* c, double* a) {
#pragma unroll
  for (int g = 0; g < VB; g += 4) {
    const int k = k4 + g;
    if (k + 4 <= nnz) {
      const int4 cc = __ldg(reinterpret_cast<const int4*>(ci + k));
      const double2 p = __ldg(reinterpret_cast<const double2*>(v + k));
      const double2 q = __ldg(reinterpret_cast<const double2*>(v + k + 2));
      c[g] = cc.x; c[g + 1] = cc.y; c[g + 2] = cc.z; c[g + 3] = cc.w;
      a[g] = p.x; a[g + 1] = p.y; a[g + 2] = q.x; a[g + 3] = q.y;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        c[g + j] = k + j < nnz ? __ldg(ci + k + j) : 0;
        a[g + j] = k + j < nnz ? __ldg(v + k + j) : 0.0;
      }
    }
  }
}

template <int VB>
__device__ __forceinline__ double dot_ordered_vec(int s, int e, int nnz, const int32_t* __restrict__ ci,
                                                  const double* __restrict__ v,
                                                  const double* __restrict__ x) {
  double acc = 0.0;
  for (int k4 = s & ~3; k4 < e; k4 += VB) {
    int c[VB];
    double a[VB], xv[VB];
    load_group<VB>(k4, nnz, ci, v, c, a);
#pragma unroll
    for (int j = 0; j < VB; ++j) xv[j] = (k4 + j >= s && k4 + j < e) ? __ldg(x + c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < VB; ++j)
      if (k4 + j >= s && k4 + j < e) acc = __dadd_rn(acc, __dmul_rn(a[j], xv[j]));
  }
  return acc;
}

template <int VB>
__device__ __forceinline__ void dot_ordered_fc_vec(int s, int e, int nnz, const int32_t* __restrict__ ci,
                                                   const double* __restrict__ v,
                                                   const double* __restrict__ x, double& sf, double& sc) {
  sf = 0.0;
  sc = 0.0;
  for (int k4 = s & ~3; k4 < e; k4 += VB) {
    int c[VB];
    double a[VB], xv[VB];
    load_group<VB>(k4, nnz, ci, v, c, a);
#pragma unroll
    for (int j = 0; j < VB; ++j)
      xv[j] = (k4 + j >= s && k4 + j < e) ? __ldg(x + (c[j] & 0x7fffffff)) : 0.0;
#pragma unroll
    for (int j = 0; j < VB; ++j) {
      if (k4 + j >= s && k4 + j < e) {
        const double p = __dmul_rn(a[j], xv[j]);
        if (c[j] >= 0)
          sf = __dadd_rn(sf, p);
        else
          sc = __dadd_rn(sc, p);
      }
    }
  }
}

// ---- prefetching form (used by the PDL row kernels, tiled.cuh) -------------
// The matrix is constant during a solve, so a row kernel may load its row
// bounds and first batch of (column, value) pairs BEFORE griddepcontrol.wait
// -- overlapping them with the tail of the kernel it depends on -- and only
// the x gathers wait for the predecessor. VEC: batches start at the 16-byte
// aligned group containing s and use vector loads (load_group).
template <int VB, bool VEC>
struct RowBatch {
  int c[VB];
  double a[VB];
  __device__ __forceinline__ void load(int k0, int e, int nnz, const int32_t* __restrict__ ci,
                                       const double* __restrict__ v) {
    if (VEC) {
      load_group<VB>(k0, nnz, ci, v, c, a);
    } else {
#pragma unroll
      for (int j = 0; j < VB; ++j) {
        c[j] = k0 + j < e ? __ldg(ci + k0 + j) : 0;
        a[j] = k0 + j < e ? __ldg(v + k0 + j) : 0.0;
      }
    }
  }
};

template <int VB, bool VEC>
__device__ __forceinline__ int batch_start(int s) {
  return VEC ? (s & ~3) : s;
}

// Software-pipelined batches (measured 0.953 -> 0.868 ms per C2 iteration):
// batch k+1's (column, value) loads are issued together with batch k's x
// gathers, so a row costs one dependent memory round trip per batch instead
// of two. The adds stay one left-to-right chain per row.
template <int VB, bool VEC>
__device__ __forceinline__ double dot_prefetched(int s, int e, int nnz, const int32_t* __restrict__ ci,
                                                 const double* __restrict__ v, const double* __restrict__ x,
                                                 RowBatch<VB, VEC>& b) {
  double acc = 0.0;
  for (int k0 = batch_start<VB, VEC>(s); k0 < e; k0 += VB) {
    double xv[VB];
#pragma unroll
    for (int j = 0; j < VB; ++j) xv[j] = (k0 + j >= s && k0 + j < e) ? __ldg(x + b.c[j]) : 0.0;
    RowBatch<VB, VEC> nb;
    if (k0 + VB < e) nb.load(k0 + VB, e, nnz, ci, v);
#pragma unroll
    for (int j = 0; j < VB; ++j)
      if (k0 + j >= s && k0 + j < e) acc = __dadd_rn(acc, __dmul_rn(b.a[j], xv[j]));
    b = nb;
  }
  return acc;
}

// F-row variant: columns with bit 31 set are C columns; the F and C partial
// sums are kept apart (solve.cpp:72-80).
template <int VB, bool VEC>
__device__ __forceinline__ void dot_fc_prefetched(int s, int e, int nnz, const int32_t* __restrict__ ci,
                                                  const double* __restrict__ v, const double* __restrict__ x,
                                                  RowBatch<VB, VEC>& b, double& sf, double& sc) {
  sf = 0.0;
  sc = 0.0;
  for (int k0 = batch_start<VB, VEC>(s); k0 < e; k0 += VB) {
    double xv[VB];
#pragma unroll
    for (int j = 0; j < VB; ++j) xv[j] = (k0 + j >= s && k0 + j < e) ? __ldg(x + (b.c[j] & 0x7fffffff)) : 0.0;
    int cc[VB];
    double aa[VB];
#pragma unroll
    for (int j = 0; j < VB; ++j) {
      cc[j] = b.c[j];
      aa[j] = b.a[j];
    }
    if (k0 + VB < e) b.load(k0 + VB, e, nnz, ci, v);
#pragma unroll
    for (int j = 0; j < VB; ++j) {
      if (k0 + j >= s && k0 + j < e) {
        const double p = __dmul_rn(aa[j], xv[j]);
        if (cc[j] >= 0)
          sf = __dadd_rn(sf, p);
        else
          sc = __dadd_rn(sc, p);
      }
    }
  }
}

}  // namespace airg
