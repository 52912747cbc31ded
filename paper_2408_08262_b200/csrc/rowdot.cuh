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

}  // namespace airg
