// The coarse tail of the V-cycle as ONE persistent kernel.
//
// Below a few 10^5 rows every V-cycle operation is a few microseconds of
// work behind a kernel boundary, and the C2 hierarchy has a dozen such
// levels (2 x 6 boundaries each plus the coarse iterations). The tail kernel
// runs the restriction of those levels, the coarse polynomial iterations and
// their prolongation / F-smoothing as a list of PHASES -- each phase is one
// of the row operations of solve.cu, over all rows of one operator -- with
// a grid-wide barrier between consecutive phases. All CTAs are co-resident
// (cooperative launch), rows are spread over the whole grid, and each row is
// the same sequential, separately rounded sum as in the per-level kernels,
// so the result is bit-identical to the kernel-per-phase V-cycle.
//
// Vectors written by an earlier phase of the same launch are read with
// L2-coherent loads (ld.global.cg, never a stale L1 line); only the matrices
// go through the read-only path.
//
// Two barriers: k_tail spans the whole GPU with a software grid barrier
// (cooperative launch); k_tail_cluster runs the small levels on ONE thread-
// block cluster (up to 16 SMs) with the hardware cluster barrier.
#pragma once

#include <cooperative_groups.h>

#include "rowdot.cuh"

namespace airg {

enum TailKind : int {
  kTailStore = 0,    // out = A x                               (restriction)
  kTailCres = 1,     // out = b - A x                           (coarse residual)
  kTailCupd = 2,     // out = (first ? 0 : out) + 1.0 * (A x)   (coarse update)
  kTailProlong = 3,  // out[i] = 0 + 1.0 * (0 + 1.0 * x[idx[i]]) or 0
  kTailFres1 = 4,    // out[k] = (b[idx k] - A_F x) - A_C x; out2[k] = A_C x
  kTailFres2 = 5,    // out[k] = (b[idx k] - A_FF x) - in2[k]
  kTailFupd = 6,     // out[idx k] += A x
};

struct TailPhase {
  int kind;
  int n;  // rows
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
  const double* x;
  const double* b;
  const int32_t* idx;
  double* out;
  double* out2;
  const double* in2;
  int first;
};

constexpr int kTailThreads = 1024;  // one CTA per SM: few barrier arrivals

// the software grid barrier lives in common.cuh (grid_barrier)
__device__ __forceinline__ void tail_grid_barrier(unsigned* bar, unsigned nblocks) { grid_barrier(bar, nblocks); }

// ordered row sums with coherent x loads (x may have been written earlier in
// this launch)
__device__ __forceinline__ double tail_dot(int s, int e, const int32_t* __restrict__ ci,
                                           const double* __restrict__ v, const double* x) {
  double acc = 0.0;
  for (int k0 = s; k0 < e; k0 += kRowBatch) {
    int c[kRowBatch];
    double a[kRowBatch], xv[kRowBatch];
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) {
      c[j] = k0 + j < e ? __ldg(ci + k0 + j) : 0;
      a[j] = k0 + j < e ? __ldg(v + k0 + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) xv[j] = (k0 + j < e) ? __ldcg(x + c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j)
      if (k0 + j < e) acc = __dadd_rn(acc, __dmul_rn(a[j], xv[j]));
  }
  return acc;
}

__device__ __forceinline__ void tail_dot_fc(int s, int e, const int32_t* __restrict__ ci,
                                            const double* __restrict__ v, const double* x, double& sf,
                                            double& sc) {
  sf = 0.0;
  sc = 0.0;
  for (int k0 = s; k0 < e; k0 += kRowBatch) {
    int c[kRowBatch];
    double a[kRowBatch], xv[kRowBatch];
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) {
      c[j] = k0 + j < e ? __ldg(ci + k0 + j) : 0;
      a[j] = k0 + j < e ? __ldg(v + k0 + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kRowBatch; ++j) xv[j] = (k0 + j < e) ? __ldcg(x + (c[j] & 0x7fffffff)) : 0.0;
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

__device__ __forceinline__ void tail_row(const TailPhase& P, int i) {
  switch (P.kind) {
    case kTailProlong: {
      const int j = __ldg(P.idx + i);
      const double pe = j >= 0 ? __dadd_rn(0.0, __dmul_rn(1.0, __ldcg(P.x + j))) : 0.0;
      P.out[i] = __dadd_rn(0.0, __dmul_rn(1.0, pe));
      return;
    }
    case kTailFres1: {
      double sf, sc;
      tail_dot_fc(__ldg(P.rp + i), __ldg(P.rp + i + 1), P.ci, P.v, P.x, sf, sc);
      P.out2[i] = sc;
      P.out[i] = __dsub_rn(__dsub_rn(__ldcg(P.b + __ldg(P.idx + i)), sf), sc);
      return;
    }
    default:
      break;
  }
  const double acc = tail_dot(__ldg(P.rp + i), __ldg(P.rp + i + 1), P.ci, P.v, P.x);
  switch (P.kind) {
    case kTailStore:
      P.out[i] = acc;
      break;
    case kTailCres:
      P.out[i] = __dsub_rn(__ldcg(P.b + i), acc);
      break;
    case kTailCupd: {
      const double e0 = P.first ? 0.0 : __ldcg(P.out + i);
      P.out[i] = __dadd_rn(e0, __dmul_rn(1.0, acc));
      break;
    }
    case kTailFres2:
      P.out[i] = __dsub_rn(__dsub_rn(__ldcg(P.b + __ldg(P.idx + i)), acc), __ldcg(P.in2 + i));
      break;
    case kTailFupd: {
      const int r = __ldg(P.idx + i);
      P.out[r] = __dadd_rn(__ldcg(P.out + r), acc);
      break;
    }
    default:
      break;
  }
}

// The phase table travels as the kernel's parameter block (captured into the
// CUDA graph with the launch; <= 32 KB of parameters on sm_70+).
constexpr int kMaxTailPhases = 256;
struct TailTable {
  int nph;
  TailPhase ph[kMaxTailPhases];
};
static_assert(sizeof(TailTable) < 32000, "tail table exceeds the kernel parameter limit");

__global__ void __launch_bounds__(kTailThreads) k_tail(const __grid_constant__ TailTable t, unsigned* bar) {
  const int nthreads = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nph = t.nph;
  for (int p = 0; p < nph; ++p) {
    const TailPhase& P = t.ph[p];
    for (int i = tid; i < P.n; i += nthreads) tail_row(P, i);
    if (p + 1 < nph) tail_grid_barrier(bar, gridDim.x);
  }
}

// One cluster of CTAs walks the phase list; rows are spread over the
// cluster's threads and consecutive phases are separated by the hardware
// cluster barrier (release / acquire at cluster scope).
__global__ void __launch_bounds__(kTailThreads) k_tail_cluster(const __grid_constant__ TailTable t) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int nthreads = (int)cl.num_blocks() * blockDim.x;
  const int tid = (int)cl.block_rank() * blockDim.x + threadIdx.x;
  const int nph = t.nph;
  for (int p = 0; p < nph; ++p) {
    const TailPhase& P = t.ph[p];
    for (int i = tid; i < P.n; i += nthreads) tail_row(P, i);
    if (p + 1 < nph) cl.sync();
  }
}

}  // namespace airg
