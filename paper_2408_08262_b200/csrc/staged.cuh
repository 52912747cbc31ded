// Row kernels with the block's matrix slice staged in shared memory by the
// bulk-copy (TMA) engine before the dependency wait (AIRG_STAGE=1).
//
// A 128-row block of a CSR operator owns one contiguous nnz range
// [rp[r0], rp[r0+128]). The matrix is constant during a solve, so the block
// issues two cp.async.bulk copies (values, then column indices) of that
// range into shared memory BEFORE griddepcontrol.wait: the copy engine
// streams the slice with full-line requests while the predecessor kernel
// drains, and no (column, value) pair occupies a register or an L1
// wavefront of a per-thread uncoalesced load. After the wait a thread walks
// its row from shared memory and only the x gathers go to global memory --
// the sole dependent round trip left on the row's critical path. Each row is
// still one sequential, separately rounded sum in column order, so the bits
// are those of rows_thread / rows_thread_fc (sparse.cpp:193-198,
// solve.cpp:72-80).
//
// Bulk copies move 16-byte multiples from 16-byte aligned addresses: the
// staged range starts at rp[r0] rounded down to 4 entries, the bulk part
// ends at rp[r1] rounded down to 4 entries, and the <= 3 entries after it
// are stored by the threads. Blocks whose range exceeds the view's capacity
// (TileView::stage entries) walk their rows from global memory instead.
#pragma once

// included by tiled.cuh before its launch macros (TileView, has_pre, the
// ordered dots are defined above that point)

namespace airg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

template <class E, class = void>
struct pre_of {
  using type = int;
};
template <class E>
struct pre_of<E, std::void_t<typename E::Pre>> {
  using type = typename E::Pre;
};

#ifndef AIRG_STAGE_XB
#define AIRG_STAGE_XB 8
#endif
constexpr int kStageXB = AIRG_STAGE_XB;  // x gathers in flight per thread

// ordered row sums from the staged slice (sv/sci indexed from k0a)
template <bool FC>
__device__ __forceinline__ void staged_dot(int s, int e, int k0a, const double* sv, const int32_t* sci,
                                           const double* __restrict__ x, double& sf, double& sc) {
  sf = 0.0;
  sc = 0.0;
  for (int k0 = s; k0 < e; k0 += kStageXB) {
    double xv[kStageXB];
    int cs[kStageXB];
#pragma unroll
    for (int j = 0; j < kStageXB; ++j) {
      cs[j] = k0 + j < e ? sci[k0 + j - k0a] : 0;
      xv[j] = k0 + j < e ? __ldg(x + (FC ? (cs[j] & 0x7fffffff) : cs[j])) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kStageXB; ++j) {
      if (k0 + j < e) {
        const double p = __dmul_rn(sv[k0 + j - k0a], xv[j]);
        if (FC && cs[j] < 0)
          sc = __dadd_rn(sc, p);
        else
          sf = __dadd_rn(sf, p);
      }
    }
  }
}

template <class Epi, bool FC>
__global__ void __launch_bounds__(kTileThreads) rows_staged(TileView m, const double* __restrict__ x, Epi epi) {
  extern __shared__ __align__(16) unsigned char stage_raw[];
  __shared__ __align__(8) unsigned long long mbar;
  double* sv = reinterpret_cast<double*>(stage_raw);
  int32_t* sci = reinterpret_cast<int32_t*>(sv + m.stage);
  const int r0 = blockIdx.x * kTileThreads;
  const int i = r0 + threadIdx.x;
  const bool live = i < m.nrows;
  const int r1 = min(r0 + kTileThreads, m.nrows);
  const int K0 = __ldg(m.rp + r0), K1 = __ldg(m.rp + r1);
  const int k0a = K0 & ~3;
  const bool staged = K1 - k0a <= m.stage;
  const int k1f = max(K1 & ~3, k0a);
  const uint32_t bar = smem_u32(&mbar);
  int s = 0, e = 0;
  if (live) {
    s = __ldg(m.rp + i);
    e = __ldg(m.rp + i + 1);
  }
  if (staged) {
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t nb = (uint32_t)(k1f - k0a);
      mbar_arrive_tx(bar, nb * 12u);
      if (nb) {
        bulk_g2s(sv, m.v + k0a, nb * 8u, bar);
        bulk_g2s(sci, m.ci + k0a, nb * 4u, bar);
      }
    }
    for (int k = k1f + (int)threadIdx.x; k < K1; k += kTileThreads) {
      sv[k - k0a] = __ldg(m.v + k);
      sci[k - k0a] = __ldg(m.ci + k);
    }
  }
  typename pre_of<Epi>::type pre{};
  if constexpr (has_pre<Epi>::value) {
    if (live) pre = epi.pre(i);
  }
  pdl_wait();
  pdl_trigger();
  if (staged) {
    mbar_wait(bar, 0);
    __syncthreads();
  }
  if (live) {
    double sf, sc;
    if (staged) {
      staged_dot<FC>(s, e, k0a, sv, sci, x, sf, sc);
    } else if (FC) {
      dot_ordered_fc(s, e, m.ci, m.v, x, sf, sc);
    } else {
      sf = dot_ordered(s, e, m.ci, m.v, x);
      sc = 0.0;
    }
    if constexpr (FC) {
      if constexpr (has_pre<Epi>::value)
        epi.row2_pre(i, sf, sc, pre);
      else
        epi.row2(i, sf, sc);
    } else {
      if constexpr (has_pre<Epi>::value)
        epi.row_pre(i, sf, pre);
      else
        epi.row(i, sf);
    }
  }
  if constexpr (!FC) epi.finish();
}

inline size_t stage_smem(const TileView& m) { return (size_t)m.stage * 12u; }

}  // namespace airg
