// Long-row kernels with a warp's 32 rows staged as products (AIRG_W32=1).
//
// A warp owns 32 consecutive rows, i.e. one contiguous nnz range. Phase 1
// walks that range with unit stride across the lanes -- column, value and x
// gather of entry k on lane k % 32, U entries per lane in flight -- and
// stores each product a_k * x_{c_k}, rounded exactly as the reference rounds
// it, in the warp's slice of shared memory (plus the C-column flag for the
// F-row residual). Phase 2 (after __syncwarp) has each lane add ITS row's
// products in column order from 0.0: the reference's sequential sum
// (sparse.cpp:193-198; solve.cpp:72-80), so the bits are those of the
// thread-per-row kernels, while every global load of phase 1 is coalesced
// and independent of the others. Warps whose range exceeds the slice walk
// their rows per thread from global memory.
#pragma once

// included by tiled.cuh before its launch macros

namespace airg {

#ifndef AIRG_W32_CAP
#define AIRG_W32_CAP 1024
#endif
#ifndef AIRG_W32_U
#define AIRG_W32_U 4
#endif
constexpr int kW32Cap = AIRG_W32_CAP;  // products per warp slice
constexpr int kW32U = AIRG_W32_U;      // entries per lane in flight in phase 1

template <bool FC>
constexpr size_t w32_smem() {
  return (size_t)(kTileThreads / 32) * kW32Cap * (sizeof(double) + (FC ? 1 : 0));
}

template <class Epi, bool FC>
__global__ void rows_w32(TileView m, const double* __restrict__ x, Epi epi);

// slices above 48 KB need the opt-in once per instantiation
template <class Epi, bool FC>
inline size_t w32_smem_checked() {
  static const size_t b = [] {
    if (w32_smem<FC>() > 48 * 1024)
      cudaFuncSetAttribute(rows_w32<Epi, FC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w32_smem<FC>());
    return w32_smem<FC>();
  }();
  return b;
}

template <class Epi, bool FC>
__global__ void __launch_bounds__(kTileThreads) rows_w32(TileView m, const double* __restrict__ x, Epi epi) {
  extern __shared__ __align__(16) unsigned char w32_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* prod = reinterpret_cast<double*>(w32_raw) + w * kW32Cap;
  uint8_t* isc = w32_raw + (size_t)(kTileThreads / 32) * kW32Cap * sizeof(double) + w * kW32Cap;
  const int r0 = (blockIdx.x * (kTileThreads / 32) + w) * 32;
  const int i = r0 + lane;
  const bool live = i < m.nrows;
  const bool warp_live = r0 < m.nrows;
  const int r1 = min(r0 + 32, m.nrows);
  int s = 0, e = 0, K0 = 0, K1 = 0;
  if (warp_live) {
    K0 = __ldg(m.rp + r0);
    K1 = __ldg(m.rp + r1);
  }
  if (live) {
    s = __ldg(m.rp + i);
    e = __ldg(m.rp + i + 1);
  }
  const int cnt = K1 - K0;
  const bool staged = cnt <= kW32Cap;
  // first U entries of every lane: static matrix data, before the wait
  int c[kW32U];
  double a[kW32U];
  if (staged) {
#pragma unroll
    for (int u = 0; u < kW32U; ++u) {
      const int k = lane + 32 * u;
      c[u] = k < cnt ? __ldg(m.ci + K0 + k) : 0;
      a[u] = k < cnt ? __ldg(m.v + K0 + k) : 0.0;
    }
  }
  typename pre_of<Epi>::type pre{};
  if constexpr (has_pre<Epi>::value) {
    if (live) pre = epi.pre(i);
  }
  pdl_wait();
  pdl_trigger();
  double sf = 0.0, sc = 0.0;
  if (staged) {
    for (int k0 = 0; k0 < cnt; k0 += 32 * kW32U) {
      double xv[kW32U];
#pragma unroll
      for (int u = 0; u < kW32U; ++u) {
        const int k = k0 + lane + 32 * u;
        xv[u] = k < cnt ? __ldg(x + (FC ? (c[u] & 0x7fffffff) : c[u])) : 0.0;
      }
      int cn[kW32U];
      double an[kW32U];
#pragma unroll
      for (int u = 0; u < kW32U; ++u) {
        const int k = k0 + 32 * kW32U + lane + 32 * u;
        cn[u] = k < cnt ? __ldg(m.ci + K0 + k) : 0;
        an[u] = k < cnt ? __ldg(m.v + K0 + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kW32U; ++u) {
        const int k = k0 + lane + 32 * u;
        if (k < cnt) {
          prod[k] = __dmul_rn(a[u], xv[u]);
          if (FC) isc[k] = c[u] < 0;
        }
        c[u] = cn[u];
        a[u] = an[u];
      }
    }
    __syncwarp();
    if (live) {
      for (int k = s - K0; k < e - K0; ++k) {
        const double p = prod[k];
        if (FC && isc[k])
          sc = __dadd_rn(sc, p);
        else
          sf = __dadd_rn(sf, p);
      }
    }
  } else if (live) {
    if (FC)
      dot_ordered_fc(s, e, m.ci, m.v, x, sf, sc);
    else
      sf = dot_ordered(s, e, m.ci, m.v, x);
  }
  if (live) {
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

}  // namespace airg
