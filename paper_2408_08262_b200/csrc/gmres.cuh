// Device-resident GMRES kernels (solve.cu: the one-GPU solve; dist.cu: the
// distributed solve over row slabs). Included inside namespace airg { namespace
// { ... } } of each translation unit (every TU gets its own copy).
#pragma once

#include "hier.cuh"

namespace airg {
namespace {

constexpr int kGmMax = 32;      // restart lengths served on the device (m <= 32)
constexpr int kGmThreads = 256;
inline int gm_blocks(int64_t n) { return (int)std::max<int64_t>(1, (n + kGmThreads - 1) / kGmThreads); }


// Sum K per-lane vectors (K a power of two <= 32) over the warp: butterfly
// adds over the lane bits >= log2 K, then a transpose-reduce over the low
// bits (K (5 - log2 K) + K - 1 shuffles instead of 5 K); on return lane l
// holds the warp total of entry l mod K.
template <int K>
__device__ __forceinline__ double warp_transpose_sum(double (&v)[K]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= K; o >>= 1) {
#pragma unroll
    for (int t = 0; t < K; ++t) v[t] += __shfl_xor_sync(0xffffffffu, v[t], o);
  }
#pragma unroll
  for (int s = K / 2; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int t = 0; t < s; ++t) {
      const double send = up ? v[t] : v[t + s];
      const double keep = up ? v[t + s] : v[t];
      v[t] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// One element per thread (a grid of n / 256 blocks: enough independent
// loads in flight to cover the HBM latency); V_0..V_j of the element in
// registers, so the update and the following dots read V once; the dots of
// a warp reduced by one transpose-reduce. The code is specialised on K, the
// basis size rounded up to a power of two (warp-uniform branch on the
// device-side j): ncu showed the fixed 32-wide version issue bound (65 %).
// MODE 0: dots V_k . w;  1: w -= V h, then dots V_k . w;  2: w -= V h, then |w|^2;
// 3: dots V_k . w and V_k . v_j (fast mode's Gram-corrected CGS2, below).
// Per block, one partial per k: part[k * nblocks + block] (MODE 3: the Gram
// column at rows kGmMax + 1 + k).
template <int MODE, int K, bool LAZY>
__device__ __forceinline__ void gm_sweep_body(int64_t n, int jp1, const double* __restrict__ V,
                                              double* __restrict__ w, const double* hs, const double* vss,
                                              double* __restrict__ vnext, double* __restrict__ vin,
                                              double (*red)[kGmMax], double (*red2)[kGmMax],
                                              double* __restrict__ part, int vhint) {
  const int64_t i = (int64_t)blockIdx.x * kGmThreads + threadIdx.x;
  const bool live = i < n;
  double vk[K];
  if (LAZY && vhint) {  // fast mode: the basis is streamed with L2 evict_first
    const unsigned long long pol = l2_policy(vhint);
#pragma unroll
    for (int k = 0; k < K; ++k) vk[k] = (live && k < jp1) ? ld_hint(V + (int64_t)k * n + i, pol) : 0.0;
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) vk[k] = (live && k < jp1) ? __ldg(V + (int64_t)k * n + i) : 0.0;
  }
  if (LAZY) {  // V holds each v_k unnormalised; vss[k] = 1 / |v_k| (k_gm_step)
#pragma unroll
    for (int k = 0; k < K; ++k) vk[k] *= vss[k];
  }
  double wi = live ? w[i] : 0.0;
  if (MODE > 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) wi = fma(-hs[k], vk[k], wi);
    if (live) {
      if (LAZY && MODE == 2) {  // the next basis vector, unnormalised, and the V-cycle input
        vnext[i] = wi;
        vin[i] = wi;
      } else {
        w[i] = wi;
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 3) {  // V^T w and V^T v_j (the Gram column of the newest vector)
    double vj = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (k == jp1 - 1) vj = vk[k];
    if constexpr (K <= 16) {  // both K-vectors in ONE 2K-wide transpose-reduce
      double both[2 * K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        both[k] = vk[k] * wi;
        both[K + k] = vk[k] * vj;
      }
      const double t = warp_transpose_sum<2 * K>(both);
      const int e = lane & (2 * K - 1);
      if (lane < 2 * K) {
        if (e < K)
          red[warp][e] = t;
        else
          red2[warp][e - K] = t;
      }
    } else {
      double gk[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        gk[k] = vk[k] * vj;
        vk[k] *= wi;
      }
      const double t = warp_transpose_sum<K>(vk);
      const double tg = warp_transpose_sum<K>(gk);
      if (lane < K) {
        red[warp][lane] = t;
        red2[warp][lane] = tg;
      }
    }
  } else if (MODE < 2) {
#pragma unroll
    for (int k = 0; k < K; ++k) vk[k] *= wi;
    const double t = warp_transpose_sum<K>(vk);
    if (lane < K) red[warp][lane] = t;
  } else {
    double p = wi * wi;
#pragma unroll
    for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if (lane == 0) red[warp][0] = p;
  }
  __syncthreads();
  if ((int)threadIdx.x < (MODE != 2 ? jp1 : 1)) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kGmThreads / 32; ++q) v += red[q][threadIdx.x];
    part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = v;
  }
  if (MODE == 3 && (int)threadIdx.x >= 32 && (int)threadIdx.x < 32 + jp1) {
    const int k = threadIdx.x - 32;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kGmThreads / 32; ++q) v += red2[q][k];
    part[(int64_t)(kGmMax + 1 + k) * gridDim.x + blockIdx.x] = v;
  }
}

// LAZY (fast mode): the basis is stored unnormalised with its scales in vs
// (see GmPieces::step); MODE 2 then writes w'' = w - V h straight into
// V_{j+1} and the V-cycle input instead of w (no separate v = w / |w| pass).
template <int MODE, bool LAZY>
__global__ void __launch_bounds__(kGmThreads) k_gm_sweep(int64_t n, const double* __restrict__ V,
                                                         double* __restrict__ w, const GmDev* __restrict__ st,
                                                         const double* __restrict__ h, double* __restrict__ part,
                                                         const double* __restrict__ vs, double* __restrict__ Vw,
                                                         double* __restrict__ vin, int vhint) {
  __shared__ double hs[kGmMax];
  __shared__ double vss[LAZY ? kGmMax : 1];
  __shared__ double red[kGmThreads / 32][kGmMax];
  __shared__ double red2[MODE == 3 ? kGmThreads / 32 : 1][kGmMax];
  pdl_wait();
  pdl_trigger();
  const int jp1 = st->j + 1;
  if (threadIdx.x < kGmMax) {
    hs[threadIdx.x] = ((MODE == 1 || MODE == 2) && (int)threadIdx.x < jp1) ? h[threadIdx.x] : 0.0;
    if (LAZY) vss[threadIdx.x] = (int)threadIdx.x < jp1 ? vs[threadIdx.x] : 0.0;
  }
  __syncthreads();
  double* vnext = LAZY ? Vw + (int64_t)jp1 * n : nullptr;
  if (jp1 <= 4)
    gm_sweep_body<MODE, 4, LAZY>(n, jp1, V, w, hs, vss, vnext, vin, red, red2, part, vhint);
  else if (jp1 <= 8)
    gm_sweep_body<MODE, 8, LAZY>(n, jp1, V, w, hs, vss, vnext, vin, red, red2, part, vhint);
  else if (jp1 <= 16)
    gm_sweep_body<MODE, 16, LAZY>(n, jp1, V, w, hs, vss, vnext, vin, red, red2, part, vhint);
  else
    gm_sweep_body<MODE, 32, LAZY>(n, jp1, V, w, hs, vss, vnext, vin, red, red2, part, vhint);
}

// Fast-mode sweeps over the unnormalised basis (n even): two or four
// elements per thread with 16-byte loads of every column, the basis streamed
// in chunks of eight columns whatever j is -- registers no longer scale with the basis
// (the K-specialised register tile above needs 94 registers at K = 32: 23 %
// occupancy). MODE 3: the dots V_k . w and V_k . v_j (Gram column), one
// 16-wide transpose-reduce per chunk; MODE 2: w'' = w - V h into V_{j+1} and
// the V-cycle input, |w''|^2. Partials as k_gm_sweep (grid = n / (512 P)).
template <int MODE, int P>
__global__ void __launch_bounds__(kGmThreads) k_gm_sweep_fast(int64_t n, const double* __restrict__ V,
                                                              const double* __restrict__ w,
                                                              const GmDev* __restrict__ st,
                                                              const double* __restrict__ h, double* __restrict__ part,
                                                              const double* __restrict__ vs, double* __restrict__ Vw,
                                                              double* __restrict__ vin) {
  // P double2 pairs (2P elements) per thread, CH columns per chunk (16
  // measured 1.5-3 % slower per iteration)
  constexpr int CH = 8;
  __shared__ double hs[kGmMax];
  __shared__ double vss[kGmMax];
  __shared__ double red[kGmThreads / 32][2 * kGmMax];
  pdl_wait();
  pdl_trigger();
  const int jp1 = st->j + 1;
  if (threadIdx.x < kGmMax) {
    const bool in = (int)threadIdx.x < jp1;
    const double sc = in ? vs[threadIdx.x] : 0.0;
    vss[threadIdx.x] = sc;
    hs[threadIdx.x] = (MODE == 2 && in) ? h[threadIdx.x] * sc : 0.0;
  }
  __syncthreads();
  const int64_t i0 = 2 * P * ((int64_t)blockIdx.x * kGmThreads + threadIdx.x);
  const unsigned long long pol = l2_policy(1);
  const double2 zero2 = make_double2(0.0, 0.0);
  bool live[P];
  double2 wv[P];
#pragma unroll
  for (int u = 0; u < P; ++u) {
    live[u] = i0 + 2 * u < n;
    wv[u] = live[u] ? *reinterpret_cast<const double2*>(w + i0 + 2 * u) : zero2;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 3) {
    double2 vj[P];
    const double sj = vss[jp1 - 1];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      vj[u] = live[u] ? ld2_hint(V + (int64_t)(jp1 - 1) * n + i0 + 2 * u, pol) : zero2;
      vj[u].x *= sj;
      vj[u].y *= sj;
    }
    for (int c0 = 0; c0 < jp1; c0 += CH) {
      double2 vk[CH][P];
#pragma unroll
      for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int u = 0; u < P; ++u)
          vk[q][u] = (live[u] && c0 + q < jp1) ? ld2_hint(V + (int64_t)(c0 + q) * n + i0 + 2 * u, pol) : zero2;
      double both[2 * CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        double a = 0.0, g = 0.0;
#pragma unroll
        for (int u = 0; u < P; ++u) {
          a = fma(vk[q][u].x, wv[u].x, fma(vk[q][u].y, wv[u].y, a));
          g = fma(vk[q][u].x, vj[u].x, fma(vk[q][u].y, vj[u].y, g));
        }
        const double sk = (c0 + q < kGmMax) ? vss[c0 + q] : 0.0;
        both[q] = sk * a;
        both[CH + q] = sk * g;
      }
      const double t = warp_transpose_sum<2 * CH>(both);
      if (lane < 2 * CH) {
        const int k = c0 + (lane < CH ? lane : lane - CH);
        if (k < kGmMax) red[warp][lane < CH ? k : kGmMax + k] = t;
      }
    }
    __syncthreads();
    if ((int)threadIdx.x < jp1) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kGmThreads / 32; ++q) v += red[q][threadIdx.x];
      part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = v;
    }
    if ((int)threadIdx.x >= 32 && (int)threadIdx.x < 32 + jp1) {
      const int k = threadIdx.x - 32;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kGmThreads / 32; ++q) v += red[q][kGmMax + k];
      part[(int64_t)(kGmMax + 1 + k) * gridDim.x + blockIdx.x] = v;
    }
  } else {
    double2 acc[P];
#pragma unroll
    for (int u = 0; u < P; ++u) acc[u] = wv[u];
    for (int c0 = 0; c0 < jp1; c0 += CH) {
      double2 vk[CH][P];
#pragma unroll
      for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int u = 0; u < P; ++u)
          vk[q][u] = (live[u] && c0 + q < jp1) ? ld2_hint(V + (int64_t)(c0 + q) * n + i0 + 2 * u, pol) : zero2;
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const double hk = (c0 + q < kGmMax) ? hs[c0 + q] : 0.0;
#pragma unroll
        for (int u = 0; u < P; ++u) {
          acc[u].x = fma(-hk, vk[q][u].x, acc[u].x);
          acc[u].y = fma(-hk, vk[q][u].y, acc[u].y);
        }
      }
    }
    double p = 0.0;
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (live[u]) {
        *reinterpret_cast<double2*>(Vw + (int64_t)jp1 * n + i0 + 2 * u) = acc[u];
        *reinterpret_cast<double2*>(vin + i0 + 2 * u) = acc[u];
      }
      p = fma(acc[u].x, acc[u].x, fma(acc[u].y, acc[u].y, p));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if (lane == 0) red[warp][0] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kGmThreads / 32; ++q) v += red[q][0];
      part[blockIdx.x] = v;
    }
  }
}

// h[k] = sum over blocks of part[k][.] (k <= j, or k = 0 for the norm):
// one 1024-thread block per k, eight independent partial loads per thread
// in flight, a fixed reduction tree (deterministic)
constexpr int kFinThreads = 1024;
__global__ void __launch_bounds__(kFinThreads) k_gm_finish(const double* __restrict__ part, int nb,
                                                           const GmDev* __restrict__ st, int norm,
                                                           double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  // blocks 0..kGmMax-1: rows k <= j; blocks kGmMax..: the Gram rows kGmMax+1+k
  const int kb = blockIdx.x;
  const int k = kb < kGmMax ? kb : kb - kGmMax;
  if (k > (norm ? 0 : st->j)) return;
  const int row = kb < kGmMax ? k : kGmMax + 1 + k;
  __shared__ double sm[32];
  const double* p = part + (int64_t)row * nb;
  double s = 0.0;
  for (int b0 = threadIdx.x; b0 < nb; b0 += 8 * kFinThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int b = b0 + u * kFinThreads;
      v[u] = b < nb ? __ldg(p + b) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = sm[threadIdx.x];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[row] = s;
  }
}

// w = A z and Z_j = z (z = the V-cycle output; j from the device state)
// (lazy basis: the V-cycle ran on the unnormalised v_j, so z and A z are
// scaled by vs[j] = 1 / |v_j| here -- the V-cycle is linear)
struct EpiGmSpmv {
  double* w;
  const double* z;
  double* Z;
  const GmDev* st;
  int64_t n;
  const double* vs;  // null: v_j stored normalised
  __device__ void row(int i, double acc) const {
    const int j = st->j;
    if (vs) {
      const double s = vs[j];
      w[i] = s * acc;
      Z[(int64_t)j * n + i] = s * z[i];
    } else {
      w[i] = acc;
      Z[(int64_t)j * n + i] = z[i];
    }
  }
  __device__ void finish() const {}
};

// ||b||, the first cycle's start (x = 0, r = b, beta = ||b||)
__global__ void k_gm_init(cudaGraphConditionalHandle hout, int cond, const double* __restrict__ bb, GmDev* st,
                          double* __restrict__ hist) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const double bnorm = sqrt(*bb);
  st->bnorm = bnorm;
  st->beta = bnorm;
  st->its = 0;
  st->j = 0;
  st->restarts = 0;
  st->converged = bnorm == 0.0;
  st->rel = bnorm == 0.0 ? 0.0 : 1.0;
  if (st->cap > 0) hist[0] = bnorm == 0.0 ? 0.0 : 1.0;
  if (cond) cudaGraphSetConditional(hout, (bnorm != 0.0 && st->maxit > 0) ? 1u : 0u);
}

// cycle start: v_0 = r / beta (into V_0 and the V-cycle input), g = beta e_1
__global__ void k_gm_cycle(cudaGraphConditionalHandle hin, int cond, int64_t n, const double* __restrict__ r, GmDev* st,
                           double* __restrict__ V, double* __restrict__ vin, double* __restrict__ g,
                           double* __restrict__ vs) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = r[i] / st->beta;
    V[i] = v;
    vin[i] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x <= st->m) g[threadIdx.x] = threadIdx.x == 0 ? st->beta : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (vs) vs[0] = 1.0;  // v_0 is stored normalised
    st->j = 0;
    st->more = st->its < st->maxit;
    if (cond) cudaGraphSetConditional(hin, st->its < st->maxit ? 1u : 0u);
  }
}

// Fast mode's CGS2 with one sweep fewer: the reorthogonalisation
// coefficients h2 = V^T (w - V h1) = h1 - G h1 from the Gram matrix G = V^T V
// (its newest column comes with the first dots), so w'' = w - V (h1 + h2)
// is one sweep. Equal to CGS2 in exact arithmetic; it corrects the basis's
// loss of orthogonality, not the cancellation in forming w - V h1 (the
// parity tests bound the solve). d[0..j] = h1, d[kGmMax+1..] = G's column j;
// out: h2 (so k_gm_step's hcol = h1 + h2 is unchanged) and hsum = h1 + h2.
__global__ void k_gm_gram(const GmDev* __restrict__ st, const double* __restrict__ d, double* __restrict__ G,
                          double* __restrict__ h2, double* __restrict__ hsum) {
  __shared__ double h1s[kGmMax];
  pdl_wait();
  pdl_trigger();
  const int j = st->j, t = threadIdx.x;
  const int m1 = kGmMax + 1;
  if (t <= j) {
    h1s[t] = d[t];
    const double gk = d[kGmMax + 1 + t];
    G[t * m1 + j] = gk;
    G[j * m1 + t] = gk;
  }
  __syncthreads();
  if (t > j) return;
  double s = 0.0;
  for (int l = 0; l <= j; ++l) s = fma(G[t * m1 + l], h1s[l], s);
  const double c = h1s[t] - s;
  h2[t] = c;
  hsum[t] = h1s[t] + c;
}

// the Arnoldi step's scalar work (gmres_poly-free, oracle gmres() order):
// hcol = h1 + h2, h_{j+1,j} = |w|, previous rotations, the new rotation, g,
// the history, and the inner-loop test
__global__ void k_gm_step(cudaGraphConditionalHandle hin, int cond, GmDev* st, const double* __restrict__ h1,
                          const double* __restrict__ h2, const double* __restrict__ nrm2, double* __restrict__ H,
                          double* __restrict__ cs, double* __restrict__ sn, double* __restrict__ g,
                          double* __restrict__ hist, double* __restrict__ vs) {
  __shared__ double hcol[kGmMax + 1], c_s[kGmMax], s_s[kGmMax];
  pdl_wait();
  pdl_trigger();
  if (!st->more) return;  // a step enqueued past the end of the inner loop (host-driven loops)
  const int j = st->j, m = st->m, t = threadIdx.x;
  if (t <= j) hcol[t] = h1[t] + h2[t];  // operands staged by the warp
  if (t < j) {
    c_s[t] = cs[t];
    s_s[t] = sn[t];
  }
  __syncwarp();
  if (t != 0) return;
  const double hn = sqrt(*nrm2);
  hcol[j + 1] = hn;
  for (int k = 0; k < j; ++k) {
    const double a = c_s[k] * hcol[k] + s_s[k] * hcol[k + 1];
    hcol[k + 1] = -s_s[k] * hcol[k] + c_s[k] * hcol[k + 1];
    hcol[k] = a;
  }
  const double den = hypot(hcol[j], hcol[j + 1]);
  const double cj = den > 0.0 ? hcol[j] / den : 1.0;
  const double sj = den > 0.0 ? hcol[j + 1] / den : 0.0;
  cs[j] = cj;
  sn[j] = sj;
  hcol[j] = den;
  const double gj = g[j];
  g[j + 1] = -sj * gj;
  g[j] = cj * gj;
  for (int k = 0; k <= j; ++k) H[k + (int64_t)j * (m + 1)] = hcol[k];
  const long long its = st->its + 1;
  st->its = its;
  const double est = fabs(-sj * gj) / st->bnorm;
  if (its < st->cap) hist[its] = est;
  st->hn = hn;
  st->est = est;
  if (vs) vs[j + 1] = hn > 0.0 ? 1.0 / hn : 0.0;
  st->j = j + 1;
  const bool more = j + 1 < m && its < st->maxit && !(est <= st->rtol) && hn != 0.0;
  st->more = more;
  if (cond) cudaGraphSetConditional(hin, more ? 1u : 0u);
}

// v_{j+1} = w / h_{j+1,j} (j already advanced by k_gm_step), also the V-cycle input
__global__ void k_gm_next(int64_t n, const double* __restrict__ w, const GmDev* __restrict__ st,
                          double* __restrict__ V, double* __restrict__ vin) {
  pdl_wait();
  pdl_trigger();
  const double hn = st->hn;
  double* vj = V + (int64_t)st->j * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = hn > 0.0 ? w[i] / hn : 0.0;
    vj[i] = v;
    vin[i] = v;
  }
}

// y = H(0:j, 0:j) \ g(0:j) (back substitution, one thread)
__global__ void k_gm_ysolve(const GmDev* __restrict__ st, const double* __restrict__ H, const double* __restrict__ g,
                            double* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const int j = st->j, m = st->m;
  for (int k = j - 1; k >= 0; --k) {
    double s = g[k];
    for (int q = k + 1; q < j; ++q) s -= H[k + (int64_t)q * (m + 1)] * y[q];
    y[k] = s / H[k + (int64_t)k * (m + 1)];
  }
}

// x += Z(:, 0:j) y (element per thread; the sum in column order)
__global__ void __launch_bounds__(kGmThreads) k_gm_xupdate(int64_t n, const GmDev* __restrict__ st,
                                                           const double* __restrict__ Z,
                                                           const double* __restrict__ y, double* __restrict__ x) {
  __shared__ double ys[kGmMax];
  pdl_wait();
  pdl_trigger();
  const int j = st->j;
  if (threadIdx.x < kGmMax) ys[threadIdx.x] = (int)threadIdx.x < j ? y[threadIdx.x] : 0.0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double zk[kGmMax];
#pragma unroll
  for (int k = 0; k < kGmMax; ++k) zk[k] = k < j ? __ldg(Z + (int64_t)k * n + i) : 0.0;
  double s = x[i];
#pragma unroll
  for (int k = 0; k < kGmMax; ++k)
    if (k < j) s += ys[k] * zk[k];
  x[i] = s;
}

// end of a cycle: beta = ||b - A x||, the outer test
__global__ void k_gm_restart(cudaGraphConditionalHandle hout, int cond, GmDev* st, const double* __restrict__ rr) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const double beta = sqrt(*rr);
  st->beta = beta;
  const double rel = beta / st->bnorm;
  st->rel = rel;
  st->restarts += 1;
  const bool conv = rel <= st->rtol;
  st->converged = conv;
  if (cond) cudaGraphSetConditional(hout, (!conv && beta != 0.0 && st->its < st->maxit) ? 1u : 0u);
}


}  // namespace
}  // namespace airg
