// PMISR-DDC CF splitting on the GPU (reference: proj/src/coarsening.cpp,
// proj/src/sparse.cpp:270-340).
//
// * strength (coarsening.cpp:83-105): thread per row; off-diagonal max,
//   threshold alpha*max as one rounded multiply, |a|>0 && |a|>=threshold.
//   S is written in A's column order (sorted); |S^T| comes from exact
//   integer atomics, S^T itself is never materialised.
// * weights (coarsening.cpp:50-63): w_i = deg_i + uniform01(mix(seed,
//   0x57454947), i) with the reference splitmix64 on the global row index,
//   one rounded add -> bit-identical and partition independent.
// * PMISR (coarsening.cpp:107-160) is one-shot: the D-set test compares a
//   node with ALL its S u S^T neighbours, settled or not, and weights never
//   change, so a node that is not a strict local minimum of (w, i) in sweep
//   1 is not one in any later sweep; sweep 2 always finds D empty and
//   breaks (probe-verified). Hence F = {deg = 0} u {strict
//   local minima}, C = the rest, for every max_loops >= 1. The GPU computes
//   it with one atomic-free pass over the edges of S: each edge marks its
//   (w, i)-larger endpoint "not minimal" (idempotent byte stores).
// * DDC (coarsening.cpp:219-330): theta per F row in column order, global
//   max via atomicMax on the (non-negative) bit pattern, 1000-bin histogram
//   with shared-memory privatisation, single-thread alpha_diag scan with the
//   reference's strict '<', one-shot conversion theta > alpha && theta != 0.
#include "sparse.cuh"

#include <cooperative_groups.h>

namespace airg {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t mix(uint64_t seed, uint64_t key) {
  return splitmix64(seed ^ splitmix64(key));
}

__global__ void strength_count(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const double* __restrict__ v, double alpha,
                               int32_t* __restrict__ s_cnt, int32_t* __restrict__ st_cnt, int row_base) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = row_base + r;  // global row (rows of a slab carry global columns)
  const int s = rp[r], e = rp[r + 1];
  double off_max = 0.0;
  for (int k = s; k < e; ++k)
    if (ci[k] != i) off_max = fmax(off_max, fabs(v[k]));
  const double thr = __dmul_rn(alpha, off_max);
  int cnt = 0;
  for (int k = s; k < e; ++k) {
    const double mag = fabs(v[k]);
    const int c = ci[k];
    if (c != i && mag > 0.0 && mag >= thr) {
      ++cnt;
      atomicAdd(st_cnt + c, 1);
    }
  }
  s_cnt[r] = cnt;
}

__global__ void strength_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ v, double alpha,
                              const int32_t* __restrict__ srp, int32_t* __restrict__ sci, int row_base) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = row_base + r;
  const int s = rp[r], e = rp[r + 1];
  double off_max = 0.0;
  for (int k = s; k < e; ++k)
    if (ci[k] != i) off_max = fmax(off_max, fabs(v[k]));
  const double thr = __dmul_rn(alpha, off_max);
  int o = srp[r];
  for (int k = s; k < e; ++k) {
    const double mag = fabs(v[k]);
    const int c = ci[k];
    if (c != i && mag > 0.0 && mag >= thr) sci[o++] = c;
  }
}

__device__ __forceinline__ bool row_contains(const int32_t* __restrict__ rp,
                                             const int32_t* __restrict__ ci, int row, int key) {
  int lo = rp[row], hi = rp[row + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ci[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < rp[row + 1] && ci[lo] == key;
}

__global__ void make_weights(int n, const int32_t* __restrict__ srp, const int32_t* __restrict__ sci,
                             const int32_t* __restrict__ st_cnt, uint64_t stream_key, int mode,
                             double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t deg = (int64_t)(srp[i + 1] - srp[i]) + st_cnt[i];
  if (mode == 1) {  // |S_i u S_i^T| = |S_i| + |S_i^T| - |{j in S_i : i in S_j}|
    for (int k = srp[i]; k < srp[i + 1]; ++k)
      if (row_contains(srp, sci, sci[k], i)) --deg;
  }
  const double u = (double)(mix(stream_key, (uint64_t)i) >> 11) * 0x1.0p-53;
  w[i] = __dadd_rn((double)deg, u);
}

__device__ __forceinline__ bool weight_less(const double* w, int i, int j) {
  const double wi = w[i], wj = w[j];
  return wi != wj ? wi < wj : i < j;
}

__global__ void mark_not_minimal(int n, const int32_t* __restrict__ srp,
                                 const int32_t* __restrict__ sci, const double* __restrict__ w,
                                 uint8_t* __restrict__ notmin) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = srp[i]; k < srp[i + 1]; ++k) {
    const int j = sci[k];
    if (weight_less(w, j, i))
      notmin[i] = 1;
    else
      notmin[j] = 1;
  }
}

// F = {w < 1} u {strict local minima}; everything else C (see header).
__global__ void pmisr_labels(int n, const uint8_t* __restrict__ notmin, const double* __restrict__ w,
                             uint8_t* __restrict__ label) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  label[i] = (w[i] < 1.0 || !notmin[i]) ? AIRG_F : AIRG_C;
}

__global__ void in_degree(int n, const int32_t* __restrict__ srp, const int32_t* __restrict__ sci,
                          int32_t* __restrict__ st_cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = srp[i]; k < srp[i + 1]; ++k) atomicAdd(st_cnt + sci[k], 1);
}

// ---- label map (sparse.cpp:270-290)
__global__ void label_isf(int n, const uint8_t* __restrict__ label, int32_t* __restrict__ isf,
                          unsigned long long* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t l = label[i];
  if (l > AIRG_C) atomicMin(bad, (unsigned long long)i);
  isf[i] = l == AIRG_F;
}
__global__ void label_fill(int n, const uint8_t* __restrict__ label, const int32_t* __restrict__ fpos,
                           int32_t* __restrict__ f2s, int32_t* __restrict__ f2f,
                           int32_t* __restrict__ c2f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int fp = fpos[i];
  if (label[i] == AIRG_F) {
    f2s[i] = fp;
    f2f[fp] = i;
  } else {
    f2s[i] = i - fp;
    c2f[i - fp] = i;
  }
}

// ---- extract_blocks (sparse.cpp:292-340)
// Row slabs: local row r is global row rb + r; its F (C) sub-index is offset
// by fb (cb), the number of F (C) points before the slab. Whole matrix: 0s.
__global__ void blocks_count(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const uint8_t* __restrict__ label, const int32_t* __restrict__ f2s,
                             int32_t* __restrict__ ff, int32_t* __restrict__ fc,
                             int32_t* __restrict__ cf, int32_t* __restrict__ af, int rb, int fb, int cb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  int nF = 0, nC = 0;
  for (int k = rp[r]; k < rp[r + 1]; ++k) (label[ci[k]] == AIRG_F ? nF : nC)++;
  const int sub = f2s[i] - (label[i] == AIRG_F ? fb : cb);
  if (label[i] == AIRG_F) {
    ff[sub] = nF;
    fc[sub] = nC;
    if (af) af[sub] = nF + nC;
  } else {
    cf[sub] = nF;
  }
}
__global__ void blocks_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, const uint8_t* __restrict__ label,
                            const int32_t* __restrict__ f2s, const int32_t* __restrict__ ffrp,
                            int32_t* __restrict__ ffci, double* __restrict__ ffv,
                            const int32_t* __restrict__ fcrp, int32_t* __restrict__ fcci,
                            double* __restrict__ fcv, const int32_t* __restrict__ cfrp,
                            int32_t* __restrict__ cfci, double* __restrict__ cfv,
                            const int32_t* __restrict__ afrp, int32_t* __restrict__ afci,
                            double* __restrict__ afv, int rb, int fb, int cb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  const int sub = f2s[i] - (label[i] == AIRG_F ? fb : cb);
  if (label[i] == AIRG_F) {
    int of = ffrp[sub], oc = fcrp[sub];
    int oa = afci ? afrp[sub] : 0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const int j = ci[k];
      const bool jf = label[j] == AIRG_F;
      if (jf) {
        ffci[of] = f2s[j];
        ffv[of++] = v[k];
      } else {
        fcci[oc] = f2s[j];
        fcv[oc++] = v[k];
      }
      if (afci) {
        afci[oa] = jf ? j : (int)((unsigned)j | 0x80000000u);
        afv[oa++] = v[k];
      }
    }
  } else {
    int o = cfrp[sub];
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const int j = ci[k];
      if (label[j] == AIRG_F) {
        cfci[o] = f2s[j];
        cfv[o++] = v[k];
      }
    }
  }
}

// ---- dominance report / ddc
__global__ void theta_rows(int nf, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, double* __restrict__ theta,
                           unsigned long long* __restrict__ maxbits,
                           unsigned long long* __restrict__ bad_row, int rb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long tb = 0;
  if (i < nf) {
    double off = 0.0, diag = 0.0;
    bool seen = false;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      if (ci[k] == rb + i) {
        diag = fabs(v[k]);
        seen = true;
      } else {
        off = __dadd_rn(off, fabs(v[k]));
      }
    }
    if (!seen || diag == 0.0) {
      atomicMin(bad_row, (unsigned long long)i);
      theta[i] = 0.0;
    } else {
      const double t = __ddiv_rn(off, diag);
      theta[i] = t;
      tb = (unsigned long long)__double_as_longlong(t);
    }
  }
  block_max(maxbits, tb);
}

__global__ void theta_hist(int nf, const double* __restrict__ theta,
                           const unsigned long long* __restrict__ maxbits, int64_t bins,
                           unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int sh[];
  const bool priv = bins <= 8192;
  if (priv)
    for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const double mx = __longlong_as_double((long long)*maxbits);
  const double width = mx > 0.0 ? __ddiv_rn(mx, (double)bins) : 1.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    int64_t b = (int64_t)__ddiv_rn(theta[i], width);
    if (b > bins - 1) b = bins - 1;
    if (priv)
      atomicAdd(sh + b, 1u);
    else
      atomicAdd(hist + b, 1ull);
  }
  __syncthreads();
  if (priv)
    for (int b = threadIdx.x; b < bins; b += blockDim.x)
      if (sh[b]) atomicAdd(hist + b, (unsigned long long)sh[b]);
}

// coarsening.cpp:290-315 with n_f read from the device counter. The
// reference scans k = bins-1 .. 0, accumulating above += hist[k] and keeping
// k when |above - target| is STRICTLY smaller than the best so far (initially
// k = bins, above = 0). That is the largest k among the minimisers of
// err_k = |S_k - target| over k in [0, bins] (S_k = suffix sum, S_bins = 0):
// one block computes the suffix sums in shared memory, every thread scores
// its bins with the same rounded ops, and an (err, -k) min-reduction picks
// the winner -- identical to the serial scan, without ~bins dependent
// global loads on one thread. Falls back to the serial scan for bins > 8192.
constexpr int kSelThreads = 1024;
// one block of kSelThreads threads (the kernel below, or block 0 of the
// persistent small-level split)
__device__ __forceinline__ void ddc_select_block(const unsigned long long* __restrict__ nfp, long long nf_val,
                                                 const unsigned long long* __restrict__ hist, int64_t bins,
                                                 double fraction, const unsigned long long* __restrict__ maxbits,
                                                 int selection, double direct_alpha, double* __restrict__ out) {
  __shared__ unsigned suf[8192 + 1];  // counts <= n_f < 2^31
  __shared__ double werr[kSelThreads / 32];
  __shared__ int64_t wk[kSelThreads / 32];
  const double max_theta = __longlong_as_double((long long)__ldcg(maxbits));
  const int t = threadIdx.x;
  if (selection == 2 || max_theta == 0.0) {  // direct alpha (DdcSelection::direct) / nothing dominant
    if (t == 0) {
      out[0] = selection == 2 ? direct_alpha : 0.0;
      out[1] = max_theta;
    }
    return;
  }
  const double target = __dmul_rn(fraction, (double)(nfp ? (long long)__ldcg(nfp) : nf_val));
  if (bins > 8192) {  // serial scan
    if (t != 0) return;
    int64_t above = 0, best_k = bins;
    double best_err = fabs(__dsub_rn((double)above, target));
    for (int64_t k = bins; k-- > 0;) {
      above += (int64_t)__ldcg(hist + k);
      const double err = fabs(__dsub_rn((double)above, target));
      if (err < best_err) {
        best_err = err;
        best_k = k;
      }
    }
    out[0] = __dmul_rn((double)best_k, __ddiv_rn(max_theta, (double)bins));
    out[1] = max_theta;
    return;
  }
  const int nb = (int)bins;
  for (int k = t; k < nb; k += kSelThreads) suf[k] = (unsigned)__ldcg(hist + k);
  if (t == 0) suf[nb] = 0;
  __syncthreads();
  // suffix sums: each thread owns a contiguous chunk; serial within, scan of chunk totals
  const int chunk = (nb + kSelThreads - 1) / kSelThreads;
  const int lo = t * chunk, hi = min(nb, lo + chunk);
  unsigned acc = 0;
  for (int k = hi - 1; k >= lo; --k) acc += suf[k];
  // exclusive suffix scan of the chunk totals across the block (integers: exact)
  __shared__ unsigned wtot[kSelThreads / 32];
  const int lane = t & 31, wid = t >> 5;
  unsigned incl = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_down_sync(0xffffffffu, incl, o);
    if (lane + o < 32) incl += y;
  }
  if (lane == 0) wtot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const unsigned wv = lane < kSelThreads / 32 ? wtot[lane] : 0u;
    unsigned wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_down_sync(0xffffffffu, wi, o);
      if (lane + o < 32) wi += y;
    }
    if (lane < kSelThreads / 32) wtot[lane] = wi - wv;  // sum over later warps
  }
  __syncthreads();
  unsigned run = (incl - acc) + wtot[wid];
  for (int k = hi - 1; k >= lo; --k) {
    run += suf[k];
    suf[k] = run;  // S_k
  }
  __syncthreads();
  double best_err = INFINITY;
  int64_t best_k = -1;
  for (int k = t; k <= nb; k += kSelThreads) {
    const double err = fabs(__dsub_rn((double)(int64_t)suf[k], target));
    if (err < best_err || (err == best_err && k > best_k)) {
      best_err = err;
      best_k = k;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double e2 = __shfl_xor_sync(0xffffffffu, best_err, o);
    const int64_t k2 = __shfl_xor_sync(0xffffffffu, best_k, o);
    if (e2 < best_err || (e2 == best_err && k2 > best_k)) {
      best_err = e2;
      best_k = k2;
    }
  }
  if ((t & 31) == 0) {
    werr[t >> 5] = best_err;
    wk[t >> 5] = best_k;
  }
  __syncthreads();
  if (t < 32) {
    best_err = werr[t];
    best_k = wk[t];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double e2 = __shfl_xor_sync(0xffffffffu, best_err, o);
      const int64_t k2 = __shfl_xor_sync(0xffffffffu, best_k, o);
      if (e2 < best_err || (e2 == best_err && k2 > best_k)) {
        best_err = e2;
        best_k = k2;
      }
    }
    if (t == 0) {
      out[0] = __dmul_rn((double)best_k, __ddiv_rn(max_theta, (double)bins));
      out[1] = max_theta;
    }
  }
}

__global__ void __launch_bounds__(kSelThreads)
fcf_select(const unsigned long long* __restrict__ nfp, long long nf_val,
           const unsigned long long* __restrict__ hist, int64_t bins, double fraction,
           const unsigned long long* __restrict__ maxbits, int selection, double direct_alpha,
           double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  ddc_select_block(nfp, nf_val, hist, bins, fraction, maxbits, selection, direct_alpha, out);
}

__global__ void ddc_convert(int nf, const double* __restrict__ theta, const double* __restrict__ sel,
                            const int32_t* __restrict__ f2f, uint8_t* __restrict__ label,
                            unsigned long long* __restrict__ count) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nf) return;
  const double t = theta[k];
  if (t > sel[0] && t != 0.0) {
    label[f2f[k]] = AIRG_C;
    atomicAdd(count, 1ull);
  }
}

// ---- PMIS / PMIS-swap (coarsening.cpp:169-217; the paper's baselines) -------
// Rounds over the unassigned nodes: i joins D (-> C) when no unassigned
// S u S^T neighbour is (w, i)-larger; D's unassigned neighbours -> F. Each
// round is two passes over S's edges (every edge serves both directions)
// plus a labelling pass; the set semantics make the rounds order-free.
constexpr uint8_t kUnassigned = 2;
__global__ void pmis_marks(int n, const int32_t* __restrict__ srp, const int32_t* __restrict__ sci,
                           const double* __restrict__ w, const uint8_t* __restrict__ label,
                           uint8_t* __restrict__ notmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || label[i] != kUnassigned) return;
  for (int k = srp[i]; k < srp[i + 1]; ++k) {
    const int j = sci[k];
    if (label[j] != kUnassigned) continue;
    if (weight_less(w, i, j))
      notmax[i] = 1;
    else
      notmax[j] = 1;
  }
}
__global__ void pmis_select(int n, const uint8_t* __restrict__ notmax, uint8_t* __restrict__ label,
                            uint8_t* __restrict__ in_d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool d = label[i] == kUnassigned && !notmax[i];
  in_d[i] = d;
  if (d) label[i] = AIRG_C;
}
__global__ void pmis_neighbours(int n, const int32_t* __restrict__ srp, const int32_t* __restrict__ sci,
                                const uint8_t* __restrict__ in_d, uint8_t* __restrict__ label) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool di = in_d[i];
  for (int k = srp[i]; k < srp[i + 1]; ++k) {
    const int j = sci[k];
    if (di && label[j] == kUnassigned) label[j] = AIRG_F;
    if (in_d[j] && label[i] == kUnassigned) label[i] = AIRG_F;
  }
}
__global__ void pmis_count(int n, const uint8_t* __restrict__ label, unsigned long long* __restrict__ cnt,
                           int swap, uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool u = false;
  if (i < n) {
    u = label[i] == kUnassigned;
    if (out) out[i] = swap ? (label[i] == AIRG_C ? AIRG_F : AIRG_C) : label[i];
  }
  block_add(cnt, u ? 1ull : 0ull);
}

}  // namespace

void strength(Ctx& c, const Csr& a, double alpha, Strength& g, int row_base) {
  if (row_base == 0 && a.n != a.m) throw InvalidArgument("strength: matrix must be square");
  g.n = a.n;
  DBuf<int32_t> s_cnt(c, (size_t)a.n);
  g.st_cnt.alloc(c, (size_t)std::max(a.n, a.m));
  g.st_cnt.zero(c);
  g.rp.alloc(c, (size_t)a.n + 1);
  if (a.n)
    LAUNCH(c, strength_count, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, a.v.p, alpha,
           s_cnt.p, g.st_cnt.p, row_base);
  g.nnz = exclusive_scan(c, s_cnt.p, g.rp.p, a.n);
  g.ci.alloc(c, (size_t)g.nnz);
  if (a.n)
    LAUNCH(c, strength_fill, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, a.v.p, alpha,
           g.rp.p, g.ci.p, row_base);
}

void pmisr(Ctx& c, const Strength& g, int64_t max_loops, uint64_t seed, int weight_mode,
           uint8_t* d_labels, double* d_weights) {
  if (max_loops < 1) throw InvalidArgument("pmisr: max_loops must be >= 1");
  const int n = g.n;
  if (n == 0) return;
  DBuf<double> wbuf;
  double* w = d_weights;
  if (!w) {
    wbuf.alloc(c, (size_t)n);
    w = wbuf.p;
  }
  const uint64_t key = splitmix64_host(seed ^ splitmix64_host(0x57454947ull));
  LAUNCH(c, make_weights, blocks_for(n, 256), 256, 0, n, g.rp.p, g.ci.p, g.st_cnt.p, key,
         weight_mode, w);
  pmisr_with_weights(c, g, max_loops, w, d_labels);
}

void pmis(Ctx& c, const Strength& g, bool swap, uint64_t seed, uint8_t* d_labels) {
  const int n = g.n;
  if (n == 0) return;
  DBuf<double> w(c, (size_t)n);
  const uint64_t key = splitmix64_host(seed ^ splitmix64_host(0x57454947ull));
  LAUNCH(c, make_weights, blocks_for(n, 256), 256, 0, n, g.rp.p, g.ci.p, g.st_cnt.p, key, 0, w.p);
  DBuf<uint8_t> label(c, (size_t)n), notmax(c, (size_t)n), in_d(c, (size_t)n);
  DBuf<unsigned long long> cnt(c, 1);
  CUDA_CHECK(cudaMemsetAsync(label.p, kUnassigned, n, c.stream));
  for (int64_t round = 0;; ++round) {
    if (round > n) throw RuntimeError("pmis: no progress");
    notmax.zero(c);
    LAUNCH(c, pmis_marks, blocks_for(n, 256), 256, 0, n, g.rp.p, g.ci.p, w.p, label.p, notmax.p);
    LAUNCH(c, pmis_select, blocks_for(n, 256), 256, 0, n, notmax.p, label.p, in_d.p);
    LAUNCH(c, pmis_neighbours, blocks_for(n, 256), 256, 0, n, g.rp.p, g.ci.p, in_d.p, label.p);
    cnt.zero(c);
    LAUNCH(c, pmis_count, blocks_for(n, 256), 256, 0, n, label.p, cnt.p, 0, (uint8_t*)nullptr);
    if (read1(c, cnt.p) == 0) break;
  }
  cnt.zero(c);
  LAUNCH(c, pmis_count, blocks_for(n, 256), 256, 0, n, label.p, cnt.p, swap ? 1 : 0, d_labels);
}

void pmisr_with_weights(Ctx& c, const Strength& g, int64_t max_loops, const double* w,
                        uint8_t* d_labels) {
  if (max_loops < 1) throw InvalidArgument("pmisr: max_loops must be >= 1");
  const int n = g.n;
  if (n == 0) return;
  DBuf<uint8_t> notmin(c, (size_t)n);
  notmin.zero(c);
  LAUNCH(c, mark_not_minimal, blocks_for(n, 256), 256, 0, n, g.rp.p, g.ci.p, w, notmin.p);
  LAUNCH(c, pmisr_labels, blocks_for(n, 256), 256, 0, n, notmin.p, w, d_labels);
}

void strength_from_pattern(Ctx& c, const Csr& s, Strength& g) {
  if (s.n != s.m) throw InvalidArgument("StrengthGraph: pattern must be square");
  g.n = s.n;
  g.nnz = s.nnz;
  g.rp.alloc(c, (size_t)s.n + 1);
  g.ci.alloc(c, (size_t)s.nnz);
  CUDA_CHECK(cudaMemcpyAsync(g.rp.p, s.rp.p, sizeof(int32_t) * (s.n + 1), cudaMemcpyDeviceToDevice, c.stream));
  if (s.nnz) CUDA_CHECK(cudaMemcpyAsync(g.ci.p, s.ci.p, sizeof(int32_t) * s.nnz, cudaMemcpyDeviceToDevice, c.stream));
  g.st_cnt.alloc(c, (size_t)s.n);
  g.st_cnt.zero(c);
  if (s.n) LAUNCH(c, in_degree, blocks_for(s.n, 256), 256, 0, s.n, g.rp.p, g.ci.p, g.st_cnt.p);
}

void build_label_map(Ctx& c, const uint8_t* d_labels, int32_t n, LabelMap& map) {
  map.n = n;
  map.label.alloc(c, (size_t)n);
  if (n) CUDA_CHECK(cudaMemcpyAsync(map.label.p, d_labels, n, cudaMemcpyDeviceToDevice, c.stream));
  DBuf<int32_t> isf(c, (size_t)n), fpos(c, (size_t)n + 1);
  DBuf<unsigned long long> bad(c, 1);
  CUDA_CHECK(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), c.stream));
  if (n) LAUNCH(c, label_isf, blocks_for(n, 256), 256, 0, n, d_labels, isf.p, bad.p);
  const int64_t nf = exclusive_scan(c, isf.p, fpos.p, n);
  const unsigned long long b = read1(c, bad.p);
  if (b != ~0ull)
    throw InvalidArgument("build_label_map: unassigned label at row " + std::to_string(b));
  map.nf = (int32_t)nf;
  map.nc = (int32_t)(n - nf);
  map.fine_to_sub.alloc(c, (size_t)n);
  map.f_to_fine.alloc(c, (size_t)map.nf);
  map.c_to_fine.alloc(c, (size_t)map.nc);
  if (n)
    LAUNCH(c, label_fill, blocks_for(n, 256), 256, 0, n, d_labels, fpos.p, map.fine_to_sub.p,
           map.f_to_fine.p, map.c_to_fine.p);
}

void extract_blocks(Ctx& c, const Csr& a, const LabelMap& map, Blocks& out, bool want_af) {
  if (a.n != a.m || a.n != map.n) throw InvalidArgument("extract_blocks: label length mismatch");
  extract_block_rows(c, a, 0, map, 0, map.nf, 0, map.nc, out, want_af);
}

// Rows [rb, rb + a.n) of the operator (global columns, global map): the F
// rows of the slab are F sub-indices [fb, fe), its C rows [cb, ce); block
// columns stay global sub-indices (af: global fine columns).
void extract_block_rows(Ctx& c, const Csr& a, int rb, const LabelMap& map, int fb, int fe, int cb, int ce,
                        Blocks& out, bool want_af) {
  const int n = a.n, nf = fe - fb, nc = ce - cb;
  DBuf<int32_t> ffc(c, (size_t)nf), fcc(c, (size_t)nf), cfc(c, (size_t)nc), afc(c, want_af ? (size_t)nf : 0);
  if (n)
    LAUNCH(c, blocks_count, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, map.label.p,
           map.fine_to_sub.p, ffc.p, fcc.p, cfc.p, want_af ? afc.p : nullptr, rb, fb, cb);
  auto finish = [&](Csr& m, int rows, int cols, const int32_t* cnt) {
    m.n = rows;
    m.m = cols;
    m.rp.alloc(c, (size_t)rows + 1);
    m.nnz = exclusive_scan(c, cnt, m.rp.p, rows);
    m.ci.alloc(c, (size_t)m.nnz);
    m.v.alloc(c, (size_t)m.nnz);
  };
  finish(out.aff, nf, map.nf, ffc.p);
  finish(out.afc, nf, map.nc, fcc.p);
  finish(out.acf, nc, map.nf, cfc.p);
  if (want_af) finish(out.af, nf, map.n, afc.p);
  if (n)
    LAUNCH(c, blocks_fill, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, a.v.p, map.label.p,
           map.fine_to_sub.p, out.aff.rp.p, out.aff.ci.p, out.aff.v.p, out.afc.rp.p, out.afc.ci.p,
           out.afc.v.p, out.acf.rp.p, out.acf.ci.p, out.acf.v.p,
           want_af ? out.af.rp.p : nullptr, want_af ? out.af.ci.p : nullptr,
           want_af ? out.af.v.p : nullptr, rb, fb, cb);
}

namespace {
struct ThetaScratch {
  DBuf<double> theta;
  DBuf<unsigned long long> u;  // [0] max bits, [1] bad row, [2] converted
};
void theta_pass(Ctx& c, const Csr& aff, ThetaScratch& s, int rb = 0) {
  s.theta.alloc(c, (size_t)aff.n);
  s.u.alloc(c, 3);
  const unsigned long long init[3] = {0ull, ~0ull, 0ull};
  to_device(c, s.u.p, init, 3);
  if (aff.n)
    LAUNCH(c, theta_rows, blocks_for(aff.n, 256), 256, 0, aff.n, aff.rp.p, aff.ci.p, aff.v.p,
           s.theta.p, s.u.p, s.u.p + 1, rb);
}
// histogram of one 8-bit digit of the theta bit patterns (theta >= 0: the
// bit order is the value order) among the values whose higher digits match
__global__ void theta_digit_hist(int n, const double* __restrict__ theta, unsigned long long prefix,
                                 unsigned long long mask, int shift, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(theta[i]);
    if ((bits & mask) == prefix) atomicAdd(&sh[(bits >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, sh[b]);
}
// the k-th smallest theta (0-based) by an 8-pass radix select over the bits
double theta_kth(Ctx& c, const double* theta, int n, int64_t k) {
  DBuf<unsigned> hist(c, 256);
  unsigned long long prefix = 0, mask = 0;
  const int blocks = (int)std::min<int64_t>(blocks_for(n, 256), 4 * c.num_sms);
  for (int shift = 56; shift >= 0; shift -= 8) {
    hist.zero(c);
    LAUNCH(c, theta_digit_hist, blocks, 256, 0, n, theta, prefix, mask, shift, hist.p);
    unsigned h[256];
    to_host(c, h, hist.p, 256);
    int d = 0;
    for (; d < 255 && (int64_t)h[d] <= k; ++d) k -= h[d];
    prefix |= (unsigned long long)d << shift;
    mask |= 255ull << shift;
  }
  double v;
  memcpy(&v, &prefix, sizeof v);
  return v;
}

void throw_zero_diag(unsigned long long row) {
  throw RuntimeError("dominance_report: zero diagonal in A_ff row " + std::to_string(row));
}
}  // namespace

DdcResult ddc(Ctx& c, const Csr& aff, const LabelMap& map, uint8_t* d_labels, double fraction,
              int64_t bins, int selection, double direct_alpha, bool convert) {
  if (aff.n != map.nf) throw InvalidArgument("ddc: a_ff does not match label map");
  if (fraction <= 0.0 || fraction > 1.0) throw InvalidArgument("ddc: fraction must be in (0, 1]");
  if (bins < 1) throw InvalidArgument("dominance_report: bins >= 1");
  ThetaScratch s;
  theta_pass(c, aff, s);
  if (selection == 1) {
    // exact order statistic (coarsening.cpp:270-288): the value with
    // round(fraction * n_F) rows strictly above it, by a radix select
    const int nf = aff.n;
    unsigned long long u0[3];
    to_host(c, u0, s.u.p, 3);
    if (u0[1] != ~0ull) throw_zero_diag(u0[1]);
    double mx;
    memcpy(&mx, &u0[0], sizeof mx);
    int64_t target = (int64_t)std::llround(fraction * (double)nf);
    target = std::min<int64_t>(std::max<int64_t>(target, 0), nf);
    double a;
    if (target == 0 || mx == 0.0)
      a = mx;
    else if (target == nf)
      a = -1.0;
    else
      a = theta_kth(c, s.theta.p, nf, nf - target - 1);
    selection = 2;  // then the direct path with the selected value
    direct_alpha = a;
  }
  DBuf<unsigned long long> hist(c, (size_t)bins);
  hist.zero(c);
  DBuf<double> sel(c, 2);
  const int nf = aff.n;
  if (nf) {
    const int blocks = (int)std::min<int64_t>(blocks_for(nf, 256), 4 * c.num_sms);
    const size_t smem = bins <= 8192 ? (size_t)bins * sizeof(unsigned) : 0;
    LAUNCH(c, theta_hist, blocks, 256, smem, nf, s.theta.p, s.u.p, bins, hist.p);
  }
  LAUNCH(c, fcf_select, 1, kSelThreads, 0, (const unsigned long long*)nullptr, (long long)nf, hist.p, bins,
         fraction, s.u.p, selection, direct_alpha, sel.p);
  if (convert && nf)
    LAUNCH(c, ddc_convert, blocks_for(nf, 256), 256, 0, nf, s.theta.p, sel.p, map.f_to_fine.p,
           d_labels, s.u.p + 2);
  unsigned long long u[3];
  double sv[2];
  to_host(c, u, s.u.p, 3);
  to_host(c, sv, sel.p, 2);
  if (u[1] != ~0ull) throw_zero_diag(u[1]);
  DdcResult r;
  r.converted = (int64_t)u[2];
  r.alpha_diag = sv[0];
  r.max_theta = sv[1];
  return r;
}

// dominance_report (coarsening.cpp:219-250): theta per F row, max, and the
// bins-bin histogram over [0, max] (width max/bins, 1 when max == 0)
double dominance_report(Ctx& c, const Csr& aff, int64_t bins, double* d_theta, int64_t* h_hist) {
  if (bins < 1) throw InvalidArgument("dominance_report: bins >= 1");
  ThetaScratch s;
  theta_pass(c, aff, s);
  const int nf = aff.n;
  DBuf<unsigned long long> hist(c, (size_t)bins);
  hist.zero(c);
  if (nf) {
    const int blocks = (int)std::min<int64_t>(blocks_for(nf, 256), 4 * c.num_sms);
    const size_t smem = bins <= 8192 ? (size_t)bins * sizeof(unsigned) : 0;
    LAUNCH(c, theta_hist, blocks, 256, smem, nf, s.theta.p, s.u.p, bins, hist.p);
    if (d_theta)
      CUDA_CHECK(cudaMemcpyAsync(d_theta, s.theta.p, sizeof(double) * nf, cudaMemcpyDeviceToDevice, c.stream));
  }
  unsigned long long u[3];
  to_host(c, u, s.u.p, 3);
  if (u[1] != ~0ull) throw_zero_diag(u[1]);
  if (h_hist) {
    std::vector<unsigned long long> hh((size_t)bins);
    to_host(c, hh.data(), hist.p, hh.size());
    for (int64_t b = 0; b < bins; ++b) h_hist[b] = (int64_t)hh[(size_t)b];
  }
  double mx;
  memcpy(&mx, &u[0], sizeof mx);
  return mx;
}

double dominance_max(Ctx& c, const Csr& aff, int rb) {
  ThetaScratch s;
  theta_pass(c, aff, s, rb);
  unsigned long long u[3];
  to_host(c, u, s.u.p, 3);
  if (u[1] != ~0ull) throw_zero_diag(u[1]);
  double mx;
  memcpy(&mx, &u[0], sizeof mx);
  return mx;
}

// ---- fused, sync-free CF split (airg_cf_split, the CF-split metric) -------------
// The labels need neither S nor A_ff as matrices: strength is a per-row
// threshold (thr_i = alpha * off_max_i) that any later pass re-applies to A's
// entries, and theta of an F row is its A row restricted to F columns in
// column order -- exactly A_ff's row, since extract_blocks keeps the order.
// So the split is seven passes over A with no scans, no allocations sized by
// a count, and no host synchronisation until the single report readback:
//   rows (thr, |S_i|, |S^T| atomics) -> weights -> not-minimal marks ->
//   labels -> theta (+max) -> histogram -> alpha (1 thread) -> convert.
// Same arithmetic as the kernels above, so the same labels bit for bit.
namespace {

// build knob: AIRG_CF_UNROLL = unroll of the 16-byte row loop
#ifndef AIRG_CF_UNROLL
#define AIRG_CF_UNROLL 1
#endif
constexpr int kCfUnroll = AIRG_CF_UNROLL;
#ifndef AIRG_CF_PIPE
#define AIRG_CF_PIPE 1
#endif
#if AIRG_CF_PIPE
#define CF_RESTRICT __restrict__
#else
#define CF_RESTRICT
#endif

// Visit the entries k = s..e-1 of one row in order, f(ci[k], v[k]). VEC:
// the aligned body as 16-byte loads (4 column indices, 2 x 2 values) --
// fewer, wider loads per thread for long rows; same order, same results.
template <bool VEC, class F>
__device__ __forceinline__ void for_row(const int32_t* __restrict__ ci, const double* __restrict__ v, int s,
                                        int e, F&& f) {
  int k = s;
  if (VEC && AIRG_CF_PIPE) {
    // software-pipelined: group k+4's loads are issued before group k is used
    for (; k < e && (k & 3); ++k) f(__ldg(ci + k), __ldg(v + k));
    if (k + 4 <= e) {
      int4 c = __ldg(reinterpret_cast<const int4*>(ci + k));
      double2 a = __ldg(reinterpret_cast<const double2*>(v + k));
      double2 b = __ldg(reinterpret_cast<const double2*>(v + k + 2));
      for (; k + 4 <= e; k += 4) {
        int4 cn = c;
        double2 an = a, bn = b;
        if (k + 8 <= e) {
          cn = __ldg(reinterpret_cast<const int4*>(ci + k + 4));
          an = __ldg(reinterpret_cast<const double2*>(v + k + 4));
          bn = __ldg(reinterpret_cast<const double2*>(v + k + 6));
        }
        f(c.x, a.x);
        f(c.y, a.y);
        f(c.z, b.x);
        f(c.w, b.y);
        c = cn;
        a = an;
        b = bn;
      }
    }
  } else if (VEC) {
    for (; k < e && (k & 3); ++k) f(__ldg(ci + k), __ldg(v + k));
#pragma unroll (kCfUnroll)
    for (; k + 4 <= e; k += 4) {
      const int4 c = __ldg(reinterpret_cast<const int4*>(ci + k));
      const double2 a = __ldg(reinterpret_cast<const double2*>(v + k));
      const double2 b = __ldg(reinterpret_cast<const double2*>(v + k + 2));
      f(c.x, a.x);
      f(c.y, a.y);
      f(c.z, b.x);
      f(c.w, b.y);
    }
  }
  for (; k < e; ++k) f(__ldg(ci + k), __ldg(v + k));
}

// long rows (mean >= AIRG_CF_VEC, default 6) take the 16-byte path
int cf_vec_rows() {
  static const int v = [] {
    const char* e = getenv("AIRG_CF_VEC");
    return e ? atoi(e) : 6;
  }();
  return v;
}


// Labels without a label pass: a row with no strong connection (weight < 1)
// is never marked "not minimal", so the PMISR label is F exactly when
// notmin == 0 -- the mark array IS the pre-DDC label array.

// Loads of data written earlier in the same launch (the persistent
// small-level split) bypass L1: COH = true -> ld.global.cg.
template <bool COH, class T>
__device__ __forceinline__ T ldc(const T* p) {
  if constexpr (COH)
    return __ldcg(p);
  else
    return *p;
}

template <bool COH>
__device__ __forceinline__ double fcf_weight_c(const int2* cnt, uint64_t key, int j) {
  const int2 c = ldc<COH>(cnt + j);
  const double u = (double)(mix(key, (uint64_t)j) >> 11) * 0x1.0p-53;
  return __dadd_rn((double)((int64_t)c.x + c.y), u);
}

// ---- one row of each pass (thread per row) ----
// strength: thr_i = alpha * max off-diagonal |a_ij|, |S_i|, |S^T| atomics
template <bool VEC>
__device__ __forceinline__ int fcf_row_strength(int i, const int32_t* __restrict__ rp,
                                                const int32_t* __restrict__ ci, const double* __restrict__ v,
                                                double alpha, double* thr, int2* cnt) {
  const int s = rp[i], e = rp[i + 1];
  double off_max = 0.0;
  for_row<VEC>(ci, v, s, e, [&](int c, double x) {
    if (c != i) off_max = fmax(off_max, fabs(x));
  });
  const double t = __dmul_rn(alpha, off_max);
  thr[i] = t;
  int c_i = 0;
  for_row<VEC>(ci, v, s, e, [&](int c, double x) {
    const double mag = fabs(x);
    if (c != i && mag > 0.0 && mag >= t) {
      ++c_i;
      atomicAdd(&cnt[c].y, 1);
    }
  });
  cnt[i].x = c_i;
  return c_i;
}

// not-minimal marks over the strong entries of row i
template <bool VEC, bool COH>
__device__ __forceinline__ void fcf_row_marks(int i, const int32_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci, const double* __restrict__ v,
                                              const double* thr, const int2* CF_RESTRICT cnt, uint64_t key,
                                              uint8_t* CF_RESTRICT notmin) {
  const double t = ldc<COH>(thr + i);
  const double wi = fcf_weight_c<COH>(cnt, key, i);
  bool mine = false;
  for_row<VEC>(ci, v, rp[i], rp[i + 1], [&](int j, double x) {
    const double mag = fabs(x);
    if (j == i || !(mag > 0.0) || !(mag >= t)) return;
    const double wj = fcf_weight_c<COH>(cnt, key, j);
    if (wj != wi ? wj < wi : j < i)  // weight_less(w, j, i)
      mine = true;
    else
      notmin[j] = 1;
  });
  if (mine) notmin[i] = 1;
}

// theta of F row i (its A_ff row); returns the bits for the max
template <bool VEC, bool COH>
__device__ __forceinline__ unsigned long long fcf_row_theta(int i, const int32_t* __restrict__ rp,
                                                            const int32_t* __restrict__ ci,
                                                            const double* __restrict__ v, const uint8_t* notmin,
                                                            double* theta, unsigned long long* bad_row) {
  double off = 0.0, diag = 0.0;
  bool seen = false;
  for_row<VEC>(ci, v, rp[i], rp[i + 1], [&](int j, double x) {
    if (ldc<COH>(notmin + j)) return;
    if (j == i) {
      diag = fabs(x);
      seen = true;
    } else {
      off = __dadd_rn(off, fabs(x));
    }
  });
  if (!seen || diag == 0.0) {
    atomicMax(bad_row, ~(unsigned long long)i);  // ~i: the max is the first bad row
    theta[i] = 0.0;
    return 0;
  }
  const double t = __ddiv_rn(off, diag);
  theta[i] = t;
  return (unsigned long long)__double_as_longlong(t);  // t >= 0: bit order = value order
}

template <bool VEC>
__global__ void fcf_rows(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                         const double* __restrict__ v, double alpha, double* __restrict__ thr,
                         int2* __restrict__ cnt, unsigned long long* __restrict__ s_total) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int c_i = i < n ? fcf_row_strength<VEC>(i, rp, ci, v, alpha, thr, cnt) : 0;
  block_add(s_total, (unsigned long long)c_i);
}

template <bool VEC>
__global__ void fcf_marks(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, const double* __restrict__ thr,
                          const int2* __restrict__ cnt, uint64_t key, uint8_t* __restrict__ notmin) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) fcf_row_marks<VEC, false>(i, rp, ci, v, thr, cnt, key, notmin);
}

// theta of an F row over A's F columns in column order (= its A_ff row);
// also the optional copy of the PMISR labels
template <bool VEC>
__global__ void fcf_theta(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, const uint8_t* __restrict__ notmin,
                          double* __restrict__ theta, uint8_t* __restrict__ label_pre,
                          unsigned long long* __restrict__ maxbits, unsigned long long* __restrict__ bad_row) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long tb = 0;
  const bool fr = i < n && !notmin[i];
  if (label_pre && i < n) label_pre[i] = fr ? AIRG_F : AIRG_C;
  if (fr) tb = fcf_row_theta<VEC, false>(i, rp, ci, v, notmin, theta, bad_row);
  block_max(maxbits, tb);
}

constexpr unsigned kFull = 0xffffffffu;

// ---- the order-free passes with G lanes per row (long rows) ----
// Strength (max, counts, S^T atomics) and the not-minimal marks do not
// depend on the order a row is visited in (max and counts are exact; the
// marks are idempotent stores), so G lanes take a row's entries k = s+lane,
// s+lane+G, ... with coalesced loads and combine by shuffles: the same
// thresholds, counts and marks as the thread-per-row passes, bit for bit.
// theta (an ordered sum) stays thread-per-row.
template <int G>
__global__ void fcf_rows_lanes(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const double* __restrict__ v, double alpha, double* __restrict__ thr,
                               int2* __restrict__ cnt, unsigned long long* __restrict__ s_total) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = t / G, lane = t & (G - 1);
  const bool live = i < n;
  int s = 0, e = 0;
  double off_max = 0.0;
  if (live) {
    s = __ldg(rp + i);
    e = __ldg(rp + i + 1);
    for (int k = s + lane; k < e; k += G)
      if (__ldg(ci + k) != i) off_max = fmax(off_max, fabs(__ldg(v + k)));
  }
  pdl_wait();
  pdl_trigger();
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) off_max = fmax(off_max, __shfl_xor_sync(kFull, off_max, o, G));
  const double tr = __dmul_rn(alpha, off_max);
  int c_i = 0;
  if (live) {
    for (int k = s + lane; k < e; k += G) {
      const int c = __ldg(ci + k);
      const double mag = fabs(__ldg(v + k));
      if (c != i && mag > 0.0 && mag >= tr) {
        ++c_i;
        atomicAdd(&cnt[c].y, 1);
      }
    }
  }
  int tot = c_i;
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o, G);
  if (live && lane == 0) {
    thr[i] = tr;
    cnt[i].x = tot;
  }
  block_add(s_total, (unsigned long long)c_i);
}

template <int G>
__global__ void fcf_marks_lanes(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, const double* __restrict__ thr,
                                const int2* __restrict__ cnt, uint64_t key, uint8_t* __restrict__ notmin) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = t / G, lane = t & (G - 1);
  const bool live = i < n;
  int s = 0, e = 0;
  if (live) {
    s = __ldg(rp + i);
    e = __ldg(rp + i + 1);
  }
  pdl_wait();
  pdl_trigger();
  bool mine = false;
  if (live) {
    const double tr = thr[i];
    const double wi = fcf_weight_c<false>(cnt, key, i);
    for (int k = s + lane; k < e; k += G) {
      const int j = __ldg(ci + k);
      const double mag = fabs(__ldg(v + k));
      if (j == i || !(mag > 0.0) || !(mag >= tr)) continue;
      const double wj = fcf_weight_c<false>(cnt, key, j);
      if (wj != wi ? wj < wi : j < i)  // weight_less(w, j, i)
        mine = true;
      else
        notmin[j] = 1;
    }
  }
  const unsigned any = __ballot_sync(kFull, mine);
  const unsigned grp = (G == 32 ? kFull : ((1u << G) - 1u)) << ((threadIdx.x & 31) & ~(G - 1));
  if (live && lane == 0 && (any & grp)) notmin[i] = 1;
}

// zero a level's scratch (counters, histogram, counts, marks) as a kernel, so
// it joins the PDL chain (a memset node would break it); waits for the
// previous split that used the same scratch
__global__ void fcf_zero(unsigned long long* __restrict__ w, int64_t words, unsigned long long* __restrict__ u8) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t k = t; k < words; k += (int64_t)gridDim.x * blockDim.x) w[k] = 0ull;
  if (u8 && t < 8) u8[t] = 0ull;
}

// lanes per row of the order-free passes: the fewest lanes (a power of two)
// with about 4 entries each, at most 4 (1 = the thread-per-row passes).
// Measured on all levels back to back: C2 2.53 -> 2.32 ms, C4 1.37 -> 1.25
// ms; caps of 2 / 16 lanes: C2 2.50 / 2.63, C4 1.32 / 1.24 ms.
int cf_lanes(int64_t n, int64_t nnz) {
  if (n <= 0) return 1;
  const double mean = (double)nnz / (double)n;
  int g = 1;
  while (g < 4 && mean > 4.0 * g) g *= 2;
  return g;
}


__global__ void fcf_labels(int n, const uint8_t* __restrict__ notmin, uint8_t* __restrict__ label,
                           unsigned long long* __restrict__ nf) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool f = false;
  if (i < n) {
    f = !notmin[i];
    label[i] = f ? AIRG_F : AIRG_C;
  }
  block_add(nf, f ? 1ull : 0ull);
}

// histogram of theta over the F rows (coarsening.cpp:290-315) and the F
// count. Rows of equal theta are common (structured operators), so lanes
// of a warp that hit the same bin add once (match + popc) instead of
// serialising on one shared-memory address.
__global__ void fcf_hist(int n, const uint8_t* __restrict__ notmin, const double* __restrict__ theta,
                         const unsigned long long* __restrict__ maxbits, int64_t bins,
                         unsigned long long* __restrict__ hist, unsigned long long* __restrict__ nf) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ unsigned int sh[];
  const bool priv = bins <= 8192;
  if (priv)
    for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const double mx = __longlong_as_double((long long)*maxbits);
  const double width = mx > 0.0 ? __ddiv_rn(mx, (double)bins) : 1.0;
  const int lane = threadIdx.x & 31;
  unsigned long long cnt = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {  // uniform trip count
    const int64_t i = base + threadIdx.x;
    long long b = -1;
    if (i < n && !notmin[i]) {
      b = (long long)__ddiv_rn(theta[i], width);
      if (b > bins - 1) b = bins - 1;
      ++cnt;
    }
    const unsigned peers = __match_any_sync(kFull, b);
    if (b >= 0 && lane == __ffs(peers) - 1) {
      if (priv)
        atomicAdd(sh + b, (unsigned)__popc(peers));
      else
        atomicAdd(hist + b, (unsigned long long)__popc(peers));
    }
  }
  block_add(nf, cnt);
  if (priv)
    for (int b = threadIdx.x; b < bins; b += blockDim.x)
      if (sh[b]) atomicAdd(hist + b, (unsigned long long)sh[b]);
}

// the one-shot conversion (coarsening.cpp:322-328) writing the final labels
// (the PMISR labels when a row had a zero diagonal: the split then fails)
__global__ void fcf_convert(int n, const uint8_t* __restrict__ notmin, const double* __restrict__ theta,
                            const double* __restrict__ sel, const unsigned long long* __restrict__ bad_row,
                            uint8_t* __restrict__ label, unsigned long long* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool conv = false;
  if (i < n) {
    const bool f = !notmin[i];
    if (f && *bad_row == 0) {
      const double t = theta[i];
      conv = t > sel[0] && t != 0.0;
    }
    label[i] = f && !conv ? AIRG_F : AIRG_C;
  }
  block_add(count, conv ? 1ull : 0ull);
}

// alpha_diag and the conversion in ONE launch: every CTA (<= one per SM)
// runs the selection block on the histogram (8 KB from L2 each) into shared
// memory -- the same value in every CTA -- and converts its grid-stride share
// of the rows; CTA 0 also writes alpha_diag / max theta for the report.
__global__ void __launch_bounds__(kSelThreads)
fcf_select_convert(int n, const unsigned long long* __restrict__ nfp, const unsigned long long* __restrict__ hist,
                   int64_t bins, double fraction, const unsigned long long* __restrict__ maxbits,
                   double* __restrict__ sel_out, const uint8_t* __restrict__ notmin,
                   const double* __restrict__ theta, const unsigned long long* __restrict__ bad_row,
                   uint8_t* __restrict__ label, unsigned long long* __restrict__ count) {
  __shared__ double ssel[2];
  pdl_wait();
  pdl_trigger();
  ddc_select_block(nfp, 0, hist, bins, fraction, maxbits, 0, 0.0, ssel);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < 2) sel_out[threadIdx.x] = ssel[threadIdx.x];
  const double sel = ssel[0];
  const bool ok = *bad_row == 0;
  unsigned long long conv = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool f = !notmin[i];
    bool c = false;
    if (f && ok) {
      const double t = theta[i];
      c = t > sel && t != 0.0;
    }
    label[i] = f && !c ? AIRG_F : AIRG_C;
    conv += c;
  }
  block_add(count, conv);
}

}  // namespace

void launch_ddc_select(Ctx& c, const unsigned long long* d_nf, const unsigned long long* d_hist, int64_t bins,
                       double fraction, const unsigned long long* d_maxbits, double* d_out) {
  LAUNCH(c, fcf_select, 1, kSelThreads, 0, d_nf, 0ll, d_hist, bins, fraction, d_maxbits, 0, 0.0, d_out);
}

size_t cf_split_zero_bytes(int64_t n, bool ddc_enabled, int64_t bins) {
  const size_t nb = ddc_enabled ? (size_t)bins : 0;
  const size_t zero_bytes = (8 + nb) * 8 + (size_t)n * 8 + (size_t)n;
  return (zero_bytes + 15) & ~(size_t)15;
}

const unsigned long long* cf_split_fused_enqueue(Ctx& c, const Csr& a, double alpha, uint64_t seed,
                                                 bool ddc_enabled, double fraction, int64_t bins,
                                                 uint8_t* d_labels, uint8_t* d_labels_pre,
                                                 unsigned long long* d_u_out, void* d_zeroed) {
  if (a.n != a.m) throw InvalidArgument("strength: matrix must be square");
  if (ddc_enabled && (fraction <= 0.0 || fraction > 1.0))
    throw InvalidArgument("ddc: fraction must be in (0, 1]");
  if (ddc_enabled && bins < 1) throw InvalidArgument("dominance_report: bins >= 1");
  const int n = a.n;
  if (n == 0) {
    if (d_u_out) CUDA_CHECK(cudaMemsetAsync(d_u_out, 0, 8 * sizeof(unsigned long long), c.stream));
    return d_u_out;
  }
  const unsigned g = blocks_for(n, 256);
  // one scratch block, zeroed by ONE memset up to notmin:
  //   [u: 8 x u64 | hist: bins x u64 | cnt: n x {|S_i|, |S^T_i|} | notmin: n bytes | pad]
  //   [thr: n doubles | theta: n doubles]
  const size_t nb = ddc_enabled ? (size_t)bins : 0;
  const size_t zero_bytes = (8 + nb) * 8 + (size_t)n * 8 + (size_t)n;
  const size_t head = (zero_bytes + 15) & ~(size_t)15;
  const bool prezeroed = d_zeroed && d_u_out;
  // the zeroed part in the caller's region, else at the front of the scratch
  const size_t bytes = (prezeroed ? 0 : head) + 2 * (size_t)n * 8;
  uint8_t* sbase = static_cast<uint8_t*>(ctx_scratch(c, bytes));
  uint8_t* base = prezeroed ? static_cast<uint8_t*>(d_zeroed) : sbase;
  // the report counters: straight into d_u_out when given (no copy-out node)
  unsigned long long* u = d_u_out ? d_u_out : reinterpret_cast<unsigned long long*>(base);
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(base) + 8;
  int2* cnt = reinterpret_cast<int2*>(hist + nb);
  uint8_t* notmin = reinterpret_cast<uint8_t*>(cnt + n);
  double* thr = reinterpret_cast<double*>(sbase + (prezeroed ? 0 : head));
  double* theta = thr + n;
  // u: [0] |S| [1] n_f_pre [2] max theta bits [3] ~(first bad row), 0 = none
  //    [4] converted [5] alpha_diag bits [6] max_theta bits (written by fcf_select)
  const bool vec = a.nnz >= (int64_t)cf_vec_rows() * n;
  const uint64_t key = splitmix64_host(seed ^ splitmix64_host(0x57454947ull));
  if (!prezeroed) {
    const int64_t words = (int64_t)((zero_bytes + 7) / 8);
    const unsigned gz = (unsigned)std::min<int64_t>(4 * c.num_sms, (words + 255) / 256 + 1);
    LAUNCH_PDL(c, fcf_zero, gz, 256, 0, reinterpret_cast<unsigned long long*>(base), words, d_u_out);
  }
  auto* k_rows = vec ? fcf_rows<true> : fcf_rows<false>;
  auto* k_marks = vec ? fcf_marks<true> : fcf_marks<false>;
  auto* k_theta = vec ? fcf_theta<true> : fcf_theta<false>;
  const int G = cf_lanes(n, a.nnz);
  if (G > 1) {
    const unsigned gl = (unsigned)(((int64_t)n * G + 255) / 256);
    auto* kr = G == 2 ? fcf_rows_lanes<2> : fcf_rows_lanes<4>;
    auto* km = G == 2 ? fcf_marks_lanes<2> : fcf_marks_lanes<4>;
    LAUNCH_PDL(c, kr, gl, 256, 0, n, a.rp.p, a.ci.p, a.v.p, alpha, thr, cnt, u);
    LAUNCH_PDL(c, km, gl, 256, 0, n, a.rp.p, a.ci.p, a.v.p, (const double*)thr, (const int2*)cnt, key, notmin);
  } else {
    LAUNCH_PDL(c, k_rows, g, 256, 0, n, a.rp.p, a.ci.p, a.v.p, alpha, thr, cnt, u);
    LAUNCH_PDL(c, k_marks, g, 256, 0, n, a.rp.p, a.ci.p, a.v.p, thr, cnt, key, notmin);
  }
  if (ddc_enabled) {
    LAUNCH_PDL(c, k_theta, g, 256, 0, n, a.rp.p, a.ci.p, a.v.p, notmin, theta, d_labels_pre, u + 2, u + 3);
    const unsigned hb = (unsigned)std::min<int64_t>(g, 4 * c.num_sms);
    const size_t smem = bins <= 8192 ? (size_t)bins * sizeof(unsigned) : 0;
    LAUNCH_PDL(c, fcf_hist, hb, 256, smem, n, notmin, theta, u + 2, bins, hist, u + 1);
    if (bins <= 8192) {
      const unsigned gs = (unsigned)std::min<int64_t>(c.num_sms, (n + kSelThreads - 1) / kSelThreads);
      LAUNCH_PDL(c, fcf_select_convert, gs, kSelThreads, 0, n, u + 1, hist, bins, fraction, u + 2,
                 reinterpret_cast<double*>(u + 5), notmin, theta, u + 3, d_labels, u + 4);
    } else {
      LAUNCH_PDL(c, fcf_select, 1, kSelThreads, 0, u + 1, 0ll, hist, bins, fraction, u + 2, 0, 0.0,
                 reinterpret_cast<double*>(u + 5));
      LAUNCH_PDL(c, fcf_convert, g, 256, 0, n, notmin, theta, reinterpret_cast<const double*>(u + 5), u + 3,
                 d_labels, u + 4);
    }
  } else {
    LAUNCH_PDL(c, fcf_labels, g, 256, 0, n, notmin, d_labels, u + 1);
    if (d_labels_pre)
      CUDA_CHECK(cudaMemcpyAsync(d_labels_pre, d_labels, n, cudaMemcpyDeviceToDevice, c.stream));
  }
  return u;
}

CfFused cf_split_fused_finish(Ctx& c, const unsigned long long* hu, bool ddc_enabled, const uint8_t* d_labels) {
  CfFused r;
  double hs[2];
  std::memcpy(hs, hu + 5, sizeof hs);
  if (ddc_enabled && hu[3] != 0) {
    // the reference names the A_ff row: the F sub-index of the fine row
    // (fcf_convert writes the PMISR labels when a row was bad)
    std::vector<uint8_t> lab((size_t)~hu[3]);
    if (!lab.empty()) to_host(c, lab.data(), d_labels, lab.size());
    int64_t sub = 0;
    for (uint8_t l : lab) sub += l == AIRG_F;
    throw RuntimeError("dominance_report: zero diagonal in A_ff row " + std::to_string(sub));
  }
  r.s_nnz = (int64_t)hu[0];
  r.n_f_pre = (int64_t)hu[1];
  r.n_converted = (int64_t)hu[4];
  r.alpha_diag = hs[0];
  r.max_theta = hs[1];
  return r;
}

CfFused cf_split_fused(Ctx& c, const Csr& a, double alpha, uint64_t seed, bool ddc_enabled,
                       double fraction, int64_t bins, uint8_t* d_labels, uint8_t* d_labels_pre) {
  NvtxRange nvtx__("airg CF split");
  const unsigned long long* u =
      cf_split_fused_enqueue(c, a, alpha, seed, ddc_enabled, fraction, bins, d_labels, d_labels_pre, nullptr);
  if (!u) return CfFused{};
  unsigned long long hu[8];
  to_host(c, hu, u, 8);
  return cf_split_fused_finish(c, hu, ddc_enabled, d_labels);
}

}  // namespace airg
