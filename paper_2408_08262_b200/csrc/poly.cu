// GMRES-polynomial approximate inverses (reference: proj/src/gmres_poly.cpp)
// and the smoother growth guard (proj/src/air.cpp:61-129).
#include <cmath>
#include <cstring>

#include "dd.cuh"
#include "rowsplit.cuh"
#include "sparse.cuh"
#include "tiled.cuh"

namespace airg {

namespace {

__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t d_mix(uint64_t seed, uint64_t key) {
  return d_splitmix64(seed ^ d_splitmix64(key));
}
// rng::standard_normal (rng.hpp:32-39)
__device__ __forceinline__ double d_standard_normal(uint64_t seed, uint64_t index) {
  const double u1 = (double)((d_mix(seed, 2 * index) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(d_mix(seed, 2 * index + 1) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

__global__ void normal_fill(int64_t n, uint64_t seed, double* __restrict__ hi,
                            double* __restrict__ lo, int64_t base = 0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  hi[i] = d_standard_normal(seed, (uint64_t)(base + i));
  if (lo) lo[i] = 0.0;
}

// K_k = A K_{k-1} in double-double (values are doubles, products exact).
__global__ void dd_spmv(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                        const double* __restrict__ v, const double* __restrict__ xh,
                        const double* __restrict__ xl, double* __restrict__ yh,
                        double* __restrict__ yl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dd acc = {0.0, 0.0};
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int c = ci[k];
    acc = dd_add(acc, dd_mul_d(dd{xh[c], xl[c]}, v[k]));
  }
  yh[i] = acc.hi;
  yl[i] = acc.lo;
}

// Gram entries G_ab = sum_i K_a[i] K_b[i] in double-double. blockIdx.y is
// the pair; partial sums per block, finished on the host.
__global__ void dd_gram(int64_t n, int ncols, const double* __restrict__ kh,
                        const double* __restrict__ kl, const int2* __restrict__ pairs,
                        double* __restrict__ part) {
  __shared__ double sh[256], sl[256];
  const int2 pr = pairs[blockIdx.y];
  const double* ah = kh + (int64_t)pr.x * n;
  const double* al = kl + (int64_t)pr.x * n;
  const double* bh = kh + (int64_t)pr.y * n;
  const double* bl = kl + (int64_t)pr.y * n;
  dd acc = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = dd_add(acc, dd_mul(dd{ah[i], al[i]}, dd{bh[i], bl[i]}));
  sh[threadIdx.x] = acc.hi;
  sl[threadIdx.x] = acc.lo;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      dd r = dd_add(dd{sh[threadIdx.x], sl[threadIdx.x]}, dd{sh[threadIdx.x + s], sl[threadIdx.x + s]});
      sh[threadIdx.x] = r.hi;
      sl[threadIdx.x] = r.lo;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t o = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 2;
    part[o] = sh[0];
    part[o + 1] = sl[0];
  }
}

// ---- assemble_fixed_sparsity (gmres_poly.cpp:197-280)
// rows r of a slab are global rows rb + r (rp/ci: the whole matrix)
__global__ void pattern_count_s1(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 int32_t* __restrict__ cnt, int rb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  bool seen = false;
  for (int k = rp[i]; k < rp[i + 1]; ++k) seen |= ci[k] == i;
  cnt[r] = rp[i + 1] - rp[i] + (seen ? 0 : 1);
}
// sorted union of row i of P, {i} and row i of A
__global__ void pattern_union_count(int n, const int32_t* __restrict__ prp,
                                    const int32_t* __restrict__ pci, const int32_t* __restrict__ arp,
                                    const int32_t* __restrict__ aci, int32_t* __restrict__ cnt,
                                    const int32_t* __restrict__ orp, int32_t* __restrict__ oci, int rb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  int p = prp ? prp[i] : 0, pe = prp ? prp[i + 1] : 0, q = arp[i], qe = arp[i + 1];
  bool diag = false;
  int last = -1, c = 0, o = orp ? orp[r] : 0;
  while (p < pe || q < qe || !diag) {
    int cand = INT32_MAX;
    if (p < pe) cand = pci[p];
    if (q < qe && aci[q] < cand) cand = aci[q];
    if (!diag && i < cand) cand = i;
    if (cand == i) diag = true;
    if (p < pe && pci[p] == cand) ++p;
    if (q < qe && aci[q] == cand) ++q;
    if (cand != last) {
      if (oci) oci[o + c] = cand;
      ++c;
    }
    last = cand;
  }
  if (cnt) cnt[r] = c;
}

__device__ __forceinline__ int find_pos(const int32_t* __restrict__ cols, int w, int key) {
  int lo = 0, hi = w;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cols[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < w && cols[lo] == key) ? lo : -1;
}

__global__ void assemble_rows(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                              const double* __restrict__ av, const int32_t* __restrict__ orp,
                              const int32_t* __restrict__ oci, double* __restrict__ ov,
                              double* __restrict__ curb, double* __restrict__ nextb,
                              const double* __restrict__ coeffs, int deg, int rb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  const int o = orp[r], w = orp[r + 1] - o;
  const int32_t* prow = oci + o;
  double* out = ov + o;
  double* cur = curb + o;
  double* next = nextb + o;
  const double a0 = coeffs[0];
  for (int k = 0; k < w; ++k) {
    out[k] = prow[k] == i ? a0 : 0.0;
    cur[k] = 0.0;
  }
  for (int k = arp[i]; k < arp[i + 1]; ++k) {
    const int p = find_pos(prow, w, aci[k]);
    cur[p] = av[k];
    if (deg >= 1) out[p] = __dadd_rn(out[p], __dmul_rn(coeffs[1], av[k]));
  }
  for (int power = 2; power <= deg; ++power) {
    for (int k = 0; k < w; ++k) next[k] = 0.0;
    for (int k = 0; k < w; ++k) {
      const double v = cur[k];
      if (v == 0.0) continue;
      const int j = prow[k];
      for (int t = arp[j]; t < arp[j + 1]; ++t) {
        const int p = find_pos(prow, w, aci[t]);
        if (p < 0) continue;  // outside the fixed pattern
        next[p] = __dadd_rn(next[p], __dmul_rn(v, av[t]));
      }
    }
    const double alpha = coeffs[power];
    for (int k = 0; k < w; ++k) out[k] = __dadd_rn(out[k], __dmul_rn(alpha, next[k]));
    double* t = cur;
    cur = next;
    next = t;
  }
}

// ---- growth estimate helpers
__global__ void sub_partial(int n, double* __restrict__ v, const double* __restrict__ q,
                            double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = v[i] - q[i];
    v[i] = x;
    s += x * x;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}
__global__ void finish_norm(const double* __restrict__ part, int np, double* __restrict__ g) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *g = sqrt(s);
  }
}
__global__ void scale_by(int n, double* __restrict__ v, const double* __restrict__ g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double gg = *g;
  if (i < n && gg != 0.0) v[i] = v[i] / gg;
}

// growth guard, one power step in two row passes (single GPU): the iterate u
// is kept unnormalised with its norm g from the previous step --
//   av = (A u) / g;   u <- u / g - Q av,  one partial of |u|^2 per block
struct EpiScaled {  // y = acc / g (g from the predecessor: read after the wait)
  double* y;
  const double* g;
  __device__ void row(int i, double acc) const { y[i] = acc / *g; }
  __device__ void finish() const {}
};
struct EpiGrowth {  // u_i <- u_i / g - (Q av)_i, |u| of the new iterate into *gout
  double* u;
  const double* g;
  double* part;
  unsigned* ticket;  // zero between launches
  double* gout;
  mutable double s;
  struct Pre {
    double ui, gg;
  };
  __device__ Pre pre(int i) const { return Pre{u[i], *g}; }  // both from the previous step's launch, two kernels back
  __device__ void row_pre(int i, double acc, const Pre& p) const {
    const double r = p.ui / p.gg - acc;
    u[i] = r;
    s += r * r;
  }
  // one partial of |u|^2 per block; the block that finishes last sums the
  // partials in index order (the same sum whichever block it is) and writes
  // the norm: no separate finishing launch on the step's chain
  __device__ void finish() const {
    __shared__ double sm[32];
    __shared__ bool last;
    double v = s;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) {
        part[blockIdx.x] = v;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
      }
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += __ldcg(part + i);
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x < 32) {
      t = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) {
        *gout = sqrt(t);
        *ticket = 0u;
      }
    }
  }
};
}  // namespace

// ---------------------------------------------------------------------------
// compute_coefficients (gmres_poly.cpp:63-171), native GPU mode. Instead of a
// Householder QR of the normalised n x (m+1) power basis in long double, the
// GPU forms the basis and its Gram matrix G = K^T K in double-double and the
// host factors G (Cholesky == QR's R up to row signs), applies the same rank
// cut (|R_kk| < 1e-12 on the normalised basis), the same candidate-degree
// least-squares solves and scores each candidate's true residual from G.
namespace {
using DV = std::vector<dd>;

// Householder reflector of x (length k): beta = -sign(x0)|x|, v0 = 1,
// tau = (beta - x0) / beta (the same convention as oracle/shim).
void dd_house(const dd* x, int k, DV& v, dd& tau, dd& beta) {
  v.assign(x, x + k);
  dd tail{0.0, 0.0};
  for (int i = 1; i < k; ++i) tail = dd_add(tail, dd_mul(x[i], x[i]));
  const dd c0 = x[0];
  if (tail.hi <= 0.0) {
    tau = dd{0.0, 0.0};
    beta = c0;
    for (int i = 1; i < k; ++i) v[i] = dd{0.0, 0.0};
    v[0] = dd{1.0, 0.0};
    return;
  }
  beta = dd_sqrt(dd_add(dd_mul(c0, c0), tail));
  if (c0.hi >= 0.0) beta = dd_neg(beta);
  const dd den = dd_sub(c0, beta);
  for (int i = 1; i < k; ++i) v[i] = dd_div(x[i], den);
  v[0] = dd{1.0, 0.0};
  tau = dd_div(dd_sub(beta, c0), beta);
}

// Minimum-norm least squares through a complete orthogonal decomposition in
// double-double, with the semantics of Eigen's CompleteOrthogonalDecomposition
// under setThreshold(thr) (gmres_poly.cpp:144-147): column-pivoted
// Householder QR (pivot = largest remaining column norm, first on ties),
// rank = #{|R_jj| > thr * max_j |R_jj|}, a right-side Householder (RZ)
// reduction of the rank-r trapezoid, y = P Z^T [T11^-1 (Q^T b)_r ; 0].
// a: m x n row-major (overwritten). Returns the rank (0: no solution).
int cod_solve(DV a, int m, int n, DV b, double thr, DV& y) {
  const int k = std::min(m, n);
  std::vector<int> perm(n);
  for (int j = 0; j < n; ++j) perm[j] = j;
  auto A = [&](int i, int j) -> dd& { return a[(size_t)i * n + j]; };
  DV x, v;
  double maxpiv = 0.0;
  for (int j = 0; j < k; ++j) {
    int best = j;
    double bestn = -1.0;
    for (int c = j; c < n; ++c) {
      dd s{0.0, 0.0};
      for (int i = j; i < m; ++i) s = dd_add(s, dd_mul(A(i, c), A(i, c)));
      if (s.hi > bestn) {
        bestn = s.hi;
        best = c;
      }
    }
    if (best != j) {
      for (int i = 0; i < m; ++i) std::swap(A(i, j), A(i, best));
      std::swap(perm[j], perm[best]);
    }
    x.resize(m - j);
    for (int i = j; i < m; ++i) x[i - j] = A(i, j);
    dd tau, beta;
    dd_house(x.data(), m - j, v, tau, beta);
    if (tau.hi != 0.0) {
      for (int c = j + 1; c < n; ++c) {
        dd s{0.0, 0.0};
        for (int i = 0; i < m - j; ++i) s = dd_add(s, dd_mul(v[i], A(j + i, c)));
        s = dd_mul(s, tau);
        for (int i = 0; i < m - j; ++i) A(j + i, c) = dd_sub(A(j + i, c), dd_mul(s, v[i]));
      }
      dd s{0.0, 0.0};  // b <- H b
      for (int i = 0; i < m - j; ++i) s = dd_add(s, dd_mul(v[i], b[j + i]));
      s = dd_mul(s, tau);
      for (int i = 0; i < m - j; ++i) b[j + i] = dd_sub(b[j + i], dd_mul(s, v[i]));
    }
    A(j, j) = beta;
    for (int i = j + 1; i < m; ++i) A(i, j) = dd{0.0, 0.0};
    maxpiv = std::max(maxpiv, fabs(beta.hi));
  }
  int r = 0;
  for (int j = 0; j < k; ++j)
    if (fabs(A(j, j).hi) > thr * maxpiv) ++r;
  if (r == 0) return 0;
  // RZ: annihilate columns [r, n) of the top r rows with right reflectors
  // acting on {kk} u [r, n)
  std::vector<DV> zv(r);
  DV ztau(r, dd{0.0, 0.0});
  if (r < n) {
    for (int kk = r - 1; kk >= 0; --kk) {
      x.assign(1 + (n - r), dd{0.0, 0.0});
      x[0] = A(kk, kk);
      for (int c = r; c < n; ++c) x[1 + c - r] = A(kk, c);
      dd tau, beta;
      dd_house(x.data(), (int)x.size(), v, tau, beta);
      for (int rr = 0; rr <= kk; ++rr) {
        dd s = dd_mul(A(rr, kk), v[0]);
        for (int c = r; c < n; ++c) s = dd_add(s, dd_mul(A(rr, c), v[1 + c - r]));
        s = dd_mul(s, tau);
        A(rr, kk) = dd_sub(A(rr, kk), dd_mul(s, v[0]));
        for (int c = r; c < n; ++c) A(rr, c) = dd_sub(A(rr, c), dd_mul(s, v[1 + c - r]));
      }
      zv[kk] = v;
      ztau[kk] = tau;
    }
  }
  DV w(n, dd{0.0, 0.0});
  for (int i = r - 1; i >= 0; --i) {
    dd s = b[i];
    for (int j = i + 1; j < r; ++j) s = dd_sub(s, dd_mul(A(i, j), w[j]));
    w[i] = dd_div(s, A(i, i));
  }
  for (int kk = 0; kk < (int)zv.size(); ++kk) {
    if (ztau[kk].hi == 0.0 || zv[kk].empty()) continue;
    const DV& zk = zv[kk];
    dd s = dd_mul(w[kk], zk[0]);
    for (int i = 1; i < (int)zk.size(); ++i) s = dd_add(s, dd_mul(zk[i], w[r + i - 1]));
    s = dd_mul(s, ztau[kk]);
    w[kk] = dd_sub(w[kk], dd_mul(s, zk[0]));
    for (int i = 1; i < (int)zk.size(); ++i) w[r + i - 1] = dd_sub(w[r + i - 1], dd_mul(s, zk[i]));
  }
  y.assign(n, dd{0.0, 0.0});
  for (int j = 0; j < n; ++j) y[perm[j]] = w[j];
  return r;
}
}  // namespace

PolyFit poly_coefficients(Ctx& c, const Csr& a, int64_t m, uint64_t seed, const RowSplit* rs) {
  if (a.n != a.m) throw InvalidArgument("compute_coefficients: matrix must be square");
  if (m < 1) throw InvalidArgument("compute_coefficients: m must be >= 1");
  const int64_t n = a.n;
  if (n == 0) throw InvalidArgument("compute_coefficients: empty matrix");
  const int nc = (int)(m + 1);
  DBuf<double> kh(c, (size_t)(n * nc)), kl(c, (size_t)(n * nc));
  const uint64_t rhs_seed = mix_host(seed, 0x504f4c59ull);
  LAUNCH(c, normal_fill, blocks_for(n, 256), 256, 0, n, rhs_seed, kh.p, kl.p);
  if (rs) {  // row slabs per rank, gathered after every power (rowsplit.cuh)
    RowSlices sl;
    sl.build(c, *rs, a);
    for (int k = 1; k <= m; ++k) {
      for (int r = 0; r < rs->P; ++r) {
        const Csr& p = sl.part[r];
        if (!rs->mine(r) || !p.n) continue;
        LAUNCH(c, dd_spmv, blocks_for(p.n, 128), 128, 0, p.n, p.rp.p, p.ci.p, p.v.p, kh.p + (k - 1) * n,
               kl.p + (k - 1) * n, kh.p + k * n + sl.s[r], kl.p + k * n + sl.s[r]);
      }
      rs->gather_vec(c, kh.p + k * n, sl.s);
      rs->gather_vec(c, kl.p + k * n, sl.s);
    }
  } else {
    for (int k = 1; k <= m; ++k)
      LAUNCH(c, dd_spmv, blocks_for(n, 128), 128, 0, (int)n, a.rp.p, a.ci.p, a.v.p,
             kh.p + (k - 1) * n, kl.p + (k - 1) * n, kh.p + k * n, kl.p + k * n);
  }
  std::vector<dd> G;
  poly_gram(c, n, nc, kh.p, kl.p, G);
  return poly_fit_gram(G, nc, m, n);
}

// G = K^T K in double-double over n rows (K: nc columns of n, hi / lo
// planes); per-block partials summed on the host in block order.
void poly_gram(Ctx& c, int64_t n, int nc, const double* kh, const double* kl, std::vector<dd>& G) {
  std::vector<int2> pairs;
  for (int x = 0; x < nc; ++x)
    for (int y = x; y < nc; ++y) pairs.push_back(make_int2(x, y));
  G.assign((size_t)nc * nc, dd{0.0, 0.0});
  if (n == 0) return;
  DBuf<int2> dpairs(c, pairs.size());
  to_device(c, dpairs.p, pairs.data(), pairs.size());
  const int gblocks = (int)std::min<int64_t>(64, blocks_for(n, 256));
  DBuf<double> part(c, pairs.size() * gblocks * 2);
  LAUNCH(c, dd_gram, dim3(gblocks, (unsigned)pairs.size()), 256, 0, n, nc, kh, kl, dpairs.p, part.p);
  std::vector<double> hp(pairs.size() * gblocks * 2);
  to_host(c, hp.data(), part.p, hp.size());
  for (size_t pi = 0; pi < pairs.size(); ++pi) {
    dd s = {0.0, 0.0};
    for (int b = 0; b < gblocks; ++b) s = dd_add(s, dd{hp[(pi * gblocks + b) * 2], hp[(pi * gblocks + b) * 2 + 1]});
    G[pairs[pi].x * nc + pairs[pi].y] = s;
    G[pairs[pi].y * nc + pairs[pi].x] = s;
  }
}

// The host half of compute_coefficients from the Gram matrix of the power
// basis over n rows (nc = m + 1 columns).
PolyFit poly_fit_gram(const std::vector<dd>& G, int nc, int64_t m, int64_t n) {
  // normalised Gram and Cholesky (upper R, row-major R[i*nc+j])
  std::vector<dd> scale(nc);
  for (int k = 0; k < nc; ++k) scale[k] = dd_sqrt(G[k * nc + k]);
  if (scale[0].hi == 0.0) throw RuntimeError("compute_coefficients: zero right-hand side");
  const int rrows = (int)std::min<int64_t>(n, nc);
  std::vector<dd> N((size_t)nc * nc), R((size_t)nc * nc, dd{0.0, 0.0});
  for (int x = 0; x < nc; ++x)
    for (int y = 0; y < nc; ++y) {
      if (scale[x].hi == 0.0 || scale[y].hi == 0.0) {
        N[x * nc + y] = dd{0.0, 0.0};
        continue;
      }
      N[x * nc + y] = dd_div(G[x * nc + y], dd_mul(scale[x], scale[y]));
    }
  int dim = 0;
  for (int k = 0; k < rrows; ++k) {
    dd d = N[k * nc + k];
    for (int j = 0; j < k; ++j) d = dd_sub(d, dd_mul(R[j * nc + k], R[j * nc + k]));
    const dd rkk = d.hi > 0.0 ? dd_sqrt(d) : dd{0.0, 0.0};
    R[k * nc + k] = rkk;
    if (fabs(rkk.hi) < 1e-12) break;  // gmres_poly.cpp:116-120
    ++dim;
    for (int j = k + 1; j < nc; ++j) {
      dd s = N[k * nc + j];
      for (int i = 0; i < k; ++i) s = dd_sub(s, dd_mul(R[i * nc + k], R[i * nc + j]));
      R[k * nc + j] = dd_div(s, rkk);
    }
  }
  if (dim == 0) throw RuntimeError("compute_coefficients: singular projected system");
  // unscale: R = R_scaled diag(scale)
  for (int i = 0; i < nc; ++i)
    for (int k = 0; k < nc; ++k) R[i * nc + k] = dd_mul(R[i * nc + k], scale[k]);
  const int lcols = (int)std::min<int64_t>(m, dim);
  int best_d = 0;
  double best_resid = INFINITY;
  std::vector<double> best_y;
  for (int d = 1; d <= lcols; ++d) {
    const int lrows = std::min(rrows, d + 1);
    // the reference's CompleteOrthogonalDecomposition with threshold 1e-12
    // (gmres_poly.cpp:141-147): column-pivoted rank decision, minimum-norm
    // solution when the unscaled block is numerically rank deficient
    std::vector<dd> H((size_t)lrows * d), rhs(lrows, dd{0.0, 0.0});
    for (int i = 0; i < lrows; ++i)
      for (int j = 0; j < d; ++j) H[i * d + j] = R[i * nc + 1 + j];
    rhs[0] = R[0];
    std::vector<dd> y;
    if (cod_solve(H, lrows, d, rhs, 1e-12, y) == 0) continue;
    bool finite = true;
    for (int j = 0; j < d; ++j) finite &= std::isfinite(y[j].hi);
    if (!finite) continue;
    // ||K_0 - sum_k y_k K_{k+1}||^2 from the Gram matrix
    dd q = G[0];
    for (int k = 0; k < d; ++k) q = dd_sub(q, dd_mul(dd_from(2.0), dd_mul(y[k], G[0 * nc + k + 1])));
    for (int k = 0; k < d; ++k)
      for (int l = 0; l < d; ++l) q = dd_add(q, dd_mul(dd_mul(y[k], y[l]), G[(k + 1) * nc + l + 1]));
    const double resid = q.hi > 0.0 ? dd_sqrt(q).hi / scale[0].hi : 0.0;
    if (resid < best_resid) {
      best_resid = resid;
      best_d = d;
      best_y.resize(d);
      for (int j = 0; j < d; ++j) best_y[j] = y[j].hi + y[j].lo;
    }
  }
  if (best_d == 0) throw RuntimeError("compute_coefficients: singular projected system");
  PolyFit f;
  f.coeffs.assign((size_t)m, 0.0);
  for (int k = 0; k < best_d; ++k) f.coeffs[k] = best_y[k];
  f.effective_order = best_d - 1;
  return f;
}

void poly_basis_fill(Ctx& c, int64_t n, int64_t base, uint64_t seed, double* hi, double* lo) {
  if (n) LAUNCH(c, normal_fill, blocks_for(n, 256), 256, 0, n, seed, hi, lo, base);
}
void poly_dd_spmv(Ctx& c, const Csr& a, const double* xh, const double* xl, double* yh, double* yl) {
  if (a.n) LAUNCH(c, dd_spmv, blocks_for(a.n, 128), 128, 0, a.n, a.rp.p, a.ci.p, a.v.p, xh, xl, yh, yl);
}

namespace {
// rows rb.. (n of them) of the sparsity-1 assembly, a local CSR with global columns
void assemble_slab_s1(Ctx& c, const Csr& a, int rb, int n, const double* d_coeffs, int64_t deg, Csr& r) {
  r.n = n;
  r.m = a.n;
  r.rp.alloc(c, (size_t)n + 1);
  DBuf<int32_t> cnt(c, (size_t)std::max(1, n));
  if (n) LAUNCH(c, pattern_count_s1, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, cnt.p, rb);
  r.nnz = exclusive_scan(c, cnt.p, r.rp.p, n);
  r.ci.alloc(c, (size_t)r.nnz);
  r.v.alloc(c, (size_t)r.nnz);
  if (!n) return;
  LAUNCH(c, pattern_union_count, blocks_for(n, 256), 256, 0, n, (const int32_t*)nullptr,
         (const int32_t*)nullptr, a.rp.p, a.ci.p, (int32_t*)nullptr, r.rp.p, r.ci.p, rb);
  DBuf<double> cur(c, (size_t)std::max<int64_t>(1, r.nnz)), nxt(c, (size_t)std::max<int64_t>(1, r.nnz));
  LAUNCH(c, assemble_rows, blocks_for(n, 128), 128, 0, n, a.rp.p, a.ci.p, a.v.p, r.rp.p, r.ci.p, r.v.p,
         cur.p, nxt.p, d_coeffs, (int)deg, rb);
}
}  // namespace

void poly_assemble_rows(Ctx& c, const Csr& a, int rb, int n, const double* h_coeffs, int64_t ncoeffs,
                        int64_t deg, Csr& out) {
  if (ncoeffs < 1) throw InvalidArgument("assemble_fixed_sparsity: empty polynomial");
  if (deg >= ncoeffs) throw InvalidArgument("assemble_fixed_sparsity: effective order exceeds coefficients");
  DBuf<double> coeffs(c, (size_t)ncoeffs);
  to_device(c, coeffs.p, h_coeffs, (size_t)ncoeffs);
  assemble_slab_s1(c, a, rb, n, coeffs.p, deg, out);
  CUDA_CHECK(cudaStreamSynchronize(c.stream));  // coeffs scratch freed on return
}

void poly_assemble(Ctx& c, const Csr& a, const double* h_coeffs, int64_t ncoeffs, int64_t deg,
                   int64_t sparsity_order, Csr& out, const RowSplit* rs) {
  if (rs && sparsity_order == 1 && a.n == a.m && ncoeffs >= 1 && deg < ncoeffs) {
    DBuf<double> coeffs(c, (size_t)ncoeffs);
    to_device(c, coeffs.p, h_coeffs, (size_t)ncoeffs);
    const std::vector<int64_t> s = rs->slabs(a.n);
    std::vector<Csr> slab(rs->P);
    for (int r = 0; r < rs->P; ++r)
      if (rs->mine(r)) assemble_slab_s1(c, a, (int)s[r], (int)(s[r + 1] - s[r]), coeffs.p, deg, slab[r]);
    gather_csr(c, *rs, s, slab, a.n, out);
    return;
  }
  if (a.n != a.m) throw InvalidArgument("assemble_fixed_sparsity: square matrix only");
  if (sparsity_order < 1) throw InvalidArgument("assemble_fixed_sparsity: sparsity_order >= 1");
  if (ncoeffs < 1) throw InvalidArgument("assemble_fixed_sparsity: empty polynomial");
  if (deg >= ncoeffs) throw InvalidArgument("assemble_fixed_sparsity: effective order exceeds coefficients");
  const int n = a.n;
  Csr r;
  r.n = r.m = n;
  r.rp.alloc(c, (size_t)n + 1);
  DBuf<int32_t> cnt(c, (size_t)n);
  Csr power;  // pattern(A^s) for s >= 2
  if (sparsity_order >= 2) {
    Csr ones;
    csr_copy(c, a, power);
    for (int64_t k = 1; k < sparsity_order; ++k) {
      Csr nxt;
      spgemm(c, power, a, nxt);
      power = std::move(nxt);
    }
  }
  if (n) {
    if (sparsity_order >= 2)
      LAUNCH(c, pattern_union_count, blocks_for(n, 256), 256, 0, n, power.rp.p, power.ci.p, a.rp.p,
             a.ci.p, cnt.p, (const int32_t*)nullptr, (int32_t*)nullptr, 0);
    else
      LAUNCH(c, pattern_count_s1, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, cnt.p, 0);
  }
  r.nnz = exclusive_scan(c, cnt.p, r.rp.p, n);
  r.ci.alloc(c, (size_t)r.nnz);
  r.v.alloc(c, (size_t)r.nnz);
  if (n) {
    LAUNCH(c, pattern_union_count, blocks_for(n, 256), 256, 0, n,
           sparsity_order >= 2 ? power.rp.p : (const int32_t*)nullptr,
           sparsity_order >= 2 ? power.ci.p : (const int32_t*)nullptr, a.rp.p, a.ci.p,
           (int32_t*)nullptr, r.rp.p, r.ci.p, 0);
    DBuf<double> coeffs(c, (size_t)ncoeffs), cur(c, (size_t)r.nnz), nxt(c, (size_t)r.nnz);
    to_device(c, coeffs.p, h_coeffs, (size_t)ncoeffs);
    LAUNCH(c, assemble_rows, blocks_for(n, 128), 128, 0, n, a.rp.p, a.ci.p, a.v.p, r.rp.p, r.ci.p,
           r.v.p, cur.p, nxt.p, coeffs.p, (int)deg, 0);
  }
  out = std::move(r);
}

// smoother_growth_estimate (air.cpp:61-95): 30 normalised power iterations
// of I - q(A) A, geometric mean of the rates of iterations 15..29. All 30
// steps are enqueued without a host round trip; the per-step norms come back
// once at the end (parallel reductions: not bit-identical to the reference's
// sequential sums, which only matters at the 0.5 acceptance boundary).
double smoother_growth(Ctx& c, const Csr& a, const Csr& q, const RowSplit* rs) {
  const int n = a.n;
  if (n == 0) return 0.0;
  constexpr int kIters = 30, kTail = 15;
  DBuf<double> v(c, (size_t)n), av(c, (size_t)n), qav(c, (size_t)n), g(c, kIters + 1);
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>(kReduceBlocks, blocks_for(n, threads));
  DBuf<double> part(c, (size_t)blocks);
  const uint64_t probe_seed = mix_host(0xA3B1C5D7ull, (uint64_t)n);
  LAUNCH(c, normal_fill, blocks_for(n, 256), 256, 0, (int64_t)n, probe_seed, v.p, (double*)nullptr);
  // norm of v: reuse sub_partial with q = 0
  DBuf<double> zero(c, (size_t)n);
  zero.zero(c);
  LAUNCH(c, sub_partial, blocks, threads, 0, n, v.p, zero.p, part.p);
  LAUNCH(c, finish_norm, 1, 1024, 0, part.p, blocks, g.p + kIters);
  if (rs) LAUNCH(c, scale_by, blocks_for(n, 256), 256, 0, n, v.p, g.p + kIters);
  RowSlices sa, sq;
  if (rs) {
    sa.build(c, *rs, a);
    sq.build(c, *rs, q);
  }
  if (!rs) {
    // two PDL-chained launches per step (v is rescaled in the next step's
    // epilogues instead of by a separate pass; the norm is finished by the
    // last block of the second launch)
    const TileView tq = tview(q);
    const int nbq = (int)rows_grid(tq, false);
    DBuf<double> qpart(c, (size_t)nbq);
    DBuf<unsigned> ticket(c, 1);
    ticket.zero(c);
    for (int k = 0; k < kIters; ++k) {
      const double* gprev = k == 0 ? g.p + kIters : g.p + k - 1;
      LAUNCH_ROWS(c, EpiScaled, tview(a), v.p, (EpiScaled{av.p, gprev}));
      LAUNCH_ROWS(c, EpiGrowth, tq, av.p, (EpiGrowth{v.p, gprev, qpart.p, ticket.p, g.p + k, 0.0}));
    }
  }
  for (int k = 0; k < (rs ? kIters : 0); ++k) {
    if (rs) {  // slab SpMVs, gathered: the norms below see the same full vectors
      split_spmv(c, *rs, sa, v.p, av.p);
      split_spmv(c, *rs, sq, av.p, qav.p);
    } else {
      spmv(c, a, v.p, av.p);
      spmv(c, q, av.p, qav.p);
    }
    LAUNCH(c, sub_partial, blocks, threads, 0, n, v.p, qav.p, part.p);
    LAUNCH(c, finish_norm, 1, 1024, 0, part.p, blocks, g.p + k);
    LAUNCH(c, scale_by, blocks_for(n, 256), 256, 0, n, v.p, g.p + k);
  }
  double hg[kIters + 1];
  to_host(c, hg, g.p, kIters + 1);
  double log_growth = 0.0;
  int tail = 0;
  for (int k = 0; k < kIters; ++k) {
    if (hg[k] == 0.0) return 0.0;
    if (k >= kTail) {
      log_growth += std::log(hg[k]);
      ++tail;
    }
  }
  return std::exp(log_growth / tail);
}

}  // namespace airg
