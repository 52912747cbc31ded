// AIRG solve on the GPU (reference: proj/src/solve.cpp).
//
// V-cycle (solve.cpp:93-146, entered with x = 0 and no pre-smoothing):
//   per level l: b_{l+1} = R_l b_l  ->  recurse  ->  x_l = P_l x_{l+1}
//   -> up_f_smooths x { r_F = (b_F - A_FF x_F) - A_FC x_C ;  x_F += Aff^-1 r_F }
//   coarsest: coarse_iterations x { r = b - A_c e (skipped first) ; e += Ac^-1 r }.
// Every kernel is thread-per-row with the reference's sequential order and
// separate rounding, so one V-cycle is bit-identical to the reference's;
// the F-point residual reads A's F rows directly (columns flagged F / C)
// instead of gathering x_F / x_C, with the two partial sums kept apart to
// reproduce (b_F - A_FF x_F) - A_FC x_C exactly.
// The whole V-cycle (+ the Richardson update and residual) is captured once
// into a CUDA graph and replayed each iteration; only the residual norm
// (parallel reduction) crosses to the host.
#include <chrono>
#include <cmath>
#include <cstring>

#include "hier.cuh"
#include "tiled.cuh"

namespace airg {

namespace {

// ---- epilogues of the tiled row kernels (tiled.cuh) --------------------------
// first F-smooth: r_F = (b_F - A_FF x_F) - A_FC x_C, keeping A_FC x_C for the
// following smooths (x_C is not changed by F-smoothing, solve.cpp:63-87)
struct EpiFres1 {
  const double* b;
  const int32_t* f2f;
  double* rf;
  double* sc_keep;
  // b_l comes from the descent (long complete): prefetched before the wait
  struct Pre {
    double bb;
  };
  __device__ Pre pre(int k) const { return Pre{b[__ldg(f2f + k)]}; }
  __device__ void row2_pre(int k, double sf, double sc, const Pre& p) const {
    sc_keep[k] = sc;
    rf[k] = __dsub_rn(__dsub_rn(p.bb, sf), sc);
  }
};
// later F-smooths: only A_FF x_F is recomputed
struct EpiFres2 {
  const double* b;
  const int32_t* f2f;
  const double* sc_keep;
  double* rf;
  __device__ void finish() const {}
  // b_l and A_FC x_C (from the first residual, three kernels back)
  struct Pre {
    double bb, sc;
  };
  __device__ Pre pre(int k) const { return Pre{b[__ldg(f2f + k)], sc_keep[k]}; }
  __device__ void row_pre(int k, double sf, const Pre& p) const {
    rf[k] = __dsub_rn(__dsub_rn(p.bb, sf), p.sc);
  }
};
// x_F += Aff^-1 r_F
struct EpiFupd {
  const int32_t* f2f;
  double* x;
  __device__ void finish() const {}
  // x_F was last written two kernels back (prolongation or the previous
  // update; the residual in between only reads it)
  struct Pre {
    int i;
    double x0;
  };
  __device__ Pre pre(int k) const {
    const int i = __ldg(f2f + k);
    return Pre{i, x[i]};
  }
  __device__ void row_pre(int, double d, const Pre& p) const { x[p.i] = __dadd_rn(p.x0, d); }
};
// coarse residual r = rhs - A_c e
struct EpiCres {
  const double* rhs;
  double* r;
  __device__ void finish() const {}
  struct Pre {  // the coarse rhs comes from the descent, >= 2 kernels back
    double rr;
  };
  __device__ Pre pre(int i) const { return Pre{rhs[i]}; }
  __device__ void row_pre(int i, double acc, const Pre& p) const { r[i] = __dsub_rn(p.rr, acc); }
};
// coarse update e += 1.0 * (Ac^-1 r)
struct EpiCupd {
  double* e;
  int first;
  __device__ void finish() const {}
  struct Pre {  // e from the previous update, two kernels back (a residual between)
    double e0;
  };
  __device__ Pre pre(int i) const { return Pre{first ? 0.0 : e[i]}; }
  __device__ void row_pre(int i, double acc, const Pre& p) const { e[i] = __dadd_rn(p.e0, __dmul_rn(1.0, acc)); }
};
// top residual r = b - A x with one partial sum of r^2 per block
struct EpiResid {
  const double* b;
  double* r;
  double* part;
  mutable double s;
  struct Pre {  // the right-hand side is constant during the solve
    double bb;
  };
  __device__ Pre pre(int i) const { return Pre{b[i]}; }
  __device__ void row_pre(int i, double acc, const Pre& p) const {
    const double ri = __dsub_rn(p.bb, acc);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  __device__ void finish() const {
    __shared__ double sm[32];  // any block size up to 1024 (SELL launches 256)
    double v = s;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
  }
};

// fast V-cycle, fused ascent (fused.cu): r1 = b_F - (A_F P) e_c
struct EpiFres1P {
  const double* b;
  const int32_t* f2f;
  double* rf;
  __device__ void finish() const {}
  struct Pre {  // b_l from the descent
    double bb;
  };
  __device__ Pre pre(int k) const { return Pre{b[__ldg(f2f + k)]}; }
  __device__ void row_pre(int k, double acc, const Pre& p) const { rf[k] = p.bb - acc; }
};
}  // namespace
}  // namespace airg
#include "fusedx.cuh"
namespace airg {
namespace {

// ec_early: e_c was produced two or more kernels back
void launch_fused_x(Ctx& c, const Level& lv, const double* ec, bool ec_early) {
  launch_fused_x_raw(c, lv.fw, lv.rf.p, lv.map.f_to_fine.p, lv.map.c_to_fine.p, (int)lv.map.nc, lv.pmap.p, ec,
                     lv.x.p, false, ec_early);
}
void launch_fused_k(Ctx& c, const Level& lv, const double* ec) {
  launch_fused_x_raw(c, lv.fk, lv.rf.p, lv.map.f_to_fine.p, lv.map.c_to_fine.p, (int)lv.map.nc, lv.pmap.p, ec,
                     lv.x.p, true, false);
}

// [b_{l+1}; y] = [R; W_k E_F^T] b_l: rows below n0 to y0, the rest to y1
struct EpiStore2 {
  double* y0;
  int n0;
  double* y1;
  __device__ void row(int r, double acc) const {
    if (r < n0)
      y0[r] = acc;
    else
      y1[r - n0] = acc;
  }
  __device__ void finish() const {}
};

// Row kernels of the solve in the configured arithmetic mode (tiled.cuh);
// `fast` must be in scope.
#define ROWS(Epi, M, x, epi) LAUNCH_ROWS_MODE(c, Epi, tview(M), x, epi, fast)
#define ROWS_FC(Epi, M, x, epi) LAUNCH_ROWS_FC_MODE(c, Epi, tview(M), x, epi, fast)

// x_l = 0 + P e_c  (solve.cpp:139-141: pe = spmv(P, ec); x += 1.0 * pe).
// Four rows per thread (int4 map load, two double2 stores; the level vectors
// come from the pool, 16-byte aligned); the last thread takes the n % 4 tail.
__device__ __forceinline__ double prolong_one(int j, const double* __restrict__ ec) {
  const double pe = j >= 0 ? __dadd_rn(0.0, __dmul_rn(1.0, ec[j])) : 0.0;
  return __dadd_rn(0.0, __dmul_rn(1.0, pe));
}
__global__ void k_prolong(int n, const int32_t* __restrict__ pmap, const double* __restrict__ ec,
                          double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = i < n ? __ldg(pmap + i) : -1;  // static data: before the dependency wait
  pdl_wait();
  pdl_trigger();
  if (i >= n) return;
  x[i] = prolong_one(j, ec);
}
__global__ void k_prolong4(int n, const int32_t* __restrict__ pmap, const double* __restrict__ ec,
                           double* __restrict__ x) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int n4 = n >> 2;
  int4 j = make_int4(-1, -1, -1, -1);
  if (q < n4) j = __ldg(reinterpret_cast<const int4*>(pmap) + q);
  pdl_wait();
  pdl_trigger();
  if (q == n4) {
    for (int i = 4 * n4; i < n; ++i) x[i] = prolong_one(__ldg(pmap + i), ec);
    return;
  }
  if (q > n4) return;
  const double a = prolong_one(j.x, ec), b = prolong_one(j.y, ec);
  const double c = prolong_one(j.z, ec), d = prolong_one(j.w, ec);
  double2* x2 = reinterpret_cast<double2*>(x);
  x2[2 * q] = make_double2(a, b);
  x2[2 * q + 1] = make_double2(c, d);
}

// x += 1.0 * e (solve.cpp:224), two entries per thread (pool vectors are
// 16-byte aligned; the last thread takes an odd tail)
__global__ void k_axpy1(int n, const double* __restrict__ e, double* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int n2 = n >> 1;
  if (q < n2) {
    const double2 ev = reinterpret_cast<const double2*>(e)[q];
    double2 xv = reinterpret_cast<double2*>(x)[q];
    xv.x = __dadd_rn(xv.x, __dmul_rn(1.0, ev.x));
    xv.y = __dadd_rn(xv.y, __dmul_rn(1.0, ev.y));
    reinterpret_cast<double2*>(x)[q] = xv;
  } else if (q == n2 && (n & 1)) {
    x[n - 1] = __dadd_rn(x[n - 1], __dmul_rn(1.0, e[n - 1]));
  }
}

__global__ void k_sum_partials(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double sm[32];
  pdl_wait();
  pdl_trigger();
  // four independent accumulators: the partial loads are issued together
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const int step = blockDim.x;
  int i = threadIdx.x;
  for (; i + 3 * step < np; i += 4 * step) {
    s0 += part[i];
    s1 += part[i + step];
    s2 += part[i + 2 * step];
    s3 += part[i + 3 * step];
  }
  for (; i < np; i += step) s0 += part[i];
  double s = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
  }
}

// Device-side convergence test of the Richardson loop (solve.cpp:196-224):
// it += 1; rel = sqrt(||r||^2) / sqrt(||b||^2) -- the same correctly rounded
// sqrt and division the host loop performs -- appended to the history; the
// WHILE condition stays 1 unless rel <= rtol or it >= max_iterations.
__global__ void k_loop_check(cudaGraphConditionalHandle hnd, const double* __restrict__ scal,
                             const double* __restrict__ par, long long* __restrict__ it,
                             double* __restrict__ hist, long long cap) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long k = *it + 1;
  *it = k;
  const double rel = sqrt(scal[0]) / sqrt(scal[1]);
  if (k < cap) hist[k] = rel;
  const bool stop = rel <= par[0] || (double)k >= par[1];
  cudaGraphSetConditional(hnd, stop ? 0u : 1u);
}

__global__ void k_stamp(const long long* __restrict__ it, double* __restrict__ hist, long long cap, int which) {
  if (threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const long long k = *it;
  const long long slot = 2 * k + which;
  if (slot < cap) hist[slot] = (double)t;
}

// ---- GMRES helpers
// partial dots of w with columns 0..j of V: grid (blocks, j+1)
__global__ void k_multidot(int64_t n, const double* __restrict__ V, const double* __restrict__ w,
                           double* __restrict__ part) {
  __shared__ double sm[32];
  const double* vk = V + (int64_t)blockIdx.y * n;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(vk[i], w[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}
__global__ void k_finish_dots(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double sm[32];
  double s = 0.0;
  const double* p = part + (int64_t)blockIdx.x * np;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += p[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
  }
}
// w -= V(:, 0..j) h  (h on device)
__global__ void k_orth_update(int64_t n, int jp1, const double* __restrict__ V,
                              const double* __restrict__ h, double* __restrict__ w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = w[i];
  for (int k = 0; k < jp1; ++k) s -= h[k] * V[(int64_t)k * n + i];
  w[i] = s;
}
// V(:, j+1) = w / hn and the V-cycle input buffer gets a copy
__global__ void k_scale_store(int64_t n, const double* __restrict__ w, double inv,
                              double* __restrict__ dst, double* __restrict__ dst2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = w[i] * inv;
  dst[i] = v;
  if (dst2) dst2[i] = v;
}
// x += Z(:, 0..j-1) y
__global__ void k_xupdate(int64_t n, int j, const double* __restrict__ Z, const double* __restrict__ y,
                          double* __restrict__ x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = x[i];
  for (int k = 0; k < j; ++k) s += y[k] * Z[(int64_t)k * n + i];
  x[i] = s;
}

constexpr int kT = 128;

// Enqueue one V-cycle from level 0 rhs b0 into levels[0].x (or the coarse
// x when there are no fine levels).
void enqueue_vcycle(Ctx& c, Hier& h, const airg_solve_config& cfg, const double* b0) {
  const bool fast = cfg.fast != 0;
  const int L = (int)h.levels.size();
  // descent: b_{l+1} = R_l b_l
  const bool fused = fast && fused_ready(h, cfg.up_f_smooths, cfg.coarse_iterations);
  for (int l = 0; l < L; ++l) {
    Level& lv = h.levels[l];
    const double* bl = l == 0 ? b0 : lv.b.p;
    double* bn = (l + 1 < L) ? h.levels[l + 1].b.p : h.cb.p;
    if (fused && lv.one_pass)  // y = W_k b_F into rf, for the one-pass ascent
      ROWS(EpiStore2, lv.dsc, bl, (EpiStore2{bn, lv.r.n, lv.rf.p}));
    else if (lv.r.n)
      ROWS(EpiStore, lv.r, bl, EpiStore{bn});
  }
  // coarse Richardson with the assembled polynomial (solve.cpp:34-59)
  const int nco = h.coarse_a.n;
  const double* rhs = L == 0 ? b0 : h.cb.p;
  if (nco && fused && h.coarse_composed) {  // e = E_k rhs (fused.cu)
    ROWS(EpiStore, h.coarse_e, rhs, EpiStore{h.cx.p});
  } else if (nco) {
    for (int64_t it = 0; it < cfg.coarse_iterations; ++it) {
      const double* r = rhs;
      if (it > 0) {
        ROWS(EpiCres, h.coarse_a, h.cx.p, (EpiCres{rhs, h.cr.p}));
        r = h.cr.p;
      }
      ROWS(EpiCupd, h.coarse_inv, r, (EpiCupd{h.cx.p, it == 0 ? 1 : 0}));
    }
    if (cfg.coarse_iterations <= 0) CUDA_CHECK(cudaMemsetAsync(h.cx.p, 0, sizeof(double) * nco, c.stream));
  }
  // ascent, fast fused form: two row passes per level (fused.cu)
  if (fused) {
    for (int l = L - 1; l >= 0; --l) {
      Level& lv = h.levels[l];
      const double* bl = l == 0 ? b0 : lv.b.p;
      const double* ec = (l + 1 < L) ? h.levels[l + 1].x.p : h.cx.p;
      if (lv.one_pass) {
        launch_fused_k(c, lv, ec);
        continue;
      }
      const bool res = cfg.up_f_smooths > 0 && lv.map.nf > 0;
      if (res) ROWS(EpiFres1P, lv.afp, ec, (EpiFres1P{bl, lv.map.f_to_fine.p, lv.rf.p}));
      launch_fused_x(c, lv, ec, res);
    }
    return;
  }
  // ascent: prolongate and F-smooth
  for (int l = L - 1; l >= 0; --l) {
    Level& lv = h.levels[l];
    const double* bl = l == 0 ? b0 : lv.b.p;
    const double* ec = (l + 1 < L) ? h.levels[l + 1].x.p : h.cx.p;
    const int n = lv.a.n, nf = lv.map.nf;
    if (n >= 4096)
      LAUNCH_PDL(c, k_prolong4, blocks_for(n / 4 + 1, 256), 256, 0, n, lv.pmap.p, ec, lv.x.p);
    else
      LAUNCH_PDL(c, k_prolong, blocks_for(n, kT), kT, 0, n, lv.pmap.p, ec, lv.x.p);
    for (int64_t s = 0; s < cfg.up_f_smooths && nf > 0; ++s) {
      if (s == 0)
        ROWS_FC(EpiFres1, lv.af, lv.x.p, (EpiFres1{bl, lv.map.f_to_fine.p, lv.rf.p, lv.sc.p}));
      else
        ROWS(EpiFres2, lv.affg, lv.x.p, (EpiFres2{bl, lv.map.f_to_fine.p, lv.sc.p, lv.rf.p}));
      ROWS(EpiFupd, lv.ffinv, lv.rf.p, (EpiFupd{lv.map.f_to_fine.p, lv.x.p}));
    }
  }
}

double* vcycle_output(Hier& h) { return h.levels.empty() ? h.cx.p : h.levels[0].x.p; }


// r = b - A x, ||r||^2 -> h.scal[0]
void enqueue_residual(Ctx& c, Hier& h, const double* b, const double* x, double* r, bool fast) {
  const Csr& a = h.top();
  ROWS(EpiResid, a, x, (EpiResid{b, r, h.part.p, 0.0}));
  const int nb = (int)rows_grid(tview(a), fast);
  LAUNCH_PDL(c, k_sum_partials, 1, 1024, 0, h.part.p, nb, h.scal.p);
}

int64_t graph_key(const Hier& h, const airg_solve_config& cfg) {
  // the fused operators' generation: a rebuild frees the buffers a cached
  // graph points to, so every build changes the key of the fused graphs
  const int64_t fused =
      (cfg.fast != 0 && fused_ready(h, cfg.up_f_smooths, cfg.coarse_iterations)) ? 1 + h.fused_gen : 0;
  return ((cfg.up_f_smooths * 1000003 + cfg.coarse_iterations * 31 + cfg.down_smooths) * 2 + (cfg.fast != 0)) *
             4096 + fused;
}

// Capture `body` into a graph executable; returns the number of kernels.
template <class F>
uint64_t capture(Ctx& c, cudaGraphExec_t* exec, F&& body) {
  if (*exec) {
    cudaGraphExecDestroy(*exec);
    *exec = nullptr;
  }
  const uint64_t before = c.launches;
  cudaGraph_t g;
  CUDA_CHECK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(c.stream, &dummy);
    if (dummy) cudaGraphDestroy(dummy);
    throw;
  }
  CUDA_CHECK(cudaStreamEndCapture(c.stream, &g));
  CUDA_CHECK(cudaGraphInstantiate(exec, g, 0));
  CUDA_CHECK(cudaGraphDestroy(g));
  const uint64_t k = c.launches - before;
  c.launches = before;
  return k;
}

void run_graph(Ctx& c, cudaGraphExec_t g, uint64_t kernels) {
  CUDA_CHECK(cudaGraphLaunch(g, c.stream));
  c.launches += kernels;
}

void check_cfg(const airg_solve_config& cfg) {
  if (cfg.down_smooths != 0)
    throw InvalidArgument("solve: down_smooths > 0 is not offered by the GPU V-cycle");
  if (cfg.rtol <= 0.0) throw InvalidArgument("richardson_solve: rtol must be positive");
}

// flops of one V-cycle exactly as the reference's primary counter tallies
// them (solve.cpp:93-146 with the coarse_solve/f_smooth counts).
uint64_t vcycle_flops(const Hier& h, const airg_solve_config& cfg) {
  uint64_t f = 0;
  for (const Level& L : h.levels) {
    f += 2 * (uint64_t)L.r.nnz;
    f += 2 * (uint64_t)L.p.nnz + 2 * (uint64_t)L.a.n;
    if (L.map.nf > 0)
      f += (uint64_t)cfg.up_f_smooths *
           (2 * (uint64_t)(L.aff.nnz + L.afc.nnz) + 2 * (uint64_t)L.map.nf + 2 * (uint64_t)L.ffinv.nnz +
            (uint64_t)L.map.nf);
  }
  const uint64_t nc = (uint64_t)h.coarse_a.n;
  for (int64_t it = 0; it < cfg.coarse_iterations; ++it) {
    if (it > 0) f += 2 * (uint64_t)h.coarse_a.nnz + 2 * nc;
    f += 2 * (uint64_t)h.coarse_inv.nnz + 2 * nc;
  }
  return f;
}

using Clock = std::chrono::steady_clock;

}  // namespace

// ---- single operations of the reference's solve / polynomial API ----------
namespace {
// Horner step (gmres_poly.cpp:188-193): acc = A acc, then acc += alpha * b
struct EpiHorner {
  const double* b;
  double alpha;
  double* y;
  __device__ void row(int i, double acc) const { y[i] = __dadd_rn(acc, __dmul_rn(alpha, b[i])); }
  __device__ void finish() const {}
};
__global__ void k_scale(int n, double a, const double* __restrict__ b, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dmul_rn(a, b[i]);
}
}  // namespace

// apply_polynomial (gmres_poly.cpp:173-195): q(A) b by Horner with
// effective_order matvecs, each product and sum rounded separately
void apply_polynomial(Ctx& c, Csr& a, const double* coeffs, int64_t ncoeffs, int64_t deg, const double* d_b,
                      double* d_y) {
  if (ncoeffs < 1) throw InvalidArgument("apply_polynomial: empty polynomial");
  if (deg < 0 || deg >= ncoeffs) throw InvalidArgument("apply_polynomial: effective_order out of range");
  if (deg > 0 && a.n != a.m) throw InvalidArgument("apply_polynomial: dimension mismatch");
  const int n = a.n;
  if (n == 0) return;
  DBuf<double> t(c, deg > 0 ? (size_t)n : 1);
  // ping-pong so that the last step lands in d_y
  double* cur = (deg % 2 == 0) ? d_y : t.p;
  double* nxt = (deg % 2 == 0) ? t.p : d_y;
  LAUNCH(c, k_scale, blocks_for(n, 256), 256, 0, n, coeffs[deg], d_b, cur);
  for (int64_t k = deg; k-- > 0;) {
    LAUNCH_ROWS(c, EpiHorner, tview(a), cur, (EpiHorner{d_b, coeffs[k], nxt}));
    std::swap(cur, nxt);
  }
}

// f_smooth (solve.cpp:63-87) on level l of a built hierarchy: x_F += Aff^-1
// ((b_F - A_FF x_F) - A_FC x_C), x of the level's size, C entries untouched
void f_smooth_level(Ctx& c, Hier& h, int64_t l, const double* d_b, double* d_x) {
  if (l < 0 || l >= (int64_t)h.levels.size()) throw InvalidArgument("f_smooth: level out of range");
  Level& lv = h.levels[(size_t)l];
  if (lv.map.nf == 0) return;
  const bool fast = false;
  ROWS_FC(EpiFres1, lv.af, d_x, (EpiFres1{d_b, lv.map.f_to_fine.p, lv.rf.p, lv.sc.p}));
  ROWS(EpiFupd, lv.ffinv, lv.rf.p, (EpiFupd{lv.map.f_to_fine.p, d_x}));
}

void vcycle(Ctx& c, Hier& h, const airg_solve_config& cfg, const double* d_b, double* d_x) {
  check_cfg(cfg);
  if (cfg.fast && !fused_ready(h, cfg.up_f_smooths, cfg.coarse_iterations))
    build_fused(c, h, cfg.up_f_smooths, cfg.coarse_iterations);
  const int n = h.top_n();
  CUDA_CHECK(cudaMemcpyAsync(h.r.p, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  const int64_t key = graph_key(h, cfg);
  if (!h.g_vc || h.g_key_vc != key) {
    h.g_vc_kernels = capture(c, &h.g_vc, [&] { enqueue_vcycle(c, h, cfg, h.r.p); });
    h.g_key_vc = key;
  }
  run_graph(c, h.g_vc, h.g_vc_kernels);
  CUDA_CHECK(cudaMemcpyAsync(d_x, vcycle_output(h), sizeof(double) * n, cudaMemcpyDeviceToDevice,
                             c.stream));
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

namespace {

// The whole Richardson loop as ONE graph launch: a conditional WHILE node
// whose body is the captured iteration (V-cycle, x += e, r = b - A x, ||r||^2)
// followed by k_loop_check, which sets the loop condition on the device. No
// host round trip between iterations. Returns false when the driver refuses
// the conditional graph (the caller then runs the host loop).
bool build_device_loop(Ctx& c, Hier& h, const airg_solve_config& cfg) {
  const int64_t key = graph_key(h, cfg);
  if (h.g_loop && h.g_key_loop == key) return true;
  if (h.g_loop) {
    cudaGraphExecDestroy(h.g_loop);
    h.g_loop = nullptr;
  }
  const int n = h.top_n();
  cudaGraph_t g = nullptr;
  CUDA_CHECK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hnd;
  cudaGraphNode_t node;
  cudaGraphNodeParams np = {};
  if (cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    return false;
  }
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = hnd;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &np) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    return false;
  }
  cudaGraph_t body = np.conditional.phGraph_out[0];
  const uint64_t before = c.launches;
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
  // AIRG_STAMPS=1 (diagnostic): %globaltimer at the start and the end of
  // every body iteration into loop_stamps (printed after the solve)
  static const bool stamps = [] {
    const char* e = getenv("AIRG_STAMPS");
    return e && e[0] == '1';
  }();
  try {
    if (stamps) LAUNCH(c, k_stamp, 1, 32, 0, h.loop_it.p, h.loop_stamps.p, (long long)h.loop_stamps.n, 0);
    enqueue_vcycle(c, h, cfg, h.r.p);
    LAUNCH_PDL(c, k_axpy1, blocks_for(n / 2 + 1, 256), 256, 0, n, vcycle_output(h), h.xsol.p);
    enqueue_residual(c, h, h.rhs.p, h.xsol.p, h.r.p, cfg.fast != 0);
    if (stamps) LAUNCH(c, k_stamp, 1, 32, 0, h.loop_it.p, h.loop_stamps.p, (long long)h.loop_stamps.n, 1);
    LAUNCH_PDL(c, k_loop_check, 1, 32, 0, hnd, (const double*)h.scal.p, (const double*)h.loop_par.p,
               h.loop_it.p, h.loop_hist.p, (long long)h.loop_hist.n);
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(c.stream, &dummy);
    cudaGraphDestroy(g);
    c.launches = before;
    throw;
  }
  cudaGraph_t captured;
  CUDA_CHECK(cudaStreamEndCapture(c.stream, &captured));
  const uint64_t k = c.launches - before;
  c.launches = before;
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  h.g_loop = exec;
  h.g_key_loop = key;
  h.g_loop_kernels = k;
  return true;
}

bool device_loop_enabled() {
  static const bool v = [] {
    const char* e = getenv("AIRG_DEVLOOP");
    return !(e && e[0] == '0');
  }();
  return v;
}

// richardson_solve (solve.cpp:167-259)
void richardson(Ctx& c, Hier& h, const airg_solve_config& cfg, airg_solve_stats& st,
                std::vector<double>& hist) {
  const Csr& a = h.top();
  const int n = a.n;
  uint64_t fc = 0;
  const uint64_t vflops = vcycle_flops(h, cfg);
  const auto t0 = Clock::now();
  CUDA_CHECK(cudaMemsetAsync(h.xsol.p, 0, sizeof(double) * n, c.stream));
  dot_async(c, h.rhs.p, h.rhs.p, n, h.scal.p + 1, h.part.p);
  const double bnorm = std::sqrt(read1(c, h.scal.p + 1));
  fc += 2 * (uint64_t)n;
  if (bnorm == 0.0) {
    st.converged = 1;
    hist.push_back(0.0);
  } else {
    const int64_t key = graph_key(h, cfg);
    if (!h.g_rich || h.g_key_rich != key) {
      h.g_rich_kernels = capture(c, &h.g_rich, [&] {
        enqueue_vcycle(c, h, cfg, h.r.p);
        const double* e = vcycle_output(h);
        LAUNCH_PDL(c, k_axpy1, blocks_for(n / 2 + 1, 256), 256, 0, n, e, h.xsol.p);
        enqueue_residual(c, h, h.rhs.p, h.xsol.p, h.r.p, cfg.fast != 0);
      });
      h.g_key_rich = key;
    }
    CUDA_CHECK(cudaMemcpyAsync(h.r.p, h.rhs.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    // device loop: the first test (rel = 1 at it = 0) on the host, the rest
    // inside the graph
    const int64_t cap = cfg.max_iterations + 1;
    const bool first_stops = 1.0 <= cfg.rtol || cfg.max_iterations <= 0;
    if (!first_stops && device_loop_enabled() && !h.loop_broken && cap <= (int64_t)1 << 20) {
      if (h.loop_hist.n < (size_t)cap) {
        // the captured k_loop_check holds the history pointer and capacity:
        // a reallocation invalidates the loop graph
        h.loop_hist.alloc(c, (size_t)cap);
        if (h.g_loop) {
          cudaGraphExecDestroy(h.g_loop);
          h.g_loop = nullptr;
        }
      }
      if (!h.loop_par.p) h.loop_par.alloc(c, 2);
      if (!h.loop_it.p) h.loop_it.alloc(c, 1);
      if (!h.loop_stamps.p) h.loop_stamps.alloc(c, 4096);
      if (!build_device_loop(c, h, cfg)) h.loop_broken = true;
    }
    if (!first_stops && device_loop_enabled() && !h.loop_broken && h.g_loop) {
      const double par[2] = {cfg.rtol, (double)cfg.max_iterations};
      to_device(c, h.loop_par.p, par, 2);
      CUDA_CHECK(cudaMemsetAsync(h.loop_it.p, 0, sizeof(long long), c.stream));
      CUDA_CHECK(cudaGraphLaunch(h.g_loop, c.stream));
      const long long its = read1(c, h.loop_it.p);
      const long long kept = std::min<long long>(its, (long long)h.loop_hist.n - 1);
      std::vector<double> hv((size_t)kept + 1);
      hv[0] = 1.0;
      if (kept > 0) to_host(c, hv.data() + 1, h.loop_hist.p + 1, (size_t)kept);
      for (double r : hv) hist.push_back(r);
      if (getenv("AIRG_STAMPS") && getenv("AIRG_STAMPS")[0] == '1') {  // diagnostic print
        std::vector<double> ts(h.loop_stamps.n);
        to_host(c, ts.data(), h.loop_stamps.p, ts.size());
        for (long long k = 0; k + 1 < its && 2 * k + 2 < (long long)ts.size(); ++k)
          fprintf(stderr, "iter %lld body %.1f us gap-to-next %.1f us\n", k, (ts[2 * k + 1] - ts[2 * k]) / 1e3,
                  (ts[2 * k + 2] - ts[2 * k + 1]) / 1e3);
      }
      c.launches += h.g_loop_kernels * (uint64_t)its;
      fc += (uint64_t)its * (vflops + 2 * (uint64_t)n) +
            (uint64_t)its * (2 * (uint64_t)a.nnz + 2 * (uint64_t)n + 2 * (uint64_t)n);
      st.final_relative_residual = hv.back();
      st.iterations = its;
      st.converged = hv.back() <= cfg.rtol ? 1 : 0;
    } else
    for (int64_t it = 0;; ++it) {
      double rel;
      if (it == 0) {
        rel = 1.0;
      } else {
        rel = std::sqrt(read1(c, h.scal.p)) / bnorm;
        fc += 2 * (uint64_t)a.nnz + 2 * (uint64_t)n + 2 * (uint64_t)n;
      }
      hist.push_back(rel);
      st.final_relative_residual = rel;
      if (rel <= cfg.rtol) {
        st.converged = 1;
        st.iterations = it;
        break;
      }
      if (it >= cfg.max_iterations) {
        st.converged = 0;
        st.iterations = it;
        break;
      }
      run_graph(c, h.g_rich, h.g_rich_kernels);
      fc += vflops + 2 * (uint64_t)n;
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  const auto t1 = Clock::now();
  st.flops = fc;
  st.shadow_flops = fc;
  st.work_units = (double)fc / (2.0 * (double)a.nnz);
  st.solve_seconds = std::chrono::duration<double>(t1 - t0).count();
}

// ---- device-resident GMRES ---------------------------------------------------
// The whole solve is ONE graph launch: an outer conditional WHILE over restart
// cycles whose body holds an inner WHILE over Arnoldi steps. Every scalar of
// the method (Hessenberg column, Givens rotations, g, y, the stopping tests)
// lives on the device; one readback at the end. One Arnoldi step:
//   z = M v_j (the captured V-cycle), w = A z with Z_j = z stored by the SpMV,
//   CGS2 in three sweeps over V_0..V_j (dots; update fused with the second
//   dots; update fused with the norm), the Givens step (one thread), and
//   v_{j+1} = w / h_{j+1,j}.
// The same steps, in the same order, as the host-driven gmres() below and the
// serial restatement (oracle/airg_oracle.c); reductions are parallel trees.
}  // namespace
}  // namespace airg
#include "gmres.cuh"
namespace airg {
namespace {

// L2 priority of the fast sweeps' basis loads (AIRG_L2_SWEEP: 1 evict_first,
// the default: 468 -> 466 us per C4 iteration; 0 default priority)
int sweep_l2() {
  static const int v = [] {
    const char* e = getenv("AIRG_L2_SWEEP");
    return (e && e[0]) ? atoi(e) : 1;
  }();
  return v;
}

// AIRG_GM_CHUNKED=0: the K-specialised register-tile sweeps in fast mode too
bool sweep_chunked() {
  static const bool v = [] {
    const char* e = getenv("AIRG_GM_CHUNKED");
    return !(e && e[0] == '0');
  }();
  return v;
}

// The GMRES orthogonalisation: the Gram-corrected two-sweep CGS2 over the
// unnormalised basis in BOTH arithmetic modes (GMRES is not part of the
// reference; exact mode's V-cycle and A z keep the reference's bits), or
// with AIRG_GM_EXACT_CGS=1 and exact mode the oracle's three-sweep CGS2.
bool gm_fast_orth(const airg_solve_config& cfg) {
  static const bool three = [] {
    const char* e = getenv("AIRG_GM_EXACT_CGS");
    return e && e[0] == '1';
  }();
  return cfg.fast != 0 || !three;
}

int gm_sweep_blocks(const Ctx&, int64_t n) { return gm_blocks(n); }

// capture helpers for building a graph with nested conditional nodes
template <class F>
std::vector<cudaGraphNode_t> capture_into(Ctx& c, cudaGraph_t g, const cudaGraphNode_t* deps, size_t ndeps,
                                          F&& body) {
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(c.stream, g, deps, nullptr, ndeps, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(c.stream, &dummy);
    throw;
  }
  cudaStreamCaptureStatus stt;
  const cudaGraphNode_t* sinks = nullptr;
  size_t ns = 0;
  CUDA_CHECK(cudaStreamGetCaptureInfo(c.stream, &stt, nullptr, nullptr, &sinks, &ns));
  std::vector<cudaGraphNode_t> out(sinks, sinks + ns);
  cudaGraph_t gg;
  CUDA_CHECK(cudaStreamEndCapture(c.stream, &gg));
  return out;
}

bool add_while(cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps, cudaGraphConditionalHandle* hnd,
               cudaGraphNode_t* node, cudaGraph_t* body) {
  if (cudaGraphConditionalHandleCreate(hnd, g, 0, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = *hnd;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  if (cudaGraphAddNode(node, g, deps.empty() ? nullptr : deps.data(), deps.size(), &np) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  *body = np.conditional.phGraph_out[0];
  return true;
}

// The pieces of the device GMRES, enqueued either into the nested
// conditional graph (cond = 1: the kernels set the WHILE handles) or, for
// profiling (AIRG_GM_FLAT=1, cond = 0), one by one under a host loop.
struct GmPieces {
  Ctx& c;
  Hier& h;
  const airg_solve_config& cfg;
  int64_t n;
  int nb, ns;  // element grid, sweep grid
  GmDev* st;
  double *V, *Z, *w, *H, *cs, *sn, *g, *y, *h1, *h2, *nrm, *part, *d, *hsum, *G;
  double* vs;  // fast mode: scales of the unnormalised basis (null: normalised basis)
  GmPieces(Ctx& c_, Hier& h_, const airg_solve_config& cfg_)
      : c(c_), h(h_), cfg(cfg_), n(h_.top_n()), nb(gm_blocks(h_.top_n())), ns(gm_sweep_blocks(c_, h_.top_n())),
        st(h_.gm_st.p), V(h_.V.p), Z(h_.Z.p),
        w(h_.w.p), H(h_.gm_H.p), cs(h_.gm_cs.p), sn(h_.gm_sn.p), g(h_.gm_g.p), y(h_.gm_y.p), h1(h_.gm_h.p),
        h2(h_.gm_h.p + (kGmMax + 1)), nrm(h_.gm_h.p + 2 * (kGmMax + 1)), part(h_.gm_part.p),
        d(h_.gm_h.p + 3 * (kGmMax + 1)), hsum(h_.gm_h.p + 5 * (kGmMax + 1)), G(h_.gm_G.p),
        vs(gm_fast_orth(cfg_) ? h_.gm_h.p + 6 * (kGmMax + 1) : nullptr) {}
  void norm_b() { dot_async(c, h.rhs.p, h.rhs.p, n, h.scal.p + 1, h.part.p); }
  void init(cudaGraphConditionalHandle hout, int cond) {
    LAUNCH(c, k_gm_init, 1, 32, 0, hout, cond, (const double*)(h.scal.p + 1), st, h.gm_hist.p);
  }
  void cycle(cudaGraphConditionalHandle hin, int cond) {
    LAUNCH(c, k_gm_cycle, (unsigned)nb, kGmThreads, 0, hin, cond, n, (const double*)h.r2.p, st, V, h.r.p, g, vs);
  }
  void tail(cudaGraphConditionalHandle hout, int cond) {
    const bool fast = cfg.fast != 0;
    LAUNCH_PDL(c, k_gm_ysolve, 1, 32, 0, (const GmDev*)st, (const double*)H, (const double*)g, y);
    LAUNCH_PDL(c, k_gm_xupdate, (unsigned)nb, kGmThreads, 0, n, (const GmDev*)st, (const double*)Z,
               (const double*)y, h.xsol.p);
    enqueue_residual(c, h, h.rhs.p, h.xsol.p, h.r2.p, fast);
    LAUNCH_PDL(c, k_gm_restart, 1, 32, 0, hout, cond, st, (const double*)h.scal.p);
  }
  // Fast mode keeps the basis UNNORMALISED: the second sweep writes
  // w'' = w - V (h1 + h2) into V_{j+1} and the V-cycle input directly,
  // k_gm_step records vs[j+1] = 1 / |w''|, the sweeps scale V_k by vs[k] in
  // registers and the A z epilogue scales z and A z by vs[j] (M is linear),
  // so no pass forms v = w / |w| (16 MB read + 32 MB written per step).
  void step(cudaGraphConditionalHandle hin, int cond) {
    const bool fast = cfg.fast != 0;    // arithmetic of the row kernels (V-cycle, A z)
    const bool fgm = gm_fast_orth(cfg);  // Gram-corrected CGS2 over the unnormalised basis
    enqueue_vcycle(c, h, cfg, h.r.p);
    const double* z = vcycle_output(h);
    ROWS(EpiGmSpmv, h.top(), z, (EpiGmSpmv{w, z, Z, st, n, vs}));
    const double* hcol1 = h1;
    const double* cV = V;
    int nsf = ns;  // partials of the last sweep
    if (fgm && n % 2 == 0 && sweep_chunked()) {  // Gram-corrected CGS2, chunked two-element sweeps
      const int pp = n % 4 == 0 ? 2 : 1;  // 4 elements per thread (C4: 437 -> 435 us per iteration)
      nsf = (int)std::max<int64_t>(1, (n / (2 * pp) + kGmThreads - 1) / kGmThreads);
      auto* k3 = pp == 2 ? &k_gm_sweep_fast<3, 2> : &k_gm_sweep_fast<3, 1>;
      auto* k2 = pp == 2 ? &k_gm_sweep_fast<2, 2> : &k_gm_sweep_fast<2, 1>;
      LAUNCH_PDL(c, k3, (unsigned)nsf, kGmThreads, 0, n, cV, (const double*)w, (const GmDev*)st,
                 (const double*)nullptr, part, (const double*)vs, V, h.r.p);
      LAUNCH_PDL(c, k_gm_finish, 2 * kGmMax, kFinThreads, 0, (const double*)part, nsf, (const GmDev*)st, 0, d);
      LAUNCH_PDL(c, k_gm_gram, 1, 32, 0, (const GmDev*)st, (const double*)d, G, h2, hsum);
      LAUNCH_PDL(c, k2, (unsigned)nsf, kGmThreads, 0, n, cV, (const double*)w, (const GmDev*)st,
                 (const double*)hsum, part, (const double*)vs, V, h.r.p);
      hcol1 = d;
    } else if (fgm) {  // Gram-corrected CGS2: two sweeps (k_gm_gram)
      LAUNCH_PDL(c, (k_gm_sweep<3, true>), (unsigned)ns, kGmThreads, 0, n, cV, w, (const GmDev*)st,
                 (const double*)nullptr, part, (const double*)vs, V, h.r.p, sweep_l2());
      LAUNCH_PDL(c, k_gm_finish, 2 * kGmMax, kFinThreads, 0, (const double*)part, ns, (const GmDev*)st, 0, d);
      LAUNCH_PDL(c, k_gm_gram, 1, 32, 0, (const GmDev*)st, (const double*)d, G, h2, hsum);
      LAUNCH_PDL(c, (k_gm_sweep<2, true>), (unsigned)ns, kGmThreads, 0, n, cV, w, (const GmDev*)st,
                 (const double*)hsum, part, (const double*)vs, V, h.r.p, sweep_l2());
      hcol1 = d;
    } else {  // CGS2 as the oracle: three sweeps
      LAUNCH_PDL(c, (k_gm_sweep<0, false>), (unsigned)ns, kGmThreads, 0, n, cV, w, (const GmDev*)st,
                 (const double*)nullptr, part, (const double*)nullptr, (double*)nullptr, (double*)nullptr, 0);
      LAUNCH_PDL(c, k_gm_finish, kGmMax, kFinThreads, 0, (const double*)part, ns, (const GmDev*)st, 0, h1);
      LAUNCH_PDL(c, (k_gm_sweep<1, false>), (unsigned)ns, kGmThreads, 0, n, cV, w, (const GmDev*)st,
                 (const double*)h1, part, (const double*)nullptr, (double*)nullptr, (double*)nullptr, 0);
      LAUNCH_PDL(c, k_gm_finish, kGmMax, kFinThreads, 0, (const double*)part, ns, (const GmDev*)st, 0, h2);
      LAUNCH_PDL(c, (k_gm_sweep<2, false>), (unsigned)ns, kGmThreads, 0, n, cV, w, (const GmDev*)st,
                 (const double*)h2, part, (const double*)nullptr, (double*)nullptr, (double*)nullptr, 0);
    }
    LAUNCH_PDL(c, k_gm_finish, 1, kFinThreads, 0, (const double*)part, nsf, (const GmDev*)st, 1, nrm);
    LAUNCH_PDL(c, k_gm_step, 1, 32, 0, hin, cond, st, hcol1, (const double*)h2, (const double*)nrm, H,
               cs, sn, g, h.gm_hist.p, vs);
    if (!fgm)
      LAUNCH_PDL(c, k_gm_next, (unsigned)nb, kGmThreads, 0, n, (const double*)w, (const GmDev*)st, V, h.r.p);
  }
};

// Build the device GMRES graph for restart m; false when the driver refuses
// nested conditional graphs (the host-driven loop is used then).
bool build_gmres_graph(Ctx& c, Hier& h, const airg_solve_config& cfg, int m) {
  const int64_t key = graph_key(h, cfg) * 1024 + m;
  if (h.g_gm && h.g_key_gm == key) return true;
  if (h.g_gm) {
    cudaGraphExecDestroy(h.g_gm);
    h.g_gm = nullptr;
  }
  GmPieces pc(c, h, cfg);
  const uint64_t before = c.launches;
  cudaGraph_t gr = nullptr;
  CUDA_CHECK(cudaGraphCreate(&gr, 0));
  bool ok = true;
  uint64_t k_init = 0, k_cycle = 0, k_step = 0, k_tail = 0;
  try {
    cudaGraphConditionalHandle hout, hin;
    cudaGraphNode_t nout, nin;
    cudaGraph_t bout, bin;
    // top level: ||b||^2, init, outer WHILE
    uint64_t c0 = c.launches;
    auto d0 = capture_into(c, gr, nullptr, 0, [&] { pc.norm_b(); });
    // the handle must exist before k_gm_init is captured: create the outer
    // node first, then capture the init kernel ahead of it
    ok = add_while(gr, {}, &hout, &nout, &bout);
    if (ok) {
      auto d1 = capture_into(c, gr, d0.data(), d0.size(), [&] { pc.init(hout, 1); });
      CUDA_CHECK(cudaGraphAddDependencies(gr, d1.data(), std::vector<cudaGraphNode_t>(d1.size(), nout).data(),
                                          d1.size()));
      k_init = c.launches - c0;
      // outer body: cycle start, inner WHILE, cycle end
      c0 = c.launches;
      ok = add_while(bout, {}, &hin, &nin, &bin);
    }
    if (ok) {
      auto e0 = capture_into(c, bout, nullptr, 0, [&] { pc.cycle(hin, 1); });
      CUDA_CHECK(cudaGraphAddDependencies(bout, e0.data(), std::vector<cudaGraphNode_t>(e0.size(), nin).data(),
                                          e0.size()));
      k_cycle = c.launches - c0;
      c0 = c.launches;
      capture_into(c, bout, &nin, 1, [&] { pc.tail(hout, 1); });
      k_tail = c.launches - c0;
      // inner body: one Arnoldi step
      c0 = c.launches;
      capture_into(c, bin, nullptr, 0, [&] { pc.step(hin, 1); });
      k_step = c.launches - c0;
    }
  } catch (...) {
    cudaGraphDestroy(gr);
    c.launches = before;
    throw;
  }
  c.launches = before;
  if (!ok) {
    cudaGraphDestroy(gr);
    return false;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, gr, 0);
  cudaGraphDestroy(gr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  h.g_gm = exec;
  h.g_key_gm = key;
  h.gm_kernels[0] = k_init;
  h.gm_kernels[1] = k_cycle + k_tail;
  h.gm_kernels[2] = k_step;
  return true;
}

// the device-resident solve; false: not available (host loop instead)
bool gmres_device(Ctx& c, Hier& h, const airg_solve_config& cfg, int m, airg_solve_stats& st,
                  std::vector<double>& hist) {
  if (!device_loop_enabled() || h.gm_broken || m > kGmMax || cfg.max_iterations <= 0) return false;
  const int64_t n = h.top_n();
  const int nb = gm_blocks(n);
  const int64_t cap = cfg.max_iterations + 1;
  if (h.gm_restart != m) {
    h.V.alloc(c, (size_t)n * (m + 1));
    h.Z.alloc(c, (size_t)n * m);
    h.gm_restart = m;
    if (h.g_gm) {
      cudaGraphExecDestroy(h.g_gm);
      h.g_gm = nullptr;
    }
  }
  if (!h.w.p) h.w.alloc(c, (size_t)n);
  if (!h.r2.p) h.r2.alloc(c, (size_t)n);
  if (!h.gm_st.p) {
    h.gm_st.alloc(c, 1);
    h.gm_H.alloc(c, (size_t)(kGmMax + 1) * kGmMax);
    h.gm_cs.alloc(c, kGmMax);
    h.gm_sn.alloc(c, kGmMax);
    h.gm_g.alloc(c, kGmMax + 1);
    h.gm_y.alloc(c, kGmMax);
    h.gm_h.alloc(c, 7 * (kGmMax + 1));
    h.gm_G.alloc(c, (size_t)(kGmMax + 1) * (kGmMax + 1));
    h.gm_part.alloc(c, (size_t)2 * (kGmMax + 1) * nb);
  }
  if (h.gm_hist.n < (size_t)cap) {
    h.gm_hist.alloc(c, (size_t)cap);
    if (h.g_gm) {  // the captured kernels hold the history pointer
      cudaGraphExecDestroy(h.g_gm);
      h.g_gm = nullptr;
    }
  }
  static const bool flat = [] {
    const char* e = getenv("AIRG_GM_FLAT");
    return e && e[0] == '1';
  }();
  if (!flat && !build_gmres_graph(c, h, cfg, m)) {
    h.gm_broken = true;
    return false;
  }
  GmDev s0 = {};
  s0.cap = (long long)h.gm_hist.n;
  s0.maxit = cfg.max_iterations;
  s0.m = m;
  s0.rtol = cfg.rtol;
  to_device(c, h.gm_st.p, &s0, 1);
  CUDA_CHECK(cudaMemsetAsync(h.xsol.p, 0, sizeof(double) * n, c.stream));
  CUDA_CHECK(cudaMemcpyAsync(h.r2.p, h.rhs.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  GmDev s1;
  if (flat) {
    // profiling form: the same kernels launched one by one (no graph), the
    // loop tests evaluated on the host from the device state
    GmPieces pc(c, h, cfg);
    const uint64_t l0 = c.launches;
    pc.norm_b();
    pc.init(0, 0);
    to_host(c, &s1, h.gm_st.p, 1);
    bool outer = s1.bnorm != 0.0 && s1.maxit > 0;
    while (outer) {
      pc.cycle(0, 0);
      bool more = s1.its < s1.maxit;
      while (more) {
        pc.step(0, 0);
        to_host(c, &s1, h.gm_st.p, 1);
        more = s1.j < s1.m && s1.its < s1.maxit && !(s1.est <= s1.rtol) && s1.hn != 0.0;
      }
      pc.tail(0, 0);
      to_host(c, &s1, h.gm_st.p, 1);
      outer = !s1.converged && s1.beta != 0.0 && s1.its < s1.maxit;
    }
    c.launches = l0 + (c.launches - l0);
  } else {
    CUDA_CHECK(cudaGraphLaunch(h.g_gm, c.stream));
    to_host(c, &s1, h.gm_st.p, 1);
  }
  const long long kept = std::min<long long>(s1.its, (long long)h.gm_hist.n - 1);
  std::vector<double> hv((size_t)kept + 1);
  to_host(c, hv.data(), h.gm_hist.p, hv.size());
  for (double r : hv) hist.push_back(r);
  st.iterations = s1.its;
  st.converged = s1.converged;
  st.final_relative_residual = s1.rel;
  if (!flat)
    c.launches += h.gm_kernels[0] + h.gm_kernels[1] * (uint64_t)s1.restarts + h.gm_kernels[2] * (uint64_t)s1.its;
  return true;
}

// Right-preconditioned restarted GMRES with flexible storage Z = M V,
// CGS2 orthogonalisation and Givens rotations; the restatement in
// oracle/airg_oracle.c (gmres) performs the same steps serially.
void gmres(Ctx& c, Hier& h, const airg_solve_config& cfg, airg_solve_stats& st,
           std::vector<double>& hist) {
  const Csr& a = h.top();
  const int64_t n = a.n;
  const int m = (int)(cfg.gmres_restart > 0 ? cfg.gmres_restart : 30);
  if (m > 512) throw InvalidArgument("gmres: restart length above 512");
  uint64_t fc = 0;
  const uint64_t vflops = vcycle_flops(h, cfg);
  {
    const auto t0 = Clock::now();
    if (gmres_device(c, h, cfg, m, st, hist)) {
      // flops as the host loop counts them: ||b||; per step the V-cycle, A z,
      // two CGS passes (4 n (j+1) each) and |w|; per cycle A x and |r|
      const uint64_t nn = (uint64_t)n;
      fc = 2 * nn;
      int64_t cycles = 0;
      for (int64_t k = 0; k < st.iterations; ++k) {
        const uint64_t j = (uint64_t)(k % m);
        if (j == 0) ++cycles;
        fc += vflops + 2 * (uint64_t)a.nnz + 8 * nn * (j + 1) + 2 * nn;
      }
      fc += (uint64_t)cycles * (2 * (uint64_t)a.nnz + 2 * nn);
      st.flops = fc;
      st.shadow_flops = fc;
      st.work_units = (double)fc / (2.0 * (double)a.nnz);
      st.solve_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
      return;
    }
  }
  if (h.gm_restart != m) {
    h.V.alloc(c, (size_t)n * (m + 1));
    h.Z.alloc(c, (size_t)n * m);
    h.w.alloc(c, (size_t)n);
    const int nb = (int)std::min<int64_t>(256, blocks_for(n, 256));
    h.hbuf.alloc(c, (size_t)(m + 2) * (nb + 4));
    h.ybuf.alloc(c, (size_t)m + 2);
    h.gm_restart = m;
  }
  const int nb = (int)std::min<int64_t>(256, blocks_for(n, 256));
  const auto t0 = Clock::now();
  CUDA_CHECK(cudaMemsetAsync(h.xsol.p, 0, sizeof(double) * n, c.stream));
  dot_async(c, h.rhs.p, h.rhs.p, n, h.scal.p + 1, h.part.p);
  const double bnorm = std::sqrt(read1(c, h.scal.p + 1));
  fc += 2 * (uint64_t)n;
  int64_t its = 0;
  st.converged = 0;
  if (bnorm == 0.0) {
    st.converged = 1;
    hist.push_back(0.0);
    st.final_relative_residual = 0.0;
  } else {
    const int64_t key = graph_key(h, cfg);
    if (!h.g_vc || h.g_key_vc != key) {
      h.g_vc_kernels = capture(c, &h.g_vc, [&] { enqueue_vcycle(c, h, cfg, h.r.p); });
      h.g_key_vc = key;
    }
    CUDA_CHECK(cudaMemcpyAsync(h.w.p, h.rhs.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
    double beta = bnorm;
    hist.push_back(1.0);
    st.final_relative_residual = 1.0;
    std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), hcol(m + 2), y(m + 1);
    std::vector<double> hh(2 * (m + 1) + 1);
    double* dh = h.hbuf.p;                     // [2][m+1] dots + [1] norm^2
    double* dpart = h.hbuf.p + 2 * (m + 1) + 2;  // partials
    while (its < cfg.max_iterations) {
      LAUNCH(c, k_scale_store, blocks_for(n, 256), 256, 0, n, h.w.p, 1.0 / beta, h.V.p, h.r.p);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      for (; j < m && its < cfg.max_iterations; ++j) {
        double* zj = h.Z.p + (int64_t)j * n;
        run_graph(c, h.g_vc, h.g_vc_kernels);  // r-buffer (= v_j) -> e
        fc += vflops;
        CUDA_CHECK(cudaMemcpyAsync(zj, vcycle_output(h), sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                   c.stream));
        spmv(c, a, zj, h.w.p);
        fc += 2 * (uint64_t)a.nnz;
        for (int pass = 0; pass < 2; ++pass) {
          LAUNCH(c, k_multidot, dim3(nb, j + 1), 256, 0, n, h.V.p, h.w.p, dpart);
          LAUNCH(c, k_finish_dots, j + 1, 256, 0, dpart, nb, dh + pass * (m + 1));
          LAUNCH(c, k_orth_update, blocks_for(n, 256), 256, 0, n, j + 1, h.V.p, dh + pass * (m + 1),
                 h.w.p);
          fc += 4 * (uint64_t)n * (uint64_t)(j + 1);
        }
        dot_async(c, h.w.p, h.w.p, n, dh + 2 * (m + 1), h.part.p);
        fc += 2 * (uint64_t)n;
        to_host(c, hh.data(), dh, 2 * (m + 1) + 1);
        for (int k = 0; k <= j; ++k) hcol[k] = hh[k] + hh[(m + 1) + k];
        const double hn = std::sqrt(hh[2 * (m + 1)]);
        hcol[j + 1] = hn;
        LAUNCH(c, k_scale_store, blocks_for(n, 256), 256, 0, n, h.w.p, hn > 0.0 ? 1.0 / hn : 0.0,
               h.V.p + (int64_t)(j + 1) * n, h.r.p);
        for (int k = 0; k < j; ++k) {
          const double t = cs[k] * hcol[k] + sn[k] * hcol[k + 1];
          hcol[k + 1] = -sn[k] * hcol[k] + cs[k] * hcol[k + 1];
          hcol[k] = t;
        }
        const double den = std::hypot(hcol[j], hcol[j + 1]);
        cs[j] = den > 0.0 ? hcol[j] / den : 1.0;
        sn[j] = den > 0.0 ? hcol[j + 1] / den : 0.0;
        hcol[j] = den;
        hcol[j + 1] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        for (int k = 0; k <= j; ++k) H[k + (size_t)j * (m + 1)] = hcol[k];
        ++its;
        const double est = std::fabs(g[j + 1]) / bnorm;
        hist.push_back(est);
        if (est <= cfg.rtol || hn == 0.0) {
          ++j;
          break;
        }
      }
      for (int k = j - 1; k >= 0; --k) {
        double s = g[k];
        for (int q = k + 1; q < j; ++q) s -= H[k + (size_t)q * (m + 1)] * y[q];
        y[k] = s / H[k + (size_t)k * (m + 1)];
      }
      to_device(c, h.ybuf.p, y.data(), (size_t)j);
      LAUNCH(c, k_xupdate, blocks_for(n, 256), 256, 0, n, j, h.Z.p, h.ybuf.p, h.xsol.p);
      enqueue_residual(c, h, h.rhs.p, h.xsol.p, h.w.p, cfg.fast != 0);
      fc += 2 * (uint64_t)a.nnz + 2 * (uint64_t)n;
      beta = std::sqrt(read1(c, h.scal.p));
      const double rel = beta / bnorm;
      st.final_relative_residual = rel;
      if (rel <= cfg.rtol) {
        st.converged = 1;
        break;
      }
      if (beta == 0.0) break;
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  const auto t1 = Clock::now();
  st.iterations = its;
  st.flops = fc;
  st.shadow_flops = fc;
  st.work_units = (double)fc / (2.0 * (double)a.nnz);
  st.solve_seconds = std::chrono::duration<double>(t1 - t0).count();
}

}  // namespace

void solve(Ctx& c, Hier& h, const airg_solve_config& cfg, const double* d_b, double* d_x,
           airg_solve_stats& st, std::vector<double>& history) {
  NvtxRange nvtx__("airg solve");
  check_cfg(cfg);
  if (cfg.fast && !fused_ready(h, cfg.up_f_smooths, cfg.coarse_iterations))
    build_fused(c, h, cfg.up_f_smooths, cfg.coarse_iterations);
  std::memset(&st, 0, sizeof st);
  const int n = h.top_n();
  CUDA_CHECK(cudaMemcpyAsync(h.rhs.p, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  if (cfg.outer == 1)
    gmres(c, h, cfg, st, history);
  else
    richardson(c, h, cfg, st, history);
  CUDA_CHECK(cudaMemcpyAsync(d_x, h.xsol.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  st.grid_complexity = h.grid_c;
  st.operator_complexity = h.op_c;
  st.storage_complexity = h.store_c;
  st.history_len = (int64_t)history.size();
  if (st.iterations > 0) {
    const double ns = st.solve_seconds * 1e9;
    st.c_grind_ns = ns / (double)n / (double)st.iterations;
    if (cfg.nddofs > 0) st.d_grind_ns = ns / (double)cfg.nddofs / (double)st.iterations;
  }
}

}  // namespace airg
