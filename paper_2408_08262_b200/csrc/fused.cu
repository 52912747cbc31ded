// Fused level operators of the fast V-cycle (airg_solve_config::fast).
//
// The reference's up-sweep on level l (solve.cpp:93-146, :63-87) is
//   x = P e_c;  k times { r_F = b_F - A_F x ;  x_F += Q r_F }     (Q = Aff^-1)
// -- a prolongation and 2k dependent row passes. Written out, with r1 the
// first residual, the k F-smooths leave
//   r_{i+1} = (I - A_ff Q) r_i,   x_F = (P e_c)_F + W_k r1,
//   W_1 = Q,  W_{k+1} = Q + W_k - (W_k A_ff) Q,   r1 = b_F - (A_F P) e_c,
// so the same V-cycle (exactly, up to rounding) runs as TWO row passes per
// level: r1 from the prolongation-fused residual operator A_F P (n_f x n_c),
// then x_l = P e_c + [W_k r1 on the F rows] in one launch whose first blocks
// are lane groups over W_k's rows and whose last blocks prolongate the C
// points (solve.cu k_fused_x). Both operators are
// formed once at setup by the SpGEMMs of spgemm.cu; at the C4 and C2 fine
// levels W_2 = 2Q - Q A_ff Q has fewer entries than Q + A_ff + Q together
// (the F-F graph is sparse), so the fused pass moves fewer bytes as well
// as halving the dependent launches of the ascent (6 -> 3 per level, with
// the restriction on the way down).
#include "hier.cuh"

namespace airg {

namespace {

__global__ void k_unflag_cols(int64_t nnz, const int32_t* __restrict__ ci, int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) out[k] = ci[k] & 0x7fffffff;
}

// C = alpha A + beta B, same shape, sorted rows (union of the patterns).
__global__ void add_count(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                          const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                          int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = arp[i], q = brp[i];
  const int pe = arp[i + 1], qe = brp[i + 1];
  int c = 0;
  while (p < pe || q < qe) {
    const int ca = p < pe ? aci[p] : INT32_MAX, cb = q < qe ? bci[q] : INT32_MAX;
    if (ca <= cb) ++p;
    if (cb <= ca) ++q;
    ++c;
  }
  cnt[i] = c;
}
__global__ void add_fill(int n, double alpha, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                         const double* __restrict__ av, double beta, const int32_t* __restrict__ brp,
                         const int32_t* __restrict__ bci, const double* __restrict__ bv,
                         const int32_t* __restrict__ crp, int32_t* __restrict__ cci, double* __restrict__ cv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = arp[i], q = brp[i], o = crp[i];
  const int pe = arp[i + 1], qe = brp[i + 1];
  while (p < pe || q < qe) {
    const int ca = p < pe ? aci[p] : INT32_MAX, cb = q < qe ? bci[q] : INT32_MAX;
    double s = 0.0;
    if (ca <= cb) s = fma(alpha, av[p++], s);
    if (cb <= ca) s = fma(beta, bv[q++], s);
    cci[o] = ca < cb ? ca : cb;
    cv[o++] = s;
  }
}

void csr_add(Ctx& c, double alpha, const Csr& a, double beta, const Csr& b, Csr& out) {
  if (a.n != b.n || a.m != b.m) throw InvalidArgument("csr_add: shape mismatch");
  const int n = a.n;
  Csr r;
  r.n = n;
  r.m = a.m;
  r.rp.alloc(c, (size_t)n + 1);
  DBuf<int32_t> cnt(c, (size_t)std::max(1, n));
  if (n) LAUNCH(c, add_count, blocks_for(n, 256), 256, 0, n, a.rp.p, a.ci.p, b.rp.p, b.ci.p, cnt.p);
  r.nnz = exclusive_scan(c, cnt.p, r.rp.p, n);
  r.ci.alloc(c, (size_t)r.nnz);
  r.v.alloc(c, (size_t)r.nnz);
  if (n)
    LAUNCH(c, add_fill, blocks_for(n, 256), 256, 0, n, alpha, a.rp.p, a.ci.p, a.v.p, beta, b.rp.p, b.ci.p, b.v.p,
           r.rp.p, r.ci.p, r.v.p);
  out = std::move(r);
}

}  // namespace

void build_fused_level(Ctx& c, Level& L, int64_t smooths) {
  const int n = L.a.n, nf = L.map.nf;
  // A_F P: A's F rows (global columns, C flags cleared) times the one-point P
  Csr afp;
  {
    Csr af;
    af.n = L.af.n;
    af.m = n;
    af.nnz = L.af.nnz;
    af.rp.alloc(c, (size_t)af.n + 1);
    af.ci.alloc(c, (size_t)af.nnz);
    af.v.alloc(c, (size_t)af.nnz);
    CUDA_CHECK(cudaMemcpyAsync(af.rp.p, L.af.rp.p, sizeof(int32_t) * (af.n + 1), cudaMemcpyDeviceToDevice, c.stream));
    if (af.nnz) {
      CUDA_CHECK(cudaMemcpyAsync(af.v.p, L.af.v.p, sizeof(double) * af.nnz, cudaMemcpyDeviceToDevice, c.stream));
      LAUNCH(c, k_unflag_cols, blocks_for(af.nnz, 256), 256, 0, af.nnz, L.af.ci.p, af.ci.p);
    }
    spgemm(c, af, L.p, afp);
  }
  // W_k by the recurrence W_{k+1} = Q + W_k - (W_k A_ff) Q
  Csr w;
  if (smooths >= 1) {
    csr_add(c, 1.0, L.ffinv, 0.0, L.ffinv, w);  // W_1 = Q (a copy)
    for (int64_t s = 1; s < smooths; ++s) {
      Csr wa, waq, qw, next;
      spgemm(c, w, L.aff, wa);
      spgemm(c, wa, L.ffinv, waq);
      csr_add(c, 1.0, L.ffinv, 1.0, w, qw);
      csr_add(c, 1.0, qw, -1.0, waq, next);
      w = std::move(next);
    }
  }
  if (smooths < 1) {  // no F-smooth: x = P e_c only (an empty W)
    w.n = w.m = nf;
    w.nnz = 0;
    w.rp.alloc(c, (size_t)nf + 1);
    CUDA_CHECK(cudaMemsetAsync(w.rp.p, 0, sizeof(int32_t) * (nf + 1), c.stream));
  }
  L.afp = std::move(afp);
  L.fw = std::move(w);
}

void build_fused(Ctx& c, Hier& h, int64_t smooths) {
  if (smooths < 0) throw InvalidArgument("fast V-cycle: up_f_smooths must be >= 0");
  if (h.fused_smooths == smooths) return;
  for (Level& L : h.levels) build_fused_level(c, L, smooths);
  h.fused_smooths = smooths;
  ++h.fused_gen;
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

}  // namespace airg
