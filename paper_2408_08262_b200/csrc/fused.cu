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
#include <chrono>
#include <cstdio>

#include <atomic>
#include <exception>
#include <thread>
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

void csr_add_impl(Ctx& c, double alpha, const Csr& a, double beta, const Csr& b, Csr& out) {
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


// one-point map of the F rows: pmap of the F point's fine index
__global__ void k_pf_map(int nf, const int32_t* __restrict__ f2f, const int32_t* __restrict__ pmap,
                         int32_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nf) out[k] = pmap[f2f[k]];
}
// [top; bottom] row offsets (same column space)
__global__ void k_vstack_rp(int nt, int nb, int64_t nnz_t, const int32_t* __restrict__ trp,
                            const int32_t* __restrict__ brp, int32_t* __restrict__ rp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nt) rp[i] = trp[i];
  else if (i <= nt + nb) rp[i] = (int32_t)nnz_t + brp[i - nt];
}

void csr_vstack(Ctx& c, const Csr& t, const Csr& b, Csr& out) {
  if (t.m != b.m) throw InvalidArgument("csr_vstack: column spaces differ");
  out.alloc(c, (int64_t)t.n + b.n, t.m, t.nnz + b.nnz);
  LAUNCH(c, k_vstack_rp, blocks_for((int64_t)t.n + b.n + 1, 256), 256, 0, t.n, b.n, t.nnz, t.rp.p, b.rp.p,
         out.rp.p);
  if (t.nnz) {
    CUDA_CHECK(cudaMemcpyAsync(out.ci.p, t.ci.p, sizeof(int32_t) * t.nnz, cudaMemcpyDeviceToDevice, c.stream));
    CUDA_CHECK(cudaMemcpyAsync(out.v.p, t.v.p, sizeof(double) * t.nnz, cudaMemcpyDeviceToDevice, c.stream));
  }
  if (b.nnz) {
    CUDA_CHECK(cudaMemcpyAsync(out.ci.p + t.nnz, b.ci.p, sizeof(int32_t) * b.nnz, cudaMemcpyDeviceToDevice,
                               c.stream));
    CUDA_CHECK(cudaMemcpyAsync(out.v.p + t.nnz, b.v.p, sizeof(double) * b.nnz, cudaMemcpyDeviceToDevice,
                               c.stream));
  }
}

// products of A B (sum over A's entries of the B row length): the SpGEMM's
// work, one block atomic
__global__ void k_products(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                           const int32_t* __restrict__ brp, unsigned long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long s = 0;
  if (i < n)
    for (int k = arp[i]; k < arp[i + 1]; ++k) s += (unsigned long long)(brp[aci[k] + 1] - brp[aci[k]]);
  block_add(out, s);
}

int64_t products(Ctx& c, const Csr& a, const Csr& b) {
  if (a.n == 0) return 0;
  DBuf<unsigned long long> d(c, 1);
  CUDA_CHECK(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), c.stream));
  LAUNCH(c, k_products, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, b.rp.p, d.p);
  unsigned long long h = 0;
  to_host(c, &h, d.p, 1);
  return (int64_t)h;
}

int64_t env_entries(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return (e && e[0]) ? atoll(e) : dflt;
}

}  // namespace

void csr_add(Ctx& c, double alpha, const Csr& a, double beta, const Csr& b, Csr& out) {
  csr_add_impl(c, alpha, a, beta, b, out);
}

void build_fused_level(Ctx& c, Level& L, int64_t smooths) {
  const int n = L.a.n, nf = L.map.nf, nc = L.map.nc;
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
  // One-pass ascent. With y = W_k b_F formed on the way DOWN (b_l is known
  // there: [b_{l+1}; y] = [R; W_k E_F^T] b_l in the restriction's launch),
  //   x_F = (P e_c)_F + W_k (b_F - A_F P e_c) = y + K e_c,  K = P_F - W_k A_F P,
  // so the ascent of the level is ONE row pass over K instead of two
  // dependent passes (A_F P, then W_k). It moves nnz(K) - nnz(A_F P) more
  // entries and saves one dependent launch and the r1 round trip: taken when
  // the extra entries stay under AIRG_ONEPASS_EXTRA (default 250 k; C4:
  // level 0, where K is 1.1x A_F P; measured per level in
  // profiles/r2_onepass_levels.txt: level 0's ascent 30 -> 17-20 us, the
  // descent's added W b_F about half of that back).
  L.one_pass = false;
  L.fk = Csr();
  L.dsc = Csr();
  const int64_t extra_max = env_entries("AIRG_ONEPASS_EXTRA", 250000);
  // K is formed only where W A_F P averages at most AIRG_ONEPASS_ROWWORK
  // products per row (default 16): on C4 level 0 (3.8 per row, 0.5 ms of
  // setup); the coarse levels' rows take 90-950 products (6-28 ms of SpGEMM
  // per level for about 1 us per V-cycle on levels 15-18, and K 5-13x A_F P
  // on the mid levels)
  const int64_t row_work = env_entries("AIRG_ONEPASS_ROWWORK", 16);
  if (extra_max >= 0 && nf > 0 && products(c, w, afp) <= row_work * (int64_t)nf) {
    Csr wafp, pf, k;
    spgemm(c, w, afp, wafp);
    {
      DBuf<int32_t> pfm(c, (size_t)nf);
      LAUNCH(c, k_pf_map, blocks_for(nf, 256), 256, 0, nf, L.map.f_to_fine.p, L.pmap.p, pfm.p);
      prolongation_from_map(c, pfm.p, nf, nc, pf);
    }
    csr_add(c, 1.0, pf, -1.0, wafp, k);
    if (k.nnz - afp.nnz <= extra_max) {
      Csr wg;
      map_columns(c, w, L.map.f_to_fine.p, n, wg);
      csr_vstack(c, L.r, wg, L.dsc);
      L.fk = std::move(k);
      L.one_pass = true;
    }
  }
  L.afp = std::move(afp);
  L.fw = std::move(w);
}

// The coarse solve (solve.cpp:34-59) from e = 0 is linear in the coarse rhs:
// e_k = E_k b with E_1 = Q, E_{k+1} = Q + E_k - Q A E_k. Composed when
// nnz(E_k) <= AIRG_COARSE_COMPOSE entries: one row pass instead of 2k - 1
// dependent ones (C4: 280 k entries for k = 3 instead of five launches over
// 57 k-entry operators).
bool compose_coarse(Ctx& c, const Csr& a, const Csr& q, int64_t its, Csr& out) {
  out = Csr();
  const int64_t cap = env_entries("AIRG_COARSE_COMPOSE", 4000000);
  if (its < 1 || a.n == 0 || cap <= 0 || a.n > 50000 || a.n != a.m || q.n != a.n || q.m != a.n) return false;
  Csr e;
  csr_add(c, 1.0, q, 0.0, q, e);
  for (int64_t k = 1; k < its; ++k) {
    Csr ae, qae, qe, next;
    spgemm(c, a, e, ae);
    spgemm(c, q, ae, qae);
    csr_add(c, 1.0, q, 1.0, e, qe);
    csr_add(c, 1.0, qe, -1.0, qae, next);
    e = std::move(next);
    if (e.nnz > cap) return false;
  }
  if (e.nnz > cap) return false;
  out = std::move(e);
  return true;
}

void build_coarse_composed(Ctx& c, Hier& h, int64_t its) {
  h.coarse_composed = compose_coarse(c, h.coarse_a, h.coarse_inv, its, h.coarse_e);
}

void build_fused(Ctx& c, Hier& h, int64_t smooths, int64_t coarse_its) {
  NvtxRange nvtx__("airg fused operators");
  if (smooths < 0) throw InvalidArgument("fast V-cycle: up_f_smooths must be >= 0");
  if (fused_ready(h, smooths, coarse_its)) return;
  const char* te = getenv("AIRG_SETUP_TIMING");
  const bool timing = te && te[0] == '1';
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what, int64_t l) {
    if (!timing) return;
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "fused %s %lld: %.2f ms\n", what, (long long)l,
            std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const bool do_levels = h.fused_smooths != smooths, do_coarse = h.fused_coarse_its != coarse_its;
  const int64_t n_tasks = (do_levels ? (int64_t)h.levels.size() : 0) + (do_coarse ? 1 : 0);
  if (!timing && setup_parallel(2) && n_tasks > 1) {
    // The levels' operators (and the composed coarse solve) are independent
    // of one another and each is a chain of short SpGEMM launches with
    // readbacks: host threads take them from a counter, finest level first,
    // each on its own worker stream. Same operators bit for bit.
    constexpr int kWorkers = 6;
    const int nw = (int)std::min<int64_t>(kWorkers, n_tasks);
    Ctx* w = ctx_workers(c, nw);
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    std::atomic<int64_t> next{0};
    std::vector<std::exception_ptr> err((size_t)nw);
    std::vector<std::thread> th;
    const int64_t n_lv = do_levels ? (int64_t)h.levels.size() : 0;
    for (int k = 0; k < nw; ++k) {
      th.emplace_back([&, k] {
        try {
          Ctx& wc = w[k];
          CUDA_CHECK(cudaSetDevice(wc.device));
          for (int64_t t = next.fetch_add(1); t < n_tasks; t = next.fetch_add(1)) {
            if (t < n_lv)
              build_fused_level(wc, h.levels[(size_t)t], smooths);
            else
              build_coarse_composed(wc, h, coarse_its);
          }
          CUDA_CHECK(cudaStreamSynchronize(wc.stream));
        } catch (...) {
          err[(size_t)k] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    for (int k = 0; k < nw; ++k) {
      c.launches += w[k].launches;
      w[k].launches = 0;
    }
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
    // the operators live on: released on the context's stream
    auto home = [&](Csr& m) { m.rp.s = m.ci.s = m.v.s = c.stream; };
    if (do_levels)
      for (Level& L : h.levels)
        for (Csr* m : {&L.afp, &L.fw, &L.fk, &L.dsc}) home(*m);
    if (do_coarse) home(h.coarse_e);
    if (do_levels) h.fused_smooths = smooths;
    if (do_coarse) h.fused_coarse_its = coarse_its;
  } else {
    if (do_levels) {
      for (size_t l = 0; l < h.levels.size(); ++l) {
        build_fused_level(c, h.levels[l], smooths);
        lap(h.levels[l].one_pass ? "level(one-pass)" : "level", (int64_t)l);
      }
      h.fused_smooths = smooths;
    }
    if (do_coarse) {
      build_coarse_composed(c, h, coarse_its);
      h.fused_coarse_its = coarse_its;
      lap("coarse", coarse_its);
    }
  }
  // the fast row kernels size their lane groups by the longest row (sparse.cu row_lanes)
  std::vector<Csr*> ms = {&h.coarse_a, &h.coarse_inv};
  if (h.coarse_composed) ms.push_back(&h.coarse_e);
  for (Level& L : h.levels) {
    for (Csr* m : {&L.r, &L.afp, &L.fw}) ms.push_back(m);
    if (L.one_pass) {
      ms.push_back(&L.fk);
      ms.push_back(&L.dsc);
    }
  }
  row_max(c, ms);
  ++h.fused_gen;
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

}  // namespace airg
