// AIRG hierarchy construction on the GPU (reference: proj/src/air.cpp:285-434).
// Host code orchestrates; every matrix operation is a device kernel (no CPU
// fallback). The level loop reads back only scalars (counts, norms, growth)
// to take the reference's data-dependent branches.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <thread>

#include "dist.cuh"
#include "hier.cuh"
#include "rowsplit.cuh"
#include "tiled.cuh"

namespace airg {

namespace {

// AIRG_CF=legacy: the setup's split as strength -> pmisr -> extract -> ddc
// kernels with S materialised (the reference's structure; same labels)
bool fused_cf_enabled() {
  static const bool v = [] {
    const char* e = getenv("AIRG_CF");
    return !(e && !strcmp(e, "legacy"));
  }();
  return v;
}

// AIRG_SETUP_TIMING=1 (diagnostic): per-phase wall times of the level loop,
// synchronised at each phase boundary, printed at the end of the setup
struct PhaseClock {
  bool on;
  Ctx& c;
  std::chrono::steady_clock::time_point t;
  double acc[8] = {};
  explicit PhaseClock(Ctx& c_) : c(c_) {
    const char* e = getenv("AIRG_SETUP_TIMING");
    on = e && e[0] == '1';
    if (on) {
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
      t = std::chrono::steady_clock::now();
    }
  }
  void lap(int k) {
    if (!on) return;
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    const auto n = std::chrono::steady_clock::now();
    acc[k] += std::chrono::duration<double, std::milli>(n - t).count();
    t = n;
  }
  void report() const {
    if (!on) return;
    fprintf(stderr, "setup phases ms: cf %.2f | inverse %.2f | R %.2f | P %.2f | RAP %.2f | coarse %.2f | fused %.2f\n",
            acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6]);
  }
};

struct Checked {
  std::vector<double> coeffs;
  int64_t eff = 0;
  Csr q;
  double growth = 0.0;
  int64_t attempts = 1;
  bool valid = false;
};

// make_checked_inverse (air.cpp:106-129): up to 6 seeded fits, keep the
// least-growing, stop once growth <= 0.5. The fits are independent (each
// its own seed, all of the same A_ff), and each is a chain of short
// latency-bound launches with two readbacks: when the first one fails the
// guard, the five retries are enqueued SIDE BY SIDE by five host threads on
// five worker streams and then walked in the reference's order with its
// stopping rule -- the same fit is kept, bit for bit (a retry the reference
// would not have reached is computed and dropped). C4: the growth guard
// rejects the first fit on levels 0-7, 48 of the setup's 63 fits.
Checked make_checked_inverse(Ctx& c, const Csr& a, int64_t order, int64_t sparsity,
                             uint64_t seed, const RowSplit* rs) {
  Checked best;
  double best_growth = INFINITY;
  auto seed_of = [&](int64_t attempt) {
    return attempt == 0 ? seed : mix_host(seed, 0x52455452ull + (uint64_t)attempt);
  };
  auto take = [&](PolyFit& fit, Csr& q, double growth, int64_t attempt) {
    if (growth < best_growth) {
      best.coeffs = fit.coeffs;
      best.eff = fit.effective_order;
      best.q = std::move(q);
      best.growth = growth;
      best.attempts = attempt + 1;
      best.valid = true;
      best_growth = growth;
    }
  };
  const bool side_by_side = !rs && setup_parallel(1);
  for (int64_t attempt = 0; attempt < (side_by_side ? 1 : 6); ++attempt) {
    PolyFit fit = poly_coefficients(c, a, order + 1, seed_of(attempt), rs);
    Csr q;
    poly_assemble(c, a, fit.coeffs.data(), (int64_t)fit.coeffs.size(), fit.effective_order,
                  sparsity, q, rs);
    const double growth = smoother_growth(c, a, q, rs);
    take(fit, q, growth, attempt);
    if (best_growth <= 0.5) break;
  }
  if (!side_by_side || best_growth <= 0.5) return best;

  constexpr int kRetries = 5;
  struct Retry {
    PolyFit fit;
    Csr q;
    double growth = 0.0;
    std::exception_ptr err;
  };
  Ctx* w = ctx_workers(c, kRetries);
  CUDA_CHECK(cudaStreamSynchronize(c.stream));  // A_ff complete before the workers read it
  Retry rt[kRetries];
  std::thread th[kRetries];
  for (int k = 0; k < kRetries; ++k) {
    th[k] = std::thread([&, k] {
      try {
        Ctx& wc = w[k];
        CUDA_CHECK(cudaSetDevice(wc.device));
        rt[k].fit = poly_coefficients(wc, a, order + 1, seed_of(k + 1), nullptr);
        poly_assemble(wc, a, rt[k].fit.coeffs.data(), (int64_t)rt[k].fit.coeffs.size(),
                      rt[k].fit.effective_order, sparsity, rt[k].q, nullptr);
        rt[k].growth = smoother_growth(wc, a, rt[k].q, nullptr);
        CUDA_CHECK(cudaStreamSynchronize(wc.stream));
      } catch (...) {
        rt[k].err = std::current_exception();
      }
    });
  }
  for (int k = 0; k < kRetries; ++k) th[k].join();
  for (int k = 0; k < kRetries; ++k) {
    c.launches += w[k].launches;
    w[k].launches = 0;
  }
  for (int k = 0; k < kRetries; ++k) {  // the reference's walk over attempts 1..5
    if (rt[k].err) std::rethrow_exception(rt[k].err);
    // a kept inverse is released on the context's stream (its worker stream is idle)
    rt[k].q.rp.s = rt[k].q.ci.s = rt[k].q.v.s = c.stream;
    take(rt[k].fit, rt[k].q, rt[k].growth, k + 1);
    if (best_growth <= 0.5) break;
  }
  return best;
}

Checked injected_inverse(Ctx& c, const Csr& a, const std::vector<double>& coeffs, int64_t eff,
                         int64_t sparsity, const RowSplit* rs) {
  Checked k;
  k.coeffs = coeffs;
  k.eff = eff;
  poly_assemble(c, a, coeffs.data(), (int64_t)coeffs.size(), eff, sparsity, k.q, rs);
  k.valid = true;
  return k;
}

}  // namespace

CheckedInverse checked_inverse(Ctx& c, const Csr& a, int64_t order, int64_t sparsity, uint64_t seed) {
  Checked k = make_checked_inverse(c, a, order, sparsity, seed, nullptr);
  CheckedInverse o;
  o.coeffs = k.coeffs;
  o.eff = k.eff;
  o.attempts = k.attempts;
  o.growth = k.growth;
  o.q = std::move(k.q);
  return o;
}
CheckedInverse fixed_inverse(Ctx& c, const Csr& a, const std::vector<double>& coeffs, int64_t eff,
                             int64_t sparsity) {
  Checked k = injected_inverse(c, a, coeffs, eff, sparsity, nullptr);
  CheckedInverse o;
  o.coeffs = k.coeffs;
  o.eff = k.eff;
  o.q = std::move(k.q);
  return o;
}

// Solve-side structures: A_FF with global columns and the per-level vectors
// (fixed pointers, so the V-cycle can be captured into a CUDA graph).
void alloc_workspace(Ctx& c, Hier& h) {
  for (size_t l = 0; l < h.levels.size(); ++l) {
    Level& L = h.levels[l];
    if (l > 0) L.b.alloc(c, (size_t)L.a.n);
    L.x.alloc(c, (size_t)L.a.n);
    L.rf.alloc(c, (size_t)std::max(1, L.map.nf));
    L.sc.alloc(c, (size_t)std::max(1, L.map.nf));
    map_columns(c, L.aff, L.map.f_to_fine.p, L.a.n, L.affg);
  }
  Csr& top = h.levels.empty() ? h.coarse_a : h.levels.front().a;
  const size_t nc = (size_t)std::max(1, h.coarse_a.n);
  h.cb.alloc(c, nc);
  h.cx.alloc(c, nc);
  h.cr.alloc(c, nc);
  const size_t n = (size_t)std::max(1, h.top_n());
  h.rhs.alloc(c, n);
  h.xsol.alloc(c, n);
  h.r.alloc(c, n);
  // one partial per residual block for any decomposition (tiled.cuh rows_grid:
  // up to 32 lanes per row in the group kernels)
  h.part.alloc(c, (size_t)(kReduceBlocks + (int64_t)top.n * 32 / kTileThreads + 8));
  h.scal.alloc(c, 64);
}

void recompute_metrics(Hier& h) {
  const Csr& top = h.top();
  const double n0 = (double)top.n, nnz0 = (double)top.nnz;
  double grid = 0.0, op = 0.0, store = 0.0;
  for (const Level& L : h.levels) {
    grid += (double)L.a.n;
    op += (double)L.a.nnz;
    store += (double)(L.ffinv.nnz + L.aff.nnz + L.afc.nnz + L.r.nnz + L.p.nnz);
  }
  grid += (double)h.coarse_a.n;
  op += (double)h.coarse_a.nnz;
  store += (double)h.coarse_inv.nnz;
  if (h.coarse_iterations > 1) store += (double)h.coarse_a.nnz;
  h.grid_c = grid / n0;
  h.op_c = op / nnz0;
  h.store_c = store / nnz0;
}

void setup(Ctx& c, const Csr& a0, const airg_setup_config& cfg, const Injection* inj, Hier& h,
           const RowSplit* rs) {
  NvtxRange nvtx__("airg setup");
  if (a0.n != a0.m) throw InvalidArgument("setup: matrix must be square");
  if (cfg.poly_order < 1 || cfg.coarse_poly_order < 1)
    throw InvalidArgument("setup: polynomial orders must be >= 1");
  if (cfg.sparsity_order < 1) throw InvalidArgument("setup: sparsity_order must be >= 1");
  if (cfg.drop_coarse < 0.0 || cfg.drop_restrict < 0.0)
    throw InvalidArgument("setup: drop tolerances must be >= 0");
  if (cfg.strength_alpha < 0.0 || cfg.strength_alpha > 1.0)
    throw InvalidArgument("setup: strength_alpha must lie in [0, 1]");
  if (cfg.cf < 0 || cfg.cf > 2) throw InvalidArgument("setup: cf must be pmisr (0), pmis (1) or pmis-swap (2)");
  if (cfg.prolongation != 0)
    throw InvalidArgument("setup: the GPU path implements one-point prolongation only");
  if (cfg.poly_order + 1 > 32 || cfg.coarse_poly_order + 1 > 32)
    throw InvalidArgument("setup: polynomial order above 31 not supported");
  h.levels.clear();
  h.coarse_iterations = cfg.coarse_iterations;
  constexpr double kCoarseAccept = 0.5;
  Checked coarse;
  Csr current;
  PhaseClock pc(c);
  with_full_diagonal(c, a0, current);  // air.cpp:307
  for (;;) {
    const int64_t built = (int64_t)h.levels.size();
    const bool forced = current.n <= cfg.poly_order + 1 ||
                        (cfg.max_levels > 0 && built + 1 >= cfg.max_levels);
    if (inj) {
      if (built >= inj->n_levels) {
        coarse = injected_inverse(c, current, inj->coarse_coeffs, inj->coarse_eff, cfg.sparsity_order, rs);
        break;
      }
    } else if (forced || current.n <= cfg.coarse_size_target) {  // air.cpp:309-320
      pc.lap(4);
      coarse = make_checked_inverse(c, current, cfg.coarse_poly_order, cfg.sparsity_order,
                                    mix_host(cfg.seed, 0xC0A12534ull + (uint64_t)built), rs);
      pc.lap(5);
      if (forced || coarse.growth <= kCoarseAccept) break;
      coarse = Checked();
    }
    h.levels.emplace_back();
    Level& L = h.levels.back();
    L.a = std::move(current);
    const int32_t n = L.a.n;
    const uint64_t level_seed = mix_host(cfg.seed, (uint64_t)built);  // air.cpp:324-325

    // --- CF split: strength -> PMISR -> extract -> DDC (air.cpp:327-355)
    Strength g;
    DBuf<uint8_t> labels(c, (size_t)n);
    Blocks blk;
    // the default PMISR-DDC split runs as the fused, sync-free split of the
    // CF-split metric (cfsplit.cu, labels bit-identical to the step-by-step
    // split); S is never materialised (P re-applies the strength test)
    const bool fused_cf = !rs && cfg.cf == 0 && cfg.weight_mode == 0 && fused_cf_enabled();
    if (!fused_cf) strength(c, L.a, cfg.strength_alpha, g);
    if (fused_cf) {
      const CfFused rep = cf_split_fused(c, L.a, cfg.strength_alpha, level_seed, cfg.ddc_enabled != 0,
                                         cfg.ddc_fraction, cfg.ddc_bins, labels.p, nullptr);
      build_label_map(c, labels.p, n, L.map);
      L.n_f_pre = rep.n_f_pre;
      L.n_converted = rep.n_converted;
      L.alpha_diag = rep.alpha_diag;
      L.max_theta_pre = rep.max_theta;
    } else if (rs && cfg.cf == 0 && cfg.weight_mode == 0 && (cfg.ddc_enabled == 0 || cfg.ddc_fraction > 0.0)) {
      // row slabs over the ranks (dist.cu): the labels, all-gathered
      const std::vector<int64_t> sl = rs->slabs(n);
      CfReport rep;
      uint8_t* mine = rs->me < 0 ? labels.p : labels.p + sl[rs->me];
      dist_cf_split(c, L.a, rs->P, rs->me, rs->comm, sl, cfg.strength_alpha, cfg.max_loops, level_seed,
                    cfg.ddc_enabled != 0, cfg.ddc_fraction, cfg.ddc_bins, mine, rep);
      rs->gather_vec(c, labels.p, sl);
      build_label_map(c, labels.p, n, L.map);
      L.n_f_pre = rep.n_f_pre;
      L.n_converted = rep.n_converted;
      L.alpha_diag = rep.alpha_diag;
      L.max_theta_pre = rep.max_theta;
      if (!cfg.ddc_enabled && L.map.nf > 0) {
        extract_blocks(c, L.a, L.map, blk, /*want_af=*/false);
        L.max_theta_pre = dominance_max(c, blk.aff);
      }
    } else {
      if (cfg.cf == 0)  // air.cpp:328-338
        pmisr(c, g, cfg.max_loops, level_seed, cfg.weight_mode, labels.p, nullptr);
      else
        pmis(c, g, cfg.cf == 2, level_seed, labels.p);
      build_label_map(c, labels.p, n, L.map);
      L.n_f_pre = L.map.nf;
      extract_blocks(c, L.a, L.map, blk, /*want_af=*/false);
      if (cfg.ddc_enabled && L.map.nf > 0) {
        DdcResult res = ddc(c, blk.aff, L.map, labels.p, cfg.ddc_fraction, cfg.ddc_bins, 0, 0.0, true);
        L.max_theta_pre = res.max_theta;
        L.alpha_diag = res.alpha_diag;
        L.n_converted = res.converted;
        if (res.converted > 0) build_label_map(c, labels.p, n, L.map);
      } else {
        L.max_theta_pre = dominance_max(c, blk.aff);
      }
    }
    extract_blocks(c, L.a, L.map, blk, /*want_af=*/true);
    L.max_theta_post = dominance_max(c, blk.aff);
    if (fused_cf && !cfg.ddc_enabled) L.max_theta_pre = L.max_theta_post;  // no DDC: the same A_ff
    L.aff = std::move(blk.aff);
    L.afc = std::move(blk.afc);
    L.acf = std::move(blk.acf);
    L.af = std::move(blk.af);

    // --- stall guards (air.cpp:362-376)
    const int32_t nc = L.map.nc;
    if (L.map.nf == 0)
      throw RuntimeError("setup: coarsening stall, no F points selected on level " +
                         std::to_string(built));
    if (nc == 0) {
      current = std::move(L.a);
      h.levels.pop_back();
      break;
    }
    if ((double)nc > 0.99 * (double)n)
      throw RuntimeError("setup: coarsening stall, level " + std::to_string(built) +
                         " coarsened by less than 1% (" + std::to_string(n) + " -> " +
                         std::to_string(nc) + ")");

    pc.lap(0);
    // P and A P need the labels and A only, not the inverse: a host thread
    // enqueues them on a worker stream (context 5; 0-4 are the retry fits')
    // while this one fits A_ff^-1 and builds R. Same products, same bits.
    Csr ap, rap;
    const bool side_p = fused_cf && !pc.on && setup_parallel(4);
    std::thread p_thread;
    std::exception_ptr p_err;
    Ctx* pw = nullptr;
    if (side_p) {
      pw = ctx_workers(c, 6) + 5;
      CUDA_CHECK(cudaStreamSynchronize(c.stream));  // A, the map and the blocks complete
      p_thread = std::thread([&] {
        try {
          CUDA_CHECK(cudaSetDevice(pw->device));
          build_prolongation_fused(*pw, L.map, L.a, cfg.strength_alpha, L.pmap, L.p);
          spgemm(*pw, L.a, L.p, ap);
          CUDA_CHECK(cudaStreamSynchronize(pw->stream));
        } catch (...) {
          p_err = std::current_exception();
        }
      });
    }
    struct Joiner {  // an exception on this thread still joins the other
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{p_thread};
    // --- approximate ideal restriction (air.cpp:378-381)
    Checked ff = inj ? injected_inverse(c, L.aff, inj->level_coeffs[built], inj->level_eff[built],
                                        cfg.sparsity_order, rs)
                     : make_checked_inverse(c, L.aff, cfg.poly_order, cfg.sparsity_order, level_seed, rs);
    L.ffinv = std::move(ff.q);
    L.coeffs = ff.coeffs;
    L.eff = ff.eff;
    L.growth = ff.growth;
    L.attempts = ff.attempts;
    pc.lap(1);
    build_restriction(c, L.acf, L.ffinv, cfg.drop_restrict, L.map, L.r, nullptr, 0, rs);
    pc.lap(2);
    if (side_p) {
      p_thread.join();
      c.launches += pw->launches;
      pw->launches = 0;
      if (p_err) std::rethrow_exception(p_err);
      // kept operators are released on the context's stream
      L.pmap.s = L.p.rp.s = L.p.ci.s = L.p.v.s = c.stream;
      ap.rp.s = ap.ci.s = ap.v.s = c.stream;
    } else if (fused_cf) {
      build_prolongation_fused(c, L.map, L.a, cfg.strength_alpha, L.pmap, L.p);
    } else {
      build_prolongation(c, L.map, g, L.a, L.pmap, L.p);
    }
    pc.lap(3);

    // --- Galerkin coarse operator (air.cpp:268-271, :386-387)
    if (rs) {  // row slabs over the ranks, gathered (rowsplit.cuh)
      split_spgemm(c, *rs, L.a, L.p, ap, -1.0, true);
      split_spgemm(c, *rs, L.r, ap, rap, cfg.drop_coarse, /*keep_diag=*/true);
    } else {
      if (!side_p) spgemm(c, L.a, L.p, ap);
      spgemm(c, L.r, ap, rap, cfg.drop_coarse, /*keep_diag=*/true);
    }
    with_full_diagonal(c, rap, current);
    pc.lap(4);
  }
  h.coarse_a = std::move(current);
  if (!coarse.valid) {
    // reached only through the all-F break (air.cpp:538-543)
    if (inj)
      coarse = injected_inverse(c, h.coarse_a, inj->coarse_coeffs, inj->coarse_eff, cfg.sparsity_order, rs);
    else
      coarse = make_checked_inverse(c, h.coarse_a, cfg.coarse_poly_order, cfg.sparsity_order,
                                    mix_host(cfg.seed, 0xC0A12534ull + (uint64_t)h.levels.size()), rs);
  }
  h.coarse_inv = std::move(coarse.q);
  h.coarse_coeffs = coarse.coeffs;
  h.coarse_eff = coarse.eff;
  h.coarse_attempts = coarse.attempts;
  h.coarse_growth = coarse.growth;
  recompute_metrics(h);
  alloc_workspace(c, h);
  pc.lap(4);
  if (cfg.fused_smooths >= 0) build_fused(c, h, cfg.fused_smooths, cfg.coarse_iterations);
  pc.lap(6);
  pc.report();
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// A device hierarchy from given level operators (the C++ airgraph:: shim
// hands the GPU solve a host airgraph::Hierarchy): per level A, A_ff, A_fc,
// A_cf, Aff^-1, R, P (one-point: <= 1 entry of 1.0 per row) and the labels;
// the coarse operator and its assembled inverse. Vector workspace as setup.
void hier_from_levels(Ctx& c, std::vector<HostLevel>& in, Csr&& coarse_a, Csr&& coarse_inv,
                      int64_t coarse_iterations, Hier& h) {
  h.levels.clear();
  h.coarse_iterations = coarse_iterations;
  for (HostLevel& hl : in) {
    h.levels.emplace_back();
    Level& L = h.levels.back();
    L.a = std::move(hl.a);
    if (L.a.n != L.a.m) throw InvalidArgument("vcycle: level operators must be square");
    build_label_map(c, hl.labels, L.a.n, L.map);
    Blocks blk;
    extract_blocks(c, L.a, L.map, blk, /*want_af=*/true);
    L.af = std::move(blk.af);
    L.aff = std::move(hl.aff);
    L.afc = std::move(hl.afc);
    L.acf = std::move(hl.acf);
    L.ffinv = std::move(hl.ffinv);
    L.r = std::move(hl.r);
    L.p = std::move(hl.p);
    if (L.aff.n != L.map.nf || L.ffinv.n != L.map.nf)
      throw InvalidArgument("vcycle: level blocks do not match the labels");
    // R and P may be absent (0 x 0) on a level built only for F-smoothing
    if ((L.r.n || L.r.m) && L.r.m != L.a.n) throw InvalidArgument("vcycle: R does not match the level");
    if ((L.p.n || L.p.m) && L.p.n != L.a.n) throw InvalidArgument("vcycle: P does not match the level");
    // one-point P -> map (-1 = empty row)
    L.pmap.alloc(c, (size_t)std::max(1, L.a.n));
    std::vector<int32_t> prp(L.p.n + 1), pci(L.p.nnz);
    std::vector<double> pv(L.p.nnz);
    to_host(c, prp.data(), L.p.rp.p, prp.size());
    to_host(c, pci.data(), L.p.ci.p, pci.size());
    to_host(c, pv.data(), L.p.v.p, pv.size());
    std::vector<int32_t> pm(L.a.n, -1);
    for (int i = 0; i < L.p.n; ++i) {
      const int k0 = prp[i], k1 = prp[i + 1];
      if (k1 - k0 > 1 || (k1 > k0 && pv[k0] != 1.0))
        throw InvalidArgument("vcycle: the GPU V-cycle takes one-point prolongation only");
      if (k1 > k0) pm[i] = pci[k0];
    }
    if (L.a.n) to_device(c, L.pmap.p, pm.data(), pm.size());
  }
  h.coarse_a = std::move(coarse_a);
  h.coarse_inv = std::move(coarse_inv);
  recompute_metrics(h);
  alloc_workspace(c, h);
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

}  // namespace airg
