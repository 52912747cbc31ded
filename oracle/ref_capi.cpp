// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the UNMODIFIED reference library compiled
// from /root/reference/proj/src (see oracle/Makefile). It lets tests/ and
// bench.py (reference arm / cpu_baseline leg) call the reference's own
// airgraph:: entry points through ctypes with the same plain-pointer shapes
// as include/airg_c.h. Nothing here is product code; the product never
// loads oracle/_ref.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "airg_c.h"
#include "airgraph/air.hpp"
#include "airgraph/coarsening.hpp"
#include "airgraph/gmres_poly.hpp"
#include "airgraph/matrix_market.hpp"
#include "airgraph/partition_model.hpp"
#include "airgraph/reports.hpp"
#include "airgraph/solve.hpp"
#include "airgraph/sparse.hpp"
#include "airgraph/transport.hpp"

using namespace airgraph;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return AIRG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return AIRG_EINVAL;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return AIRG_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return AIRG_ELOGIC;
  }
}

SparseMatrix make(int64_t n, int64_t m, const int64_t* rp, const int64_t* ci,
                  const double* v) {
  std::vector<index_t> o(rp, rp + n + 1);
  std::vector<index_t> c(ci, ci + rp[n]);
  std::vector<double> x(v, v + rp[n]);
  return SparseMatrix(n, m, std::move(o), std::move(c), std::move(x));
}

SetupConfig to_cfg(const airg_setup_config* c) {
  SetupConfig s;
  s.strength_alpha = c->strength_alpha;
  s.cf = static_cast<CfSplitting>(c->cf);
  s.ddc_enabled = c->ddc_enabled != 0;
  s.ddc_fraction = c->ddc_fraction;
  s.ddc_bins = c->ddc_bins;
  s.max_loops = c->max_loops;
  s.poly_order = c->poly_order;
  s.sparsity_order = c->sparsity_order;
  s.drop_coarse = c->drop_coarse;
  s.drop_restrict = c->drop_restrict;
  s.coarse_size_target = c->coarse_size_target;
  s.coarse_poly_order = c->coarse_poly_order;
  s.coarse_iterations = c->coarse_iterations;
  s.max_levels = c->max_levels;
  s.prolongation = static_cast<ProlongationKind>(c->prolongation);
  s.weight_mode = static_cast<WeightMode>(c->weight_mode);
  s.seed = c->seed;
  return s;
}

SolveConfig to_scfg(const airg_solve_config* c) {
  SolveConfig s;
  s.rtol = c->rtol;
  s.max_iterations = c->max_iterations;
  s.up_f_smooths = c->up_f_smooths;
  s.down_smooths = c->down_smooths;
  s.coarse_iterations = c->coarse_iterations;
  s.collect_timing = c->collect_timing != 0;
  s.nddofs = c->nddofs;
  return s;
}

struct RefHier {
  Hierarchy h;
};

const SparseMatrix* level_matrix(const Hierarchy& h, int64_t l, int which) {
  const int64_t nl = static_cast<int64_t>(h.levels.size());
  if (l == nl) {
    if (which == 0) return &h.coarse_a;
    if (which == 4) return &*h.coarse_inv.assembled;
    throw std::invalid_argument("coarse level has only A (0) and inverse (4)");
  }
  if (l < 0 || l > nl) throw std::invalid_argument("level out of range");
  const Level& lv = h.levels[l];
  switch (which) {
    case 0: return &lv.a;
    case 1: return &lv.a_ff;
    case 2: return &lv.a_fc;
    case 3: return &lv.a_cf;
    case 4: return &*lv.ff_inv.assembled;
    case 5: return &lv.r;
    case 6: return &lv.p;
  }
  throw std::invalid_argument("bad matrix selector");
}

}  // namespace

extern "C" {

int ref_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return static_cast<int>(g_err.size());
}

// ---- generic matrix handles ------------------------------------------------
int ref_mat_new(int64_t n, int64_t m, const int64_t* rp, const int64_t* ci,
                const double* v, void** out) {
  return guard([&] { *out = new SparseMatrix(make(n, m, rp, ci, v)); });
}
int ref_mat_dims(const void* h, int64_t* n, int64_t* m, int64_t* nnz) {
  auto* a = static_cast<const SparseMatrix*>(h);
  *n = a->nrows();
  *m = a->ncols();
  *nnz = a->nnz();
  return AIRG_OK;
}
int ref_mat_copy(const void* h, int64_t* rp, int64_t* ci, double* v) {
  auto* a = static_cast<const SparseMatrix*>(h);
  std::memcpy(rp, a->row_offsets().data(), sizeof(int64_t) * (a->nrows() + 1));
  std::memcpy(ci, a->col_indices().data(), sizeof(int64_t) * a->nnz());
  std::memcpy(v, a->values().data(), sizeof(double) * a->nnz());
  return AIRG_OK;
}
int ref_mat_free(void* h) {
  delete static_cast<SparseMatrix*>(h);
  return AIRG_OK;
}
// matrix_market.hpp:11-19 (read / write a coordinate real general file)
int ref_mm_read(const char* path, void** out) {
  return guard([&] { *out = new SparseMatrix(read_matrix_market(path)); });
}
int ref_mm_write(const void* h, const char* path) {
  return guard([&] { write_matrix_market(*static_cast<const SparseMatrix*>(h), path); });
}

// ---- L0 -------------------------------------------------------------------
int ref_spmv(const void* a, const double* x, double* y) {
  return guard([&] {
    auto* m = static_cast<const SparseMatrix*>(a);
    auto r = spmv(*m, std::span<const double>(x, m->ncols()));
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}
int ref_spgemm(const void* a, const void* b, void** out) {
  return guard([&] {
    *out = new SparseMatrix(spgemm(*static_cast<const SparseMatrix*>(a),
                                   *static_cast<const SparseMatrix*>(b)));
  });
}
int ref_drop(const void* a, double tol, int keep_diag, void** out) {
  return guard([&] {
    *out = new SparseMatrix(
        drop_entries(*static_cast<const SparseMatrix*>(a), tol, keep_diag != 0));
  });
}
int ref_with_full_diagonal(const void* a, void** out) {
  return guard([&] {
    *out = new SparseMatrix(static_cast<const SparseMatrix*>(a)->with_full_diagonal());
  });
}
int ref_extract_blocks(const void* a, const uint8_t* labels, void** aff,
                       void** afc, void** acf) {
  return guard([&] {
    auto* m = static_cast<const SparseMatrix*>(a);
    std::vector<CfLabel> l(m->nrows());
    for (index_t i = 0; i < m->nrows(); ++i) l[i] = static_cast<CfLabel>(labels[i]);
    BlockSplit s = extract_blocks(*m, l);
    *aff = new SparseMatrix(std::move(s.a_ff));
    *afc = new SparseMatrix(std::move(s.a_fc));
    *acf = new SparseMatrix(std::move(s.a_cf));
  });
}

// ---- L1a: CF splitting ---------------------------------------------------------
int ref_strength(const void* a, double alpha, void** s_out, int64_t* st_nnz) {
  return guard([&] {
    StrengthGraph g = strength(*static_cast<const SparseMatrix*>(a), alpha);
    std::vector<double> ones(g.s_cols.size(), 1.0);
    *s_out = new SparseMatrix(g.n, g.n, g.s_offsets, g.s_cols, std::move(ones));
    if (st_nnz) *st_nnz = static_cast<int64_t>(g.st_cols.size());
  });
}
int ref_pmisr(const void* a, double alpha, int64_t max_loops, uint64_t seed,
              int32_t weight_mode, uint8_t* labels, double* weights) {
  return guard([&] {
    StrengthGraph g = strength(*static_cast<const SparseMatrix*>(a), alpha);
    CfLabels l = pmisr(g, max_loops, seed, static_cast<WeightMode>(weight_mode));
    for (index_t i = 0; i < g.n; ++i) labels[i] = static_cast<uint8_t>(l.label[i]);
    if (weights) std::memcpy(weights, l.weight.data(), sizeof(double) * g.n);
  });
}
int ref_pmisr_with_weights(const void* s_pattern, int64_t max_loops,
                           const double* w, uint8_t* labels) {
  return guard([&] {
    auto* s = static_cast<const SparseMatrix*>(s_pattern);
    std::vector<std::vector<index_t>> rows(s->nrows());
    for (index_t i = 0; i < s->nrows(); ++i) {
      auto c = s->row_cols(i);
      rows[i].assign(c.begin(), c.end());
    }
    StrengthGraph g = StrengthGraph::from_pattern(s->nrows(), rows);
    CfLabels l = pmisr_with_weights(g, max_loops,
                                    std::vector<double>(w, w + s->nrows()));
    for (index_t i = 0; i < g.n; ++i) labels[i] = static_cast<uint8_t>(l.label[i]);
  });
}
// strength -> pmisr -> extract_blocks -> ddc, exactly as air.cpp:466-494.
int ref_cf_split(const void* a, double alpha, int64_t max_loops, uint64_t seed,
                 int32_t weight_mode, int32_t ddc_enabled, double fraction,
                 int64_t bins, uint8_t* labels, uint8_t* labels_pre,
                 airg_cf_report* rep) {
  return guard([&] {
    auto* m = static_cast<const SparseMatrix*>(a);
    StrengthGraph g = strength(*m, alpha);
    CfLabels l = pmisr(g, max_loops, seed, static_cast<WeightMode>(weight_mode));
    if (labels_pre)
      for (index_t i = 0; i < g.n; ++i) labels_pre[i] = static_cast<uint8_t>(l.label[i]);
    BlockSplit split = extract_blocks(*m, l.label);
    std::memset(rep, 0, sizeof(*rep));
    rep->n_f_pre = split.map.n_f();
    rep->s_nnz = static_cast<int64_t>(g.s_cols.size());
    if (ddc_enabled && split.map.n_f() > 0) {
      DdcOptions opt;
      opt.fraction = fraction;
      opt.bins = bins;
      DdcResult res = ddc(split.a_ff, l, split.map, opt);
      rep->max_theta = res.report.max_theta;
      rep->alpha_diag = res.alpha_diag;
      rep->n_converted = static_cast<int64_t>(res.converted.size());
      if (!res.converted.empty()) l = std::move(res.labels);
    }
    index_t nf = 0;
    for (index_t i = 0; i < g.n; ++i) {
      labels[i] = static_cast<uint8_t>(l.label[i]);
      nf += l.label[i] == CfLabel::F;
    }
    rep->n_f = nf;
    rep->n_c = g.n - nf;
  });
}
int ref_ddc(const void* a, uint8_t* labels, double fraction, int64_t bins,
            int32_t selection, double direct_alpha, airg_cf_report* rep) {
  return guard([&] {
    auto* m = static_cast<const SparseMatrix*>(a);
    CfLabels l;
    l.label.resize(m->nrows());
    for (index_t i = 0; i < m->nrows(); ++i) l.label[i] = static_cast<CfLabel>(labels[i]);
    l.weight.assign(m->nrows(), 0.5);
    BlockSplit split = extract_blocks(*m, l.label);
    DdcOptions opt;
    opt.fraction = fraction;
    opt.bins = bins;
    opt.selection = static_cast<DdcSelection>(selection);
    opt.direct_alpha_diag = direct_alpha;
    DdcResult res = ddc(split.a_ff, l, split.map, opt);
    std::memset(rep, 0, sizeof(*rep));
    rep->n_f_pre = split.map.n_f();
    rep->max_theta = res.report.max_theta;
    rep->alpha_diag = res.alpha_diag;
    rep->n_converted = static_cast<int64_t>(res.converted.size());
    for (index_t i = 0; i < m->nrows(); ++i) labels[i] = static_cast<uint8_t>(res.labels.label[i]);
  });
}

// ---- L1b: polynomials ---------------------------------------------------------
int ref_poly_coefficients(const void* a, int64_t m, uint64_t seed,
                          double* coeffs, int64_t* eff) {
  return guard([&] {
    GmresPolynomial p = compute_coefficients(*static_cast<const SparseMatrix*>(a), m, seed);
    std::memcpy(coeffs, p.coefficients.data(), sizeof(double) * p.coefficients.size());
    *eff = p.effective_order;
  });
}
int ref_poly_assemble(const void* a, const double* coeffs, int64_t ncoeffs,
                      int64_t eff, int64_t s, void** out) {
  return guard([&] {
    GmresPolynomial p;
    p.order = ncoeffs - 1;
    p.coefficients.assign(coeffs, coeffs + ncoeffs);
    p.effective_order = eff;
    *out = new SparseMatrix(
        assemble_fixed_sparsity(*static_cast<const SparseMatrix*>(a), p, s));
  });
}

// ---- L2: setup ------------------------------------------------------------------
int ref_setup(const void* a, const airg_setup_config* cfg, void** out) {
  return guard([&] {
    auto* rh = new RefHier;
    try {
      rh->h = setup(*static_cast<const SparseMatrix*>(a), to_cfg(cfg));
    } catch (...) {
      delete rh;
      throw;
    }
    *out = rh;
  });
}
int ref_hier_free(void* h) {
  delete static_cast<RefHier*>(h);
  return AIRG_OK;
}
int ref_hier_info(const void* hp, airg_hier_info* info) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    std::memset(info, 0, sizeof(*info));
    info->n_levels = static_cast<int64_t>(h.levels.size());
    info->coarse_n = h.coarse_a.nrows();
    info->coarse_nnz = h.coarse_a.nnz();
    info->coarse_inv_nnz = h.coarse_inv.assembled ? h.coarse_inv.assembled->nnz() : 0;
    info->coarse_effective_order = h.coarse_inv.effective_order;
    info->coarse_growth = h.coarse_growth;
    for (size_t k = 0; k < h.coarse_inv.coefficients.size() && k < 32; ++k)
      info->coarse_coefficients[k] = h.coarse_inv.coefficients[k];
    info->grid_complexity = h.metrics.grid_complexity;
    info->operator_complexity = h.metrics.operator_complexity;
    info->storage_complexity = h.metrics.storage_complexity;
  });
}
// reports.hpp: hierarchy_report(h).dump() and csv_row(h, stats, ...) for the
// report-schema tests (the solve statistics come from the caller)
int ref_hier_report(const void* hp, char* out, int64_t cap, int64_t* len) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    const std::string js = hierarchy_report(h).dump();
    *len = static_cast<int64_t>(js.size());
    if (out && cap > 0) std::snprintf(out, (size_t)cap, "%s", js.c_str());
  });
}
int ref_csv_row(const void* hp, int64_t iterations, double work_units, int32_t converged, double final_relres,
                double alpha, const char* cf_name, uint64_t seed, char* out, int64_t cap) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    SolveStats st;
    st.iterations = iterations;
    st.work_units = work_units;
    st.converged = converged != 0;
    st.final_relative_residual = final_relres;
    const std::string row = csv_row(h, st, alpha, cf_name, seed);
    std::snprintf(out, (size_t)cap, "%s", row.c_str());
  });
}
// partition_report(replay_triggers(h, ranks, threshold)).dump() (reports.cpp:75-101,
// partition_model.cpp:77-112)
int ref_partition_report(const void* hp, int32_t ranks, double threshold, char* out, int64_t cap, int64_t* len) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    const std::string js = partition_report(replay_triggers(h, ranks, threshold)).dump();
    *len = static_cast<int64_t>(js.size());
    if (out && cap > 0) std::snprintf(out, (size_t)cap, "%s", js.c_str());
  });
}
int ref_csv_header(char* out, int64_t cap) {
  std::snprintf(out, (size_t)cap, "%s", csv_header().c_str());
  return AIRG_OK;
}
int ref_level_info(const void* hp, int64_t l, airg_level_info* info) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    if (l < 0 || l >= static_cast<int64_t>(h.levels.size()))
      throw std::invalid_argument("level out of range");
    const Level& lv = h.levels[l];
    std::memset(info, 0, sizeof(*info));
    info->n = lv.a.nrows();
    info->nnz = lv.a.nnz();
    info->n_f = lv.map.n_f();
    info->n_c = lv.map.n_c();
    info->ddc_converted = static_cast<int64_t>(lv.ddc_converted.size());
    info->n_f_pre = info->n_f + info->ddc_converted;
    info->nnz_ff = lv.a_ff.nnz();
    info->nnz_fc = lv.a_fc.nnz();
    info->nnz_cf = lv.a_cf.nnz();
    info->nnz_ffinv = lv.ff_inv.assembled->nnz();
    info->nnz_r = lv.r.nnz();
    info->nnz_p = lv.p.nnz();
    info->max_theta_pre = lv.theta_pre.max_theta;
    info->alpha_diag = lv.theta_pre.alpha_diag;
    info->max_theta_post = lv.theta_post.max_theta;
    info->smoother_growth = lv.smoother_growth;
    info->poly_attempts = lv.poly_attempts;
    info->effective_order = lv.ff_inv.effective_order;
    for (size_t k = 0; k < lv.ff_inv.coefficients.size() && k < 32; ++k)
      info->coefficients[k] = lv.ff_inv.coefficients[k];
  });
}
int ref_hier_matrix(const void* hp, int64_t l, int32_t which, const void** out) {
  return guard([&] {
    *out = level_matrix(static_cast<const RefHier*>(hp)->h, l, which);
  });
}
int ref_hier_labels(const void* hp, int64_t l, uint8_t* labels) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    const Level& lv = h.levels.at(l);
    for (size_t i = 0; i < lv.map.label.size(); ++i)
      labels[i] = static_cast<uint8_t>(lv.map.label[i]);
  });
}

// ---- single operations (dominance_report, label map, transfer operators,
// polynomial application, one F-smooth), each calling the reference itself
int ref_dominance_report(const void* aff, int64_t bins, double* theta, int64_t* hist, double* max_theta) {
  return guard([&] {
    DominanceReport r = dominance_report(*static_cast<const SparseMatrix*>(aff), bins);
    if (theta) std::memcpy(theta, r.theta.data(), sizeof(double) * r.theta.size());
    if (hist)
      for (size_t b = 0; b < r.histogram.size(); ++b) hist[b] = r.histogram[b];
    if (max_theta) *max_theta = r.max_theta;
  });
}
static std::vector<CfLabel> to_labels(const uint8_t* labels, int64_t n) {
  std::vector<CfLabel> l((size_t)n);
  for (int64_t i = 0; i < n; ++i) l[(size_t)i] = static_cast<CfLabel>(labels[i]);
  return l;
}
int ref_build_label_map(const uint8_t* labels, int64_t n, int64_t* fine_to_sub, int64_t* f_to_fine,
                        int64_t* c_to_fine, int64_t* n_f) {
  return guard([&] {
    const std::vector<CfLabel> l = to_labels(labels, n);
    LabelMap m = build_label_map(l);
    if (fine_to_sub) std::copy(m.fine_to_sub.begin(), m.fine_to_sub.end(), fine_to_sub);
    if (f_to_fine) std::copy(m.f_to_fine.begin(), m.f_to_fine.end(), f_to_fine);
    if (c_to_fine) std::copy(m.c_to_fine.begin(), m.c_to_fine.end(), c_to_fine);
    if (n_f) *n_f = m.n_f();
  });
}
int ref_build_restriction(const void* acf, const void* ffinv, double drop, const uint8_t* labels, int64_t n,
                          void** out) {
  return guard([&] {
    const std::vector<CfLabel> l = to_labels(labels, n);
    LabelMap m = build_label_map(l);
    *out = new SparseMatrix(build_restriction(*static_cast<const SparseMatrix*>(acf),
                                              *static_cast<const SparseMatrix*>(ffinv), drop, m));
  });
}
int ref_build_prolongation(const void* a, const void* s_pattern, const uint8_t* labels, void** out) {
  return guard([&] {
    auto* am = static_cast<const SparseMatrix*>(a);
    auto* s = static_cast<const SparseMatrix*>(s_pattern);
    std::vector<std::vector<index_t>> rows(s->nrows());
    for (index_t i = 0; i < s->nrows(); ++i) {
      auto c = s->row_cols(i);
      rows[i].assign(c.begin(), c.end());
    }
    StrengthGraph g = StrengthGraph::from_pattern(s->nrows(), rows);
    CfLabels cl;
    cl.label = to_labels(labels, am->nrows());
    cl.weight.assign(am->nrows(), 0.5);
    LabelMap m = build_label_map(cl.label);
    *out = new SparseMatrix(build_prolongation(cl, m, g, *am));
  });
}
int ref_coarse_matrix(const void* r, const void* a, const void* p, double drop, void** out) {
  return guard([&] {
    *out = new SparseMatrix(coarse_matrix(*static_cast<const SparseMatrix*>(r),
                                          *static_cast<const SparseMatrix*>(a),
                                          *static_cast<const SparseMatrix*>(p), drop));
  });
}
int ref_apply_polynomial(const void* a, const double* coeffs, int64_t ncoeffs, int64_t deg, const double* b,
                         double* y) {
  return guard([&] {
    auto* m = static_cast<const SparseMatrix*>(a);
    GmresPolynomial p;
    p.order = ncoeffs - 1;
    p.coefficients.assign(coeffs, coeffs + ncoeffs);
    p.effective_order = deg;
    auto r = apply_polynomial(*m, p, std::span<const double>(b, (size_t)m->ncols()));
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}
int ref_f_smooth(const void* hp, int64_t l, const double* b, double* x) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    const Level& lv = h.levels.at(l);
    const index_t n = lv.a.nrows();
    std::vector<double> xv(x, x + n);
    f_smooth(lv, std::span<const double>(b, (size_t)n), xv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}

// ---- L3: solve -------------------------------------------------------------------
int ref_vcycle(const void* hp, const airg_solve_config* cfg, const double* b,
               double* x) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    const index_t n = h.top().nrows();
    std::vector<double> x0(n, 0.0);
    auto r = vcycle(h, std::span<const double>(b, n), x0, to_scfg(cfg));
    std::memcpy(x, r.data(), sizeof(double) * n);
  });
}
// Outer right-preconditioned restarted GMRES (CGS2, Givens) around the
// reference's own vcycle() and spmv() (solve.hpp:51-54, sparse.hpp:97-98).
// NOT in the reference (Richardson only, solve.cpp:167-259); the same steps
// as orc_solve(outer = 1) in oracle/airg_oracle.c and the GPU's solve.cu, so
// the reference arm can run the systems on which Richardson diverges (C4).
static void ref_gmres(const Hierarchy& h, const airg_solve_config* cfg, const double* b,
                      double* x, airg_solve_stats* st, double* hist, int64_t cap) {
  const SparseMatrix& a = h.top();
  const index_t n = a.nrows();
  const int64_t m = cfg->gmres_restart > 0 ? cfg->gmres_restart : 30;
  if (cfg->rtol <= 0.0) throw std::invalid_argument("gmres_solve: rtol must be positive");
  const SolveConfig scfg = to_scfg(cfg);
  int64_t hl = 0;
  auto push = [&](double v) {
    if (hist && hl < cap) hist[hl] = v;
    ++hl;
  };
  auto nrm = [&](const double* v) {
    double s = 0.0;
    for (index_t i = 0; i < n; ++i) s += v[i] * v[i];
    return std::sqrt(s);
  };
  std::vector<double> V((size_t)n * (m + 1) + 1), Z((size_t)n * m + 1), r(n), H((m + 1) * m, 0.0);
  std::vector<double> cs(m), sn(m), g(m + 1), hcol(m + 1), y(m + 1), zero(n, 0.0);
  std::fill(x, x + n, 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  const double bnorm = nrm(b);
  int64_t its = 0;
  std::memset(st, 0, sizeof(*st));
  if (bnorm == 0.0) {
    st->converged = 1;
    push(0.0);
  } else {
    std::memcpy(r.data(), b, sizeof(double) * n);
    double beta = bnorm;
    push(1.0);
    st->final_relative_residual = 1.0;
    while (its < cfg->max_iterations) {
      for (index_t i = 0; i < n; ++i) V[i] = r[i] / beta;
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int64_t j = 0;
      std::vector<double> w;
      double hn = 0.0;
      for (; j < m && its < cfg->max_iterations; ++j) {
        double* vj = V.data() + j * n;
        double* zj = Z.data() + j * n;
        std::vector<double> e = vcycle(h, std::span<const double>(vj, n), zero, scfg);
        std::memcpy(zj, e.data(), sizeof(double) * n);
        w = spmv(a, std::span<const double>(zj, n));
        for (int64_t k = 0; k <= j; ++k) hcol[k] = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
          for (int64_t k = 0; k <= j; ++k) {
            double s = 0.0;
            const double* vk = V.data() + k * n;
            for (index_t i = 0; i < n; ++i) s += vk[i] * w[i];
            y[k] = s;
          }
          for (index_t i = 0; i < n; ++i) {
            double s = w[i];
            for (int64_t k = 0; k <= j; ++k) s -= y[k] * V[k * n + i];
            w[i] = s;
          }
          for (int64_t k = 0; k <= j; ++k) hcol[k] += y[k];
        }
        hn = nrm(w.data());
        hcol[j + 1] = hn;
        double* vn = V.data() + (j + 1) * n;
        for (index_t i = 0; i < n; ++i) vn[i] = hn > 0.0 ? w[i] / hn : 0.0;
        for (int64_t k = 0; k < j; ++k) {
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
        for (int64_t k = 0; k <= j; ++k) H[k + j * (m + 1)] = hcol[k];
        ++its;
        const double est = std::fabs(g[j + 1]) / bnorm;
        push(est);
        if (est <= cfg->rtol || hn == 0.0) {
          ++j;
          break;
        }
      }
      for (int64_t k = j - 1; k >= 0; --k) {
        double s = g[k];
        for (int64_t q = k + 1; q < j; ++q) s -= H[k + q * (m + 1)] * y[q];
        y[k] = s / H[k + k * (m + 1)];
      }
      for (index_t i = 0; i < n; ++i) {
        double s = x[i];
        for (int64_t k = 0; k < j; ++k) s += y[k] * Z[k * n + i];
        x[i] = s;
      }
      std::vector<double> ax = spmv(a, std::span<const double>(x, n));
      for (index_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
      beta = nrm(r.data());
      const double rel = beta / bnorm;
      st->final_relative_residual = rel;
      if (rel <= cfg->rtol) {
        st->converged = 1;
        break;
      }
      if (beta == 0.0) break;
    }
  }
  st->iterations = its;
  st->solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  st->history_len = hl;
}

int ref_solve(const void* hp, const airg_solve_config* cfg, const double* b,
              double* x, airg_solve_stats* st, double* hist, int64_t cap) {
  return guard([&] {
    const Hierarchy& h = static_cast<const RefHier*>(hp)->h;
    if (cfg->outer == 1) {
      ref_gmres(h, cfg, b, x, st, hist, cap);
      return;
    }
    const index_t n = h.top().nrows();
    std::vector<double> xo;
    SolveStats s = richardson_solve(h, std::span<const double>(b, n), to_scfg(cfg), &xo);
    std::memcpy(x, xo.data(), sizeof(double) * n);
    std::memset(st, 0, sizeof(*st));
    st->iterations = s.iterations;
    st->converged = s.converged;
    st->final_relative_residual = s.final_relative_residual;
    st->flops = s.flops;
    st->shadow_flops = s.shadow_flops;
    st->work_units = s.work_units;
    st->grid_complexity = s.grid_complexity;
    st->operator_complexity = s.operator_complexity;
    st->storage_complexity = s.storage_complexity;
    st->solve_seconds = s.solve_seconds;
    st->wu_ratio = s.wu_ratio;
    st->c_grind_ns = s.c_grind_ns;
    st->d_grind_ns = s.d_grind_ns;
    const int64_t k = std::min<int64_t>(cap, s.residual_history.size());
    if (hist) std::memcpy(hist, s.residual_history.data(), sizeof(double) * k);
    st->history_len = static_cast<int64_t>(s.residual_history.size());
  });
}

// ---- side: the reference's own desk operator (transport.cpp) --------------
int ref_desk_problem(int64_t nx, uint64_t seed, double jitter, void** a_out,
                     double* b_out, int64_t b_cap, int64_t* n_out) {
  return guard([&] {
    StreamingProblem p = assemble_streaming(generate_mesh(nx, seed, jitter));
    *n_out = p.a.nrows();
    if (b_out && b_cap >= p.a.nrows())
      std::memcpy(b_out, p.b.data(), sizeof(double) * p.b.size());
    *a_out = new SparseMatrix(std::move(p.a));
  });
}

}  // extern "C"
