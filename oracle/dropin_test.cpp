// oracle/dropin_test.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Drop-in check at the C++ level: the reference library's own value types
// (airgraph::SparseMatrix from /root/reference, linked from oracle/_ref) are
// handed to the B200 engine through paper_2408_08262_b200/cpp/airgraph_gpu.hpp
// and the results are compared, in one process, with the reference's own
// functions using the reference's exact operator== (sparse.hpp:87).
// Built by `make -C oracle dropin`; run on a GPU box by
// tests/test_gpu_dropin.py. Exit code = number of failed checks.
#include <cstdio>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "airgraph/air.hpp"
#include "airgraph/coarsening.hpp"
#include "airgraph/rng.hpp"
#include "airgraph/solve.hpp"
#include "airgraph/sparse.hpp"
#include "airgraph/transport.hpp"
#include "airgraph_gpu.hpp"

using namespace airgraph;

static int failures = 0;
static void report(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), 8 * a.size()) == 0;
}

int main() {
  std::setvbuf(stdout, nullptr, _IONBF, 0);  // progress survives a crash
  airgraph_gpu::Context ctx(0);
  // the reference's own desk operator (transport.cpp), 4 SUPG angle blocks
  StreamingProblem p = assemble_streaming(generate_mesh(20, 3, 0.25));
  const SparseMatrix& a = p.a;
  std::vector<double> x(a.ncols());
  for (index_t i = 0; i < a.ncols(); ++i) x[i] = rng::uniform01(11, i) - 0.5;

  report(same_bits(spmv(a, x), airgraph_gpu::spmv(ctx, a, x)), "spmv bit-identical");
  report(spgemm(a, a) == airgraph_gpu::spgemm(ctx, a, a), "spgemm(A, A) == (reference operator==)");
  report(drop_entries(spgemm(a, a), 0.01) == airgraph_gpu::drop_entries(ctx, spgemm(a, a), 0.01),
         "drop_entries == ");
  report(drop_entries(a, 1.5, false) == airgraph_gpu::drop_entries(ctx, a, 1.5, false),
         "drop_entries(keep_diagonal=false) ==");

  // CF split exactly as air.cpp:466-494
  const SparseMatrix af = a.with_full_diagonal();
  const std::uint64_t seed = rng::mix(0, 0);
  StrengthGraph g = strength(af, 0.5);
  CfLabels l = pmisr(g, 3, seed);
  BlockSplit s = extract_blocks(af, l.label);
  DdcResult d = ddc(s.a_ff, l, s.map, DdcOptions{});
  if (!d.converted.empty()) l = d.labels;
  airg_cf_report rep;
  std::vector<uint8_t> gl = airgraph_gpu::cf_split(ctx, af, 0.5, 3, seed, true, 0.1, 1000, &rep);
  bool same = gl.size() == l.label.size();
  for (size_t i = 0; same && i < gl.size(); ++i) same = gl[i] == static_cast<uint8_t>(l.label[i]);
  report(same, "PMISR-DDC labels bit-identical");
  report(rep.n_converted == (int64_t)d.converted.size(), "DDC conversion count");

  // the single operations of air.hpp / coarsening.hpp / gmres_poly.hpp, on
  // the blocks of the final (post-DDC) labels
  {
    const BlockSplit s = extract_blocks(af, l.label);
    DominanceReport dr = dominance_report(s.a_ff, 1000);
    airgraph_gpu::DominanceReport gd = airgraph_gpu::dominance_report(ctx, s.a_ff, 1000);
    bool hist_ok = gd.histogram.size() == dr.histogram.size();
    for (size_t k = 0; hist_ok && k < dr.histogram.size(); ++k) hist_ok = gd.histogram[k] == dr.histogram[k];
    report(same_bits(dr.theta, gd.theta) && dr.max_theta == gd.max_theta && hist_ok,
           "dominance_report bit-identical");
    GmresPolynomial q = compute_coefficients(s.a_ff, 4, 5);
    std::vector<double> bf(s.a_ff.ncols());
    for (index_t i = 0; i < s.a_ff.ncols(); ++i) bf[i] = rng::uniform01(13, i);
    report(same_bits(apply_polynomial(s.a_ff, q, bf),
                     airgraph_gpu::apply_polynomial(ctx, s.a_ff, q.coefficients, q.effective_order, bf)),
           "apply_polynomial bit-identical");
    const SparseMatrix qa = assemble_fixed_sparsity(s.a_ff, q, 1);
    std::vector<uint8_t> lab8(l.label.size());
    for (size_t i = 0; i < lab8.size(); ++i) lab8[i] = static_cast<uint8_t>(l.label[i]);
    LabelMap map = build_label_map(l.label);
    const SparseMatrix r = build_restriction(s.a_cf, qa, 0.01, map);
    report(r == airgraph_gpu::build_restriction(ctx, s.a_cf, qa, 0.01, lab8), "build_restriction ==");
    const SparseMatrix pp = build_prolongation(l, map, g, af);
    std::vector<Triplet> st;
    for (index_t i = 0; i < g.n; ++i)
      for (index_t j : g.s_row(i)) st.push_back({i, j, 1.0});
    const SparseMatrix sp = SparseMatrix::from_triplets(g.n, g.n, st);
    report(pp == airgraph_gpu::build_prolongation(ctx, af, sp, lab8), "build_prolongation ==");
    report(coarse_matrix(r, af, pp, 0.001) == airgraph_gpu::coarse_matrix(ctx, r, af, pp, 0.001),
           "coarse_matrix ==");
  }

  // hierarchy with injected coefficients, then the Richardson solve
  SetupConfig cfg;
  cfg.poly_order = 3;
  cfg.coarse_poly_order = 3;
  cfg.coarse_iterations = 1;
  cfg.coarse_size_target = 0;
  cfg.drop_coarse = 0.0075;
  cfg.drop_restrict = 0.025;
  cfg.seed = 7;
  Hierarchy h = setup(a, cfg);
  std::vector<double> lc(32 * h.levels.size(), 0.0);
  std::vector<int64_t> le(h.levels.size());
  for (size_t k = 0; k < h.levels.size(); ++k) {
    for (size_t j = 0; j < h.levels[k].ff_inv.coefficients.size(); ++j)
      lc[32 * k + j] = h.levels[k].ff_inv.coefficients[j];
    le[k] = h.levels[k].ff_inv.effective_order;
  }
  std::vector<double> cc(32, 0.0);
  for (size_t j = 0; j < h.coarse_inv.coefficients.size(); ++j) cc[j] = h.coarse_inv.coefficients[j];
  airg_injection inj{(int64_t)h.levels.size(), 32, lc.data(), le.data(), cc.data(),
                     h.coarse_inv.effective_order};
  airg_setup_config gc;
  airg_setup_config_default(&gc);
  gc.poly_order = cfg.poly_order;
  gc.coarse_poly_order = cfg.coarse_poly_order;
  gc.coarse_iterations = cfg.coarse_iterations;
  gc.coarse_size_target = cfg.coarse_size_target;
  gc.drop_coarse = cfg.drop_coarse;
  gc.drop_restrict = cfg.drop_restrict;
  gc.seed = cfg.seed;
  airgraph_gpu::Hierarchy gh(ctx, a, gc, &inj);
  report(gh.info().n_levels == (int64_t)h.levels.size(), "level count");
  bool lab_ok = true;
  for (size_t k = 0; k < h.levels.size(); ++k) {
    auto gl2 = gh.labels((int64_t)k);
    for (size_t i = 0; i < gl2.size(); ++i)
      lab_ok &= gl2[i] == static_cast<uint8_t>(h.levels[k].map.label[i]);
  }
  report(lab_ok, "every level's CF labels bit-identical");
  SolveConfig sc;
  sc.coarse_iterations = 1;
  std::vector<double> xr;
  SolveStats sr = richardson_solve(h, p.b, sc, &xr);
  airg_solve_config gsc;
  airg_solve_config_default(&gsc);
  gsc.coarse_iterations = 1;
  std::vector<double> xg;
  airg_solve_stats sg = gh.solve(p.b, &xg, gsc);
  report(sg.iterations == sr.iterations && sg.flops == sr.flops, "iterations and flops identical");
  report(same_bits(xr, xg), "Richardson solution bit-identical");

  // error mapping onto the reference's exception types
  bool inv = false;
  try {
    airgraph_gpu::spmv(ctx, a, std::span<const double>(x.data(), x.size() - 1));
  } catch (const std::invalid_argument&) {
    inv = true;
  }
  report(inv, "dimension mismatch -> std::invalid_argument");
  bool rt = false;
  try {
    // no strong edges -> both rows F; row 1 carries an explicit zero diagonal
    SparseMatrix z = SparseMatrix::from_triplets(2, 2, {{0, 0, 1.0}}).with_full_diagonal();
    airgraph_gpu::cf_split(ctx, z, 0.5, 3, 0);
  } catch (const std::runtime_error& e) {
    rt = std::string(e.what()).find("row 1") != std::string::npos;
  }
  report(rt, "zero diagonal -> std::runtime_error naming the row");
  std::printf("%d failure(s)\n", failures);
  return failures;
}
