// Device-resident AIRG hierarchy (reference: air.hpp:45-91) plus the solve
// workspace and cached CUDA graphs.
#pragma once

#include "sparse.cuh"

namespace airg {

struct Level {
  Csr a;                     // level operator (full diagonal)
  LabelMap map;
  Csr aff, afc, acf;         // blocks (acf feeds Z; aff/afc are kept for download)
  Csr af;                    // F rows of A, global columns, bit 31 = C column
  Csr affg;                  // A_FF with global column indices (later F-smooths)
  Csr ffinv, r, p;
  DBuf<int32_t> pmap;        // one-point P as a map (-1 = empty row)
  Csr afp, fw;               // fast V-cycle (fused.cu): A_F P (n_f x n_c) and W_k (n_f x n_f)
  // one-pass ascent (fused.cu, chosen per level by the entry count): K = P_F - W_k A_F P
  // (n_f x n_c) and the descent operator [R; W_k E_F^T] ((n_c + n_f) x n)
  Csr fk, dsc;
  bool one_pass = false;
  // report
  int64_t n_f_pre = 0, n_converted = 0, attempts = 1, eff = 0;
  double max_theta_pre = 0.0, alpha_diag = 0.0, max_theta_post = 0.0, growth = 0.0;
  std::vector<double> coeffs;
  // solve workspace
  DBuf<double> b;            // level rhs (level 0 uses Hier::r)
  DBuf<double> x;            // level correction
  DBuf<double> rf;           // F residual
  DBuf<double> sc;           // A_FC x_C kept from the first F-smooth
};

struct GmDev {
  long long its;    // Arnoldi steps so far
  long long cap;    // history capacity
  long long maxit;  // max_iterations
  int j;            // column of the current cycle
  int m;            // restart length
  int converged;
  int restarts;
  int more;  // the inner loop continues (set by k_gm_cycle / k_gm_step; steps after it no-op)
  int _pad;
  double rtol, bnorm, beta, hn, rel, est;
};

struct Hier {
  std::vector<Level> levels;
  Csr coarse_a, coarse_inv;
  std::vector<double> coarse_coeffs;
  int64_t coarse_eff = 0, coarse_attempts = 1;
  double coarse_growth = 0.0;
  int64_t coarse_iterations = 3;  // SetupConfig (storage metric only)
  double grid_c = 0.0, op_c = 0.0, store_c = 0.0;
  int64_t fused_smooths = -1;  // up_f_smooths the fused operators were built for (-1: none)
  int64_t fused_gen = 0;       // bumped by every build (captured graphs hold the operators' pointers)
  int64_t fused_coarse_its = -1;  // coarse_iterations the composed coarse operator was built for
  Csr coarse_e;                   // composed coarse solve E_k (fused.cu); empty when not chosen
  bool coarse_composed = false;
  // coarse workspace
  DBuf<double> cb, cx, cr;
  // top-level solve workspace
  DBuf<double> rhs, xsol, r, part, scal;
  // outer GMRES workspace (allocated on first use)
  int64_t gm_restart = 0;
  DBuf<double> V, Z, w, hbuf, ybuf;
  // device-resident GMRES (solve.cu): state, Hessenberg / rotation scalars,
  // dot partials, history, the cycle residual and the nested-WHILE graph
  DBuf<GmDev> gm_st;
  DBuf<double> gm_H, gm_cs, gm_sn, gm_g, gm_y, gm_h, gm_part, gm_hist, r2, gm_G;
  cudaGraphExec_t g_gm = nullptr;
  int64_t g_key_gm = -1;
  uint64_t gm_kernels[3] = {0, 0, 0};  // launch, per cycle, per Arnoldi step
  bool gm_broken = false;
  // device-side Richardson loop (solve.cu): iteration count, residual
  // history, [rtol, max_iterations] and the conditional-WHILE graph
  DBuf<long long> loop_it;
  DBuf<double> loop_hist, loop_par, loop_stamps;
  cudaGraphExec_t g_loop = nullptr;
  int64_t g_key_loop = -1;
  uint64_t g_loop_kernels = 0;
  bool loop_broken = false;  // instantiation refused: host loop from then on
  // cached graphs
  cudaGraphExec_t g_rich = nullptr, g_vc = nullptr;
  int64_t g_key_rich = -1, g_key_vc = -1;
  uint64_t g_rich_kernels = 0, g_vc_kernels = 0;

  int32_t top_n() const { return levels.empty() ? coarse_a.n : levels.front().a.n; }
  const Csr& top() const { return levels.empty() ? coarse_a : levels.front().a; }
  ~Hier() {
    if (g_rich) cudaGraphExecDestroy(g_rich);
    if (g_vc) cudaGraphExecDestroy(g_vc);
    if (g_loop) cudaGraphExecDestroy(g_loop);
    if (g_gm) cudaGraphExecDestroy(g_gm);
  }
};

struct Injection {
  int64_t n_levels = -1;
  std::vector<std::vector<double>> level_coeffs;
  std::vector<int64_t> level_eff;
  std::vector<double> coarse_coeffs;
  int64_t coarse_eff = 0;
};

// make_checked_inverse (air.cpp:106-129) / a fixed polynomial on one GPU
struct CheckedInverse {
  std::vector<double> coeffs;
  int64_t eff = 0, attempts = 1;
  double growth = 0.0;
  Csr q;
};
CheckedInverse checked_inverse(Ctx& c, const Csr& a, int64_t order, int64_t sparsity, uint64_t seed);
CheckedInverse fixed_inverse(Ctx& c, const Csr& a, const std::vector<double>& coeffs, int64_t eff,
                             int64_t sparsity);

struct RowSplit;
// rs (nullable): split the setup's heavy row kernels over ranks (rowsplit.cuh)
void setup(Ctx& c, const Csr& a, const airg_setup_config& cfg, const Injection* inj, Hier& h,
           const RowSplit* rs = nullptr);
void recompute_metrics(Hier& h);
void alloc_workspace(Ctx& c, Hier& h);
// a device hierarchy from given level operators (host labels per level)
struct HostLevel {
  Csr a, aff, afc, acf, ffinv, r, p;
  const uint8_t* labels = nullptr;  // device, a.n bytes
};
void hier_from_levels(Ctx& c, std::vector<HostLevel>& in, Csr&& coarse_a, Csr&& coarse_inv,
                      int64_t coarse_iterations, Hier& h);

// fused.cu: C = alpha A + beta B (same shape, sorted rows; the union pattern)
void csr_add(Ctx& c, double alpha, const Csr& a, double beta, const Csr& b, Csr& out);
// fused.cu: the composed coarse solve E_k (k coarse Richardson steps from
// e = 0) of A with its assembled inverse Q; false when not offered
// (AIRG_COARSE_COMPOSE entries exceeded, k < 1, or a large grid)
bool compose_coarse(Ctx& c, const Csr& a, const Csr& q, int64_t its, Csr& out);
// fused.cu: the fast V-cycle's fused level operators for `smooths` F-smooths
// and the composed coarse solve for `coarse_its` coarse iterations
void build_fused(Ctx& c, Hier& h, int64_t smooths, int64_t coarse_its);
// the fused operators match a solve configuration
inline bool fused_ready(const Hier& h, int64_t smooths, int64_t coarse_its) {
  return h.fused_smooths == smooths && h.fused_coarse_its == coarse_its;
}

// solve.cu
void vcycle(Ctx& c, Hier& h, const airg_solve_config& cfg, const double* d_b, double* d_x);
void f_smooth_level(Ctx& c, Hier& h, int64_t l, const double* d_b, double* d_x);
void apply_polynomial(Ctx& c, Csr& a, const double* coeffs, int64_t ncoeffs, int64_t deg, const double* d_b,
                      double* d_y);
void solve(Ctx& c, Hier& h, const airg_solve_config& cfg, const double* d_b, double* d_x,
           airg_solve_stats& st, std::vector<double>& history);

}  // namespace airg
