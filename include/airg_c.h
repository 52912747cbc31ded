/* include/airg_c.h -- C-ABI of the B200-native AIRG hot path.
 *
 * This is the drop-in boundary. Every entry point replaces
 * one reference C++ entry point of namespace airgraph in
 * /root/reference/proj/include/airgraph/ (cited per function below); the
 * C++ mirror in paper_2408_08262_b200/cpp/airgraph_gpu.hpp rebuilds those
 * signatures and exception types on top of this ABI, and the Python mirror
 * (paper_2408_08262_b200/airg.py) binds it with ctypes.
 *
 * Conventions
 *  - Every function returns AIRG_OK (0) or a negative status; the message
 *    (with the offending row index where the reference reports one) is
 *    available from airg_last_error(), which is thread-local.
 *      AIRG_EINVAL   <-> std::invalid_argument  (shape / argument errors)
 *      AIRG_ERUNTIME <-> std::runtime_error     (zero diagonal, stall, ...)
 *      AIRG_ECUDA    CUDA runtime failure; AIRG_ENOMEM allocation failure.
 *  - Host-side CSR arrays use the reference layout: int64 row offsets and
 *    column indices, fp64 values (sparse.hpp:89-93). Device CSR is int32
 *    indices + fp64 values; upload checks the int32 range.
 *  - "d_" pointers are device pointers on the context's device; "h_"
 *    pointers are host pointers. All work is ordered on the context stream.
 *  - No torch types appear here; plain pointers and sizes only.
 */
#ifndef AIRG_C_H_
#define AIRG_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AIRG_OK 0
#define AIRG_EINVAL (-1)
#define AIRG_ERUNTIME (-2)
#define AIRG_ECUDA (-3)
#define AIRG_ENOMEM (-4)
#define AIRG_ELOGIC (-5)

/* CF labels, as airgraph::CfLabel (sparse.hpp:22). */
#define AIRG_F 0
#define AIRG_C 1
#define AIRG_UNASSIGNED 2

/* Mirrors airgraph::SetupConfig (air.hpp:16-43); same defaults from
 * airg_setup_config_default(). */
typedef struct airg_setup_config {
  double strength_alpha;      /* 0.5 */
  int32_t cf;                 /* 0 = PMISR (only GPU mode), 1 PMIS, 2 PMIS-swap */
  int32_t ddc_enabled;        /* 1 */
  double ddc_fraction;        /* 0.10 */
  int64_t ddc_bins;           /* 1000 */
  int64_t max_loops;          /* 3 */
  int64_t poly_order;         /* 6 */
  int64_t sparsity_order;     /* 1 */
  double drop_coarse;         /* 0.001 */
  double drop_restrict;       /* 0.01 */
  int64_t coarse_size_target; /* 3000 */
  int64_t coarse_poly_order;  /* 12 */
  int64_t coarse_iterations;  /* 3 */
  int64_t max_levels;         /* 0 = unlimited */
  int32_t prolongation;       /* 0 = one-point (1 = ideal: test hook, EINVAL on GPU) */
  int32_t weight_mode;        /* 0 = |S|+|S^T|, 1 = |S u S^T| */
  uint64_t seed;              /* 0 */
  int32_t fused_smooths;      /* -1 = build the fast V-cycle's fused level operators on the first
                                 fast solve; k >= 0 = build them at setup for k F-smooths */
  int32_t _pad;
} airg_setup_config;

/* Mirrors airgraph::SolveConfig (solve.hpp:11-19) plus the outer solver
 * selection (outer GMRES is new, BASELINE.json config 0 / SURVEY §8f-1). */
typedef struct airg_solve_config {
  double rtol;                /* 1e-10 */
  int64_t max_iterations;     /* 200 */
  int64_t up_f_smooths;       /* 2 */
  int64_t down_smooths;       /* 0 */
  int64_t coarse_iterations;  /* 3 */
  int32_t collect_timing;     /* 1 */
  int32_t outer;              /* 0 = Richardson (reference), 1 = right-preconditioned GMRES */
  int64_t nddofs;             /* 0 */
  int64_t gmres_restart;      /* 30 */
  int32_t fast;               /* 0 = the reference's bits (thread-per-row ordered sums, no FMA);
                                 1 = lane groups per row, FMA, tree reductions (solve within
                                 rounding of the reference: rtol, +-1 iteration, 1e-8 in x) */
  int32_t _pad2;
} airg_solve_config;

/* Mirrors airgraph::SolveStats (solve.hpp:21-39). */
typedef struct airg_solve_stats {
  int64_t iterations;
  int32_t converged;
  int32_t _pad;
  double final_relative_residual;
  uint64_t flops;
  uint64_t shadow_flops;
  double work_units;
  double grid_complexity;
  double operator_complexity;
  double storage_complexity;
  double solve_seconds;
  double wu_ratio;
  double c_grind_ns;
  double d_grind_ns;
  int64_t history_len; /* entries written to the caller's history buffer */
} airg_solve_stats;

/* Per-level summary of a built hierarchy (air.hpp:49-66). */
typedef struct airg_level_info {
  int64_t n, nnz;           /* level operator A_l */
  int64_t n_f, n_c;         /* after DDC */
  int64_t n_f_pre;          /* after PMISR, before DDC */
  int64_t ddc_converted;
  int64_t nnz_ff, nnz_fc, nnz_cf, nnz_ffinv, nnz_r, nnz_p;
  double max_theta_pre, alpha_diag, max_theta_post;
  double smoother_growth;
  int64_t poly_attempts;
  int64_t effective_order;
  double coefficients[32];  /* poly_order + 1 <= 32 */
} airg_level_info;

typedef struct airg_hier_info {
  int64_t n_levels;         /* number of fine levels (Hierarchy::levels.size()) */
  int64_t coarse_n, coarse_nnz, coarse_inv_nnz;
  int64_t coarse_effective_order;
  int64_t coarse_attempts;
  double coarse_growth;
  double coarse_coefficients[32];
  double grid_complexity, operator_complexity, storage_complexity;
} airg_hier_info;

/* Coefficient injection: the polynomial coefficients are
 * computed in x87 long double through Eigen upstream (gmres_poly.cpp:63-171)
 * and cannot be reproduced bit-for-bit on a GPU. With an injection table the
 * GPU setup uses the given per-level coefficients (and the given coarse
 * level / coarse polynomial) instead of its own double-double fit, which
 * makes the whole hierarchy bit-identical to the reference's. */
typedef struct airg_injection {
  int64_t n_levels;                  /* fine levels to build */
  int64_t stride;                    /* doubles per level in level_coeffs */
  const double* level_coeffs;        /* n_levels x stride */
  const int64_t* level_eff_order;    /* n_levels */
  const double* coarse_coeffs;       /* coarse_poly_order + 1 values */
  int64_t coarse_eff_order;
} airg_injection;

typedef struct airg_ctx airg_ctx;
typedef struct airg_csr airg_csr;
typedef struct airg_hier airg_hier;

/* ---- errors and defaults ---------------------------------------------- */
int airg_last_error(char* buf, size_t len);
void airg_setup_config_default(airg_setup_config* cfg);
void airg_solve_config_default(airg_solve_config* cfg);
const char* airg_version(void);

/* ---- context ------------------------------------------------------------ */
int airg_ctx_create(int device, airg_ctx** out);
int airg_ctx_destroy(airg_ctx* ctx);
/* Use an external cudaStream_t (passed as void*); NULL restores the
 * context's own stream. */
int airg_ctx_set_stream(airg_ctx* ctx, void* stream);
int airg_ctx_synchronize(airg_ctx* ctx);
/* Number of kernels this library launched on the context since creation
 * (bench.py reports the delta over the timed region as gpu_launches). */
int airg_ctx_launch_count(airg_ctx* ctx, uint64_t* out);

/* ---- CSR (airgraph::SparseMatrix, sparse.hpp:33-94) ---------------------- */
/* Validating upload from the reference layout (ctor checks sparse.cpp:18-46). */
int airg_csr_upload(airg_ctx* ctx, int64_t nrows, int64_t ncols,
                    const int64_t* h_row_offsets, const int64_t* h_cols,
                    const double* h_vals, airg_csr** out);
int airg_csr_info(const airg_csr* a, int64_t* nrows, int64_t* ncols,
                  int64_t* nnz);
int airg_csr_download(airg_ctx* ctx, const airg_csr* a, int64_t* h_row_offsets,
                      int64_t* h_cols, double* h_vals);
/* Device views of the CSR arrays (int32 offsets/cols, fp64 values). */
int airg_csr_device_ptrs(const airg_csr* a, const int32_t** d_row_offsets,
                         const int32_t** d_cols, const double** d_vals);
int airg_csr_destroy(airg_csr* a);

/* ---- device buffers (for C / C++ / FFI hosts that do not link CUDA) ------- */
/* Stream-ordered allocation on the context's device (synchronised). */
int airg_device_alloc(airg_ctx* ctx, size_t bytes, void** d_out);
int airg_device_free(airg_ctx* ctx, void* d_ptr);
/* to_device != 0: host -> device, else device -> host (synchronised). */
int airg_memcpy(airg_ctx* ctx, void* dst, const void* src, size_t bytes,
                int32_t to_device);

/* ---- L0 kernels ---------------------------------------------------------- */
/* y = A x (sparse.cpp:185-201): sequential per-row accumulation in column
 * order without FMA, bit-identical to the reference. */
int airg_spmv(airg_ctx* ctx, const airg_csr* a, const double* d_x, double* d_y);
/* spmv with host vectors (the reference signature's value semantics). */
int airg_spmv_host(airg_ctx* ctx, const airg_csr* a, const double* h_x, double* h_y);
/* C = A B (sparse.cpp:203-242), cancellation zeros kept, contributions to
 * each entry accumulated in A-row order. */
int airg_spgemm(airg_ctx* ctx, const airg_csr* a, const airg_csr* b,
                airg_csr** out);
/* drop_entries (sparse.cpp:244-268). */
int airg_drop(airg_ctx* ctx, const airg_csr* a, double tol, int keep_diagonal,
              airg_csr** out);
/* SparseMatrix::with_full_diagonal (sparse.cpp:132-160). */
int airg_with_full_diagonal(airg_ctx* ctx, const airg_csr* a, airg_csr** out);

/* ---- L1a CF splitting (coarsening.hpp) ----------------------------------- */
/* strength (coarsening.cpp:83-105): S as a pattern CSR (values 1.0). */
int airg_strength(airg_ctx* ctx, const airg_csr* a, double alpha,
                  airg_csr** s_out);
/* strength -> pmisr (coarsening.cpp:107-167) on the GPU. d_labels gets the
 * PMISR labels (n bytes), d_weights (nullable) the weights. */
int airg_pmisr(airg_ctx* ctx, const airg_csr* a, double alpha,
               int64_t max_loops, uint64_t seed, int32_t weight_mode,
               uint8_t* d_labels, double* d_weights);
/* pmis(strength(a, alpha), swap, seed) (coarsening.cpp:169-217): the
 * classical PMIS rounds on S u S^T, the paper's comparison splitting; swap
 * exchanges C and F (PMIS-swap). Labels F = 0, C = 1. */
int airg_pmis(airg_ctx* ctx, const airg_csr* a, double alpha, int32_t swap, uint64_t seed,
              uint8_t* d_labels);
/* pmisr_with_weights (coarsening.hpp:83-84) on a caller-supplied strength
 * pattern S (StrengthGraph::from_pattern) and caller weights (device). */
int airg_pmisr_with_weights(airg_ctx* ctx, const airg_csr* s_pattern,
                            int64_t max_loops, const double* d_weights,
                            uint8_t* d_labels);
typedef struct airg_cf_report {
  int64_t n_f_pre, n_f, n_c, n_converted;
  double max_theta, alpha_diag;
  int64_t s_nnz;
} airg_cf_report;
/* The fused CF split strength -> pmisr -> extract_blocks -> ddc
 * (air.cpp:466-494) with the global 1000-bin histogram (coarsening.cpp:
 * 219-330). d_labels_pre (nullable) receives the PMISR labels. */
int airg_cf_split(airg_ctx* ctx, const airg_csr* a, double alpha,
                  int64_t max_loops, uint64_t seed, int32_t weight_mode,
                  int32_t ddc_enabled, double ddc_fraction, int64_t ddc_bins,
                  uint8_t* d_labels, uint8_t* d_labels_pre,
                  airg_cf_report* report);
/* pmisr / pmis on a caller-supplied strength pattern S (the reference's
 * pmisr(const StrengthGraph&, ...) / pmis(g, swap, seed), coarsening.hpp:
 * 78-90): weights from |S_i| + |S^T_i| (or |S u S^T| for weight_mode 1) and
 * the seeded hash, d_weights (nullable) receives them. */
int airg_pmisr_pattern(airg_ctx* ctx, const airg_csr* s_pattern, int64_t max_loops, uint64_t seed,
                       int32_t weight_mode, uint8_t* d_labels, double* d_weights);
int airg_pmis_pattern(airg_ctx* ctx, const airg_csr* s_pattern, int32_t swap, uint64_t seed, uint8_t* d_labels);
/* ddc(a_ff, labels, map, opt) (coarsening.cpp:252-330; coarsening.hpp:133)
 * on the F block itself: d_labels (n, global) converted in place. */
int airg_ddc_block(airg_ctx* ctx, const airg_csr* a_ff, uint8_t* d_labels, int64_t n, double fraction,
                   int64_t bins, int32_t selection, double direct_alpha_diag, airg_cf_report* report);
/* airg_cf_split (weight_mode 0) on `count` matrices with one
 * synchronisation: the splits are enqueued back to back on the context
 * stream and their reports read once at the end (e.g. re-splitting every
 * level of a hierarchy, or many independent systems). seeds[i], d_labels[i]
 * and reports[i] belong to mats[i]; labels are identical to one
 * airg_cf_split call per matrix. No reference counterpart (batching of
 * air.cpp:466-494 over matrices). */
int airg_cf_split_batch(airg_ctx* ctx, const airg_csr* const* mats,
                        int64_t count, const uint64_t* seeds, double alpha,
                        int64_t max_loops, int32_t ddc_enabled,
                        double ddc_fraction, int64_t ddc_bins,
                        uint8_t* const* d_labels, airg_cf_report* reports);
/* airg_cf_split with the labels returned to host memory. */
int airg_cf_split_host(airg_ctx* ctx, const airg_csr* a, double alpha,
                       int64_t max_loops, uint64_t seed, int32_t weight_mode,
                       int32_t ddc_enabled, double ddc_fraction,
                       int64_t ddc_bins, uint8_t* h_labels,
                       airg_cf_report* report);
/* ddc on given labels (coarsening.cpp:252-330); selection 0 = histogram,
 * 2 = direct (alpha_diag given). Converts in place. */
int airg_ddc(airg_ctx* ctx, const airg_csr* a, uint8_t* d_labels,
             double fraction, int64_t bins, int32_t selection,
             double direct_alpha_diag, airg_cf_report* report);
/* dominance_report (coarsening.cpp:219-250; coarsening.hpp:106) of an A_ff
 * block: theta per row into d_theta (device, nullable), the bins-bin
 * histogram over [0, max theta] into h_hist (host int64[bins], nullable),
 * max theta. Zero diagonal: AIRG_ERUNTIME "... zero diagonal in A_ff row i". */
int airg_dominance_report(airg_ctx* ctx, const airg_csr* a_ff, int64_t bins,
                          double* d_theta, int64_t* h_hist, double* max_theta);
/* build_label_map (sparse.cpp:270-290; sparse.hpp:133): stable F-then-C
 * sub-indexing of device labels; host int64 outputs (each nullable):
 * fine_to_sub[n], f_to_fine[n_f], c_to_fine[n - n_f]. */
int airg_build_label_map(airg_ctx* ctx, const uint8_t* d_labels, int64_t n,
                         int64_t* h_fine_to_sub, int64_t* h_f_to_fine,
                         int64_t* h_c_to_fine, int64_t* n_f);
/* extract_blocks (sparse.cpp:292-340): A_ff, A_fc, A_cf (A_cc unused). */
int airg_extract_blocks(airg_ctx* ctx, const airg_csr* a,
                        const uint8_t* d_labels, airg_csr** aff,
                        airg_csr** afc, airg_csr** acf);

/* ---- L1b polynomials (gmres_poly.hpp) ------------------------------------ */
/* compute_coefficients (gmres_poly.cpp:63-171): power basis and Gram matrix
 * in double-double on the GPU, rank cut and least squares in double-double
 * on the host. h_coeffs gets m values. */
int airg_poly_coefficients(airg_ctx* ctx, const airg_csr* a, int64_t m,
                           uint64_t seed, double* h_coeffs,
                           int64_t* effective_order);
/* assemble_fixed_sparsity (gmres_poly.cpp:197-280). */
int airg_poly_assemble(airg_ctx* ctx, const airg_csr* a, const double* h_coeffs,
                       int64_t n_coeffs, int64_t effective_order,
                       int64_t sparsity_order, airg_csr** out);

/* ---- L2 setup (air.hpp) ---------------------------------------------------- */
/* setup (air.cpp:285-410). inj may be NULL (native coefficients). */
int airg_setup(airg_ctx* ctx, const airg_csr* a, const airg_setup_config* cfg,
               const airg_injection* inj, airg_hier** out);
/* setup at N GPUs (SURVEY §8e setup collectives): every heavy row kernel of
 * the setup (the CF split, the SpGEMMs of Z, A P and R (A P), the polynomial
 * assembly, the power-basis and growth SpMVs) runs on one row slab per rank
 * and the slabs are all-gathered over NCCL; every rank ends with the same
 * hierarchy, bit-identical to airg_setup's (also in native mode). rank = -1
 * emulates all ranks in this process; rank >= 0 needs a communicator and the
 * same (replicated) input on every rank. Feed the result to airg_dist_create. */
int airg_dist_setup(airg_ctx* ctx, const airg_csr* a, const airg_setup_config* cfg,
                    const airg_injection* inj, int32_t nranks, int32_t rank, void* nccl_comm,
                    airg_hier** out);
int airg_hier_info_get(const airg_hier* h, airg_hier_info* info);
int airg_hier_level_info(const airg_hier* h, int64_t level,
                         airg_level_info* info);
/* A device hierarchy from given level operators (a host airgraph::Hierarchy
 * handed to vcycle / richardson_solve / f_smooth through the C++ shim):
 * mats = n_levels x {A, A_ff, A_fc, A_cf, Aff_inv, R, P} (P one-point),
 * d_labels = per level n bytes (device), the coarse operator and its
 * assembled inverse. */
int airg_hier_from_levels(airg_ctx* ctx, int64_t n_levels, const airg_csr* const* mats,
                          const uint8_t* const* d_labels, const airg_csr* coarse_a, const airg_csr* coarse_inv,
                          int64_t coarse_iterations, airg_hier** out);
/* which: 0 A, 1 A_ff, 2 A_fc, 3 A_cf, 4 Aff_inv, 5 R, 6 P, and (fast V-cycle,
 * once built) 7 A_F P (n_f x n_c), 8 W_k (n_f x n_f), and on levels with the
 * one-pass ascent 9 K = P_F - W_k A_F P (n_f x n_c), 10 [R; W_k E_F^T]
 * ((n_c + n_f) x n); level == n_levels with which 0 / 4 / 9 gives the coarse
 * A / coarse inverse / composed coarse solve E_k. Returns a borrowed handle
 * owned by the hierarchy. */
int airg_hier_matrix(const airg_hier* h, int64_t level, int32_t which,
                     const airg_csr** out);
int airg_hier_labels(airg_ctx* ctx, const airg_hier* h, int64_t level,
                     uint8_t* h_labels);
int airg_hier_destroy(airg_hier* h);

/* ---- transfer operators (air.hpp:96-116) ----------------------------------- */
/* build_restriction(a_cf, aff_inv, drop_restrict, map) (air.cpp:154-189):
 * R = [-drop(A_cf Aff_inv, drop, keep_diagonal=false) | I] in fine columns;
 * the map is built from the n device labels. */
int airg_build_restriction(airg_ctx* ctx, const airg_csr* a_cf,
                           const airg_csr* aff_inv, double drop_restrict,
                           const uint8_t* d_labels, int64_t n, airg_csr** out);
/* build_prolongation(labels, map, g, a) (air.cpp:191-238): one-point P from
 * the strength pattern s (airg_strength of a) and a. */
int airg_build_prolongation(airg_ctx* ctx, const airg_csr* a, const airg_csr* s,
                            const uint8_t* d_labels, airg_csr** out);
/* coarse_matrix(r, a, p, drop_coarse) (air.cpp:268-271):
 * drop_entries(R (A P), drop_coarse). */
int airg_coarse_matrix(airg_ctx* ctx, const airg_csr* r, const airg_csr* a,
                       const airg_csr* p, double drop_coarse, airg_csr** out);
/* apply_polynomial(a, p, b) (gmres_poly.cpp:173-195; gmres_poly.hpp:40-43):
 * d_y = q(A) d_b by Horner over coefficients[0..effective_order] (host),
 * effective_order matvecs, products and sums rounded separately. */
int airg_apply_polynomial(airg_ctx* ctx, const airg_csr* a, const double* coeffs,
                          int64_t ncoeffs, int64_t effective_order,
                          const double* d_b, double* d_y);

/* ---- L3 solve (solve.hpp) -------------------------------------------------- */
/* f_smooth(level, b, x) (solve.cpp:63-87; solve.hpp:43-46) on level `level`
 * of a built hierarchy: x_F += Aff_inv ((b_F - A_FF x_F) - A_FC x_C) in
 * place on the device vector d_x (the level's size); C entries untouched. */
int airg_f_smooth(airg_ctx* ctx, const airg_hier* h, int64_t level,
                  const double* d_b, double* d_x);
/* vcycle (solve.cpp:150-165) from x = 0 (x_is_zero): d_x = V(d_b). */
int airg_vcycle(airg_ctx* ctx, const airg_hier* h, const airg_solve_config* cfg,
                const double* d_b, double* d_x);
/* richardson_solve (solve.cpp:167-259) or outer GMRES per cfg->outer, with
 * device-resident b and x. h_history (nullable) gets up to history_cap
 * relative residuals. */
int airg_solve(airg_ctx* ctx, const airg_hier* h, const airg_solve_config* cfg,
               const double* d_b, double* d_x, airg_solve_stats* stats,
               double* h_history, int64_t history_cap);
/* The reference-facing call with HOST buffers: H2D of b, solve, D2H of x. */
int airg_solve_host(airg_ctx* ctx, const airg_hier* h,
                    const airg_solve_config* cfg, const double* h_b,
                    double* h_x, airg_solve_stats* stats, double* h_history,
                    int64_t history_cap);

/* ---- multi-GPU: row-slab distributed solve ------------------ */
typedef struct airg_dist airg_dist;
/* NCCL bootstrap: rank 0 creates the 128-byte id, every rank passes it. */
int airg_nccl_unique_id(void* h_id128);
int airg_nccl_comm_create(int nranks, int rank, const void* h_id128, void** comm_out);
int airg_nccl_comm_destroy(void* comm);
/* Partition a built hierarchy into P contiguous row slabs per level with the
 * reference's halving rule (partition_model.cpp:77-112, threshold on the
 * local/non-local nnz ratio) and a gathered coarsest grid. rank = -1
 * emulates all P ranks on this context's GPU (phase by phase; no kernel
 * waits on another rank); rank >= 0 builds only that rank's slab and needs
 * an NCCL communicator. h_level0_starts (P+1, nullable) fixes level 0's
 * slabs (e.g. z-slabs). */
int airg_dist_create(airg_ctx* ctx, const airg_hier* h, int32_t nranks,
                     int32_t rank, void* nccl_comm, double halving_threshold,
                     const int64_t* h_level0_starts, airg_dist** out);
/* Richardson solve over the slabs: emulation takes/returns global device
 * vectors; with NCCL d_b / d_x are this rank's level-0 slab. */
/* Owned-row distributed setup (SURVEY §8e setup collectives; air.cpp:285-434
 * per rank): every rank holds and builds only its rows of every level --
 * CF split on the slabs, A_ff halo rows gathered once for the fixed-sparsity
 * assembly, distance-2 halo rows of Aff^-1 and A P for Z and R (A P), the
 * Gram matrix and growth norms reduced over the ranks, the next level's rows
 * moved to its (halved) partition, the coarsest grid gathered on rank 0.
 * a: with rank < 0 (emulation) the whole operator, split by starts[0..nranks];
 * with rank >= 0 this rank's rows starts[rank].. with global columns. The
 * result solves through airg_dist_solve like airg_dist_create's. Replaces
 * the replicated airg_dist_setup + airg_dist_create pair. */
int airg_dist_setup_owned(airg_ctx* ctx, const airg_csr* a, const int64_t* h_starts,
                          const airg_setup_config* cfg, const airg_injection* inj, int32_t nranks,
                          int32_t rank, void* nccl_comm, double threshold, airg_dist** out);
/* Setup report of an owned distribution (identical on every rank): level l
 * < n_levels as airg_level_info; level n_levels = the coarse grid (n, nnz,
 * nnz_ffinv = |Ac^-1|, coefficients, effective_order, poly_attempts,
 * smoother_growth of the coarse polynomial). info may be null (n_levels only). */
int airg_dist_report(const airg_dist* d, int64_t level, airg_level_info* info, int64_t* n_levels);
/* Global entries of the fast V-cycle's A_F P and W_k slabs of level `level`
 * (distributions built with fused operators: owned setup with fused_smooths
 * in 0..2, or dist_create of a hierarchy whose fused operators exist). */
int airg_dist_fused_nnz(const airg_dist* d, int64_t level, int64_t* nnz_afp, int64_t* nnz_w);
/* Entries of the composed coarse solve E_k held by this process (built by the
 * first fast solve; -1 when the fast V-cycle does not use it). */
int airg_dist_coarse_e_nnz(const airg_dist* d, int64_t* nnz);
/* This process's wall time of the owned setup and the device time of its
 * CF splits (all levels), in ms (0 for airg_dist_create distributions). */
int airg_dist_setup_times(const airg_dist* d, double* setup_ms, double* cf_split_ms);
int airg_dist_solve(airg_ctx* ctx, airg_dist* d, const airg_solve_config* cfg,
                    const double* d_b, double* d_x, airg_solve_stats* stats,
                    double* h_history, int64_t history_cap);
/* Halo bytes this process receives per V-cycle and per level-0 SpMV (all
 * emulated ranks in emulation mode; NVLink traffic of the solve). */
int airg_dist_halo_bytes(const airg_dist* d, const airg_solve_config* cfg, int64_t* vcycle_bytes,
                         int64_t* spmv_bytes);
/* Device bytes of one rank's share of the distributed hierarchy (its slabs
 * of every level's operators, maps and solve vectors). The distribution owns
 * its slabs: the global hierarchy may be destroyed once it is created. */
int airg_dist_rank_bytes(const airg_dist* d, int32_t rank, int64_t* bytes);
/* local_share (partition_model.cpp:66-75) of a level before / after its
 * halving decision (levels below n_levels). */
int airg_dist_level_share(const airg_dist* d, int64_t level, double* share_before, double* share_after);
/* Per level: active ranks, replay-rule ratios, total halo entries. */
int airg_dist_level_info(const airg_dist* d, int64_t level, int32_t* active,
                         double* ratio_before, double* ratio_after,
                         int32_t* triggered, int64_t* halo_entries,
                         int64_t* h_starts /* P+1, nullable */);
/* Halo transport of the solve: 0 = emulation gather kernel, 1 = NCCL
 * send/recv, 2 = NVLink peer stores (AIRG_TRANSPORT=p2p; emulated or one
 * process per GPU). */
int airg_dist_transport(const airg_dist* d, int32_t* transport);
/* Host-only rule of the p2p push (no GPU; CPU / gloo tests): the entries of
 * the receiver's sorted halo that `sender` owns, as the sender's local index
 * and the position in the receiver's [own | halo] buffer they are stored to. */
int airg_p2p_push_plan_host(int32_t nranks, const int64_t* h_starts,
                            int32_t sender, const int64_t* recv_halo,
                            int64_t n_recv_halo, int32_t receiver,
                            int32_t* src_idx, int64_t* dst_pos, int64_t cap,
                            int64_t* n_push);
int airg_dist_destroy(airg_dist* d);
/* ---- Matrix Market exchange (matrix_market.hpp:11-19) ---------------------
 * Host-side, no GPU needed. airg_mm_read parses a "coordinate real general"
 * file (1-based, duplicates summed as SparseMatrix::from_triplets,
 * sparse.cpp:48-80); the result is read out with airg_mm_dims/airg_mm_copy
 * (int64 CSR, the reference layout) and released with airg_mm_free.
 * airg_mm_write writes the reference's format ("%.17g" values). Errors are
 * AIRG_ERUNTIME with the reference's "matrix market: <path>: ..." text. */
typedef struct airg_mm airg_mm;
int airg_mm_read(const char* path, airg_mm** out);
int airg_mm_dims(const airg_mm* h, int64_t* nrows, int64_t* ncols, int64_t* nnz);
int airg_mm_copy(const airg_mm* h, int64_t* row_offsets, int64_t* col_indices, double* values);
int airg_mm_free(airg_mm* h);
int airg_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_offsets,
                  const int64_t* col_indices, const double* values);

/* The PMISR-DDC CF split (air.cpp:466-494) of a slab-partitioned operator:
 * strength on own rows, |S^T| by a reverse halo sum, global-row-index
 * weights, one forward halo exchange of weights, "not minimal" marks of
 * remote endpoints returned to their owners, DDC with a global max and
 * 1000-bin histogram (allreduce). Labels are bit-identical to airg_cf_split
 * for every partition. rank = -1 emulates all ranks (d_labels global);
 * rank >= 0 needs a communicator (d_labels = this rank's slab). */
int airg_dist_cf_split(airg_ctx* ctx, const airg_csr* a, int32_t nranks,
                       int32_t rank, void* nccl_comm, const int64_t* h_starts,
                       double alpha, int64_t max_loops, uint64_t seed,
                       int32_t ddc_enabled, double ddc_fraction,
                       int64_t ddc_bins, uint8_t* d_labels,
                       airg_cf_report* report);
/* Host-only halo plan of one rank (the rule the device build applies):
 * sorted distinct referenced indices outside [starts[rank], starts[rank+1]),
 * plus the per-owner receive counts. No GPU needed (CPU / gloo tests). */
int airg_dist_plan_host(int32_t nranks, const int64_t* h_starts, int32_t rank,
                        const int64_t* h_cols, int64_t ncols,
                        int64_t* h_halo_out, int64_t halo_cap,
                        int64_t* n_halo, int64_t* h_recv_counts);

#ifdef __cplusplus
}
#endif

#endif /* AIRG_C_H_ */
