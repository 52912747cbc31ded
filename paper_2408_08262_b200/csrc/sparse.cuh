// Internal API of the engine's device modules.
#pragma once

#include "common.cuh"
#include "dd.cuh"

namespace airg {

// sparse.cu -------------------------------------------------------------------
void csr_upload(Ctx& c, int64_t n, int64_t m, const int64_t* h_rp, const int64_t* h_ci,
                const double* h_v, Csr& out);
void csr_download(Ctx& c, const Csr& a, int64_t* h_rp, int64_t* h_ci, double* h_v);
void spmv(Ctx& c, const Csr& a, const double* x, double* y);
// row_base: the rows are global rows row_base.. of a square operator (slab: a row
// slab even when row_base is 0)
void with_full_diagonal(Ctx& c, const Csr& a, Csr& out, int row_base = 0, bool slab = false);
void drop_entries(Ctx& c, const Csr& a, double tol, bool keep_diagonal, Csr& out);
// entries per batch of the thread-per-row kernels for a matrix of n rows and
// nnz entries: 8 = aligned vector batches, 4 / 0 = 4- / 8-entry scalar batches
int row_vec(int64_t n, int64_t nnz);
// lanes per row of the fast-mode row kernels (tiled.cuh rows_lanes)
int row_lanes(int64_t n, int64_t nnz, int32_t max_row = -1);
// lanes of the exact mode's ordered-lane kernel (tiled.cuh rows_olanes) for a
// matrix of n rows and nnz entries; 0 = thread per row
int row_olanes(int64_t n, int64_t nnz);
// measure the longest row of every matrix into its max_row (one readback)
void row_max(Ctx& c, const std::vector<Csr*>& ms);
// out = a with every column j replaced by map[j] (order-preserving maps only)
void map_columns(Ctx& c, const Csr& a, const int32_t* d_map, int32_t new_ncols, Csr& out);

// spgemm.cu -------------------------------------------------------------------
// C = A B with per-entry accumulation in A-row order (sparse.cpp:203-242).
// drop_tol >= 0 fuses drop_entries(C, drop_tol, keep_diag) into the
// compaction; drop_tol < 0 keeps everything.
// bmap (device, nullable): B row of every A column -- B then holds gathered
// rows of a distributed operator; row_base: the rows of `a` are global rows
// row_base.. (diagonal of the drop rule); square_n: global row count of a
// square product computed as a row slab (-1: a.n).
void spgemm(Ctx& c, const Csr& a, const Csr& b, Csr& out, double drop_tol = -1.0,
            bool keep_diag = true, const int32_t* bmap = nullptr, int row_base = 0,
            int64_t square_n = -1);

// cfsplit.cu ------------------------------------------------------------------
struct Strength {
  int32_t n = 0;
  int64_t nnz = 0;
  DBuf<int32_t> rp, ci;     // S, sorted rows
  DBuf<int32_t> st_cnt;     // |S_i^T|
};
// row_base: the rows of `a` are global rows row_base.. of a larger operator
// (a row slab with global columns); 0 for a whole square matrix.
void strength(Ctx& c, const Csr& a, double alpha, Strength& g, int row_base = 0);
// PMISR labels (one-shot local minima, see cfsplit.cu) into d_labels.
void pmisr(Ctx& c, const Strength& g, int64_t max_loops, uint64_t seed, int weight_mode,
           uint8_t* d_labels, double* d_weights);
// pmisr_with_weights (coarsening.hpp:83-84) and a StrengthGraph from an
// externally supplied S pattern (StrengthGraph::from_pattern).
void pmisr_with_weights(Ctx& c, const Strength& g, int64_t max_loops, const double* d_w,
                        uint8_t* d_labels);
void strength_from_pattern(Ctx& c, const Csr& s, Strength& g);
// PMIS / PMIS-swap (coarsening.cpp:169-217): MIS rounds on S u S^T with the
// (|S_i| + |S_i^T|) + uniform weights; swap exchanges C and F at the end
void pmis(Ctx& c, const Strength& g, bool swap, uint64_t seed, uint8_t* d_labels);

struct LabelMap {
  int32_t n = 0, nf = 0, nc = 0;
  DBuf<uint8_t> label;
  DBuf<int32_t> fine_to_sub, f_to_fine, c_to_fine;
};
void build_label_map(Ctx& c, const uint8_t* d_labels, int32_t n, LabelMap& map);

struct Blocks {
  Csr aff, afc, acf;
  Csr af;  // A's F rows with global columns; bit 31 of a column flags a C column
};
void extract_blocks(Ctx& c, const Csr& a, const LabelMap& map, Blocks& out, bool want_af);
void extract_block_rows(Ctx& c, const Csr& a, int rb, const LabelMap& map, int fb, int fe, int cb, int ce,
                        Blocks& out, bool want_af);

struct DdcResult {
  int64_t converted = 0;
  double max_theta = 0.0, alpha_diag = 0.0;
};
// dominance_report + ddc (coarsening.cpp:219-330) on the F rows of a_ff;
// converts labels in d_labels (global rows). selection 0 histogram,
// 1 quickselect (unsupported on GPU), 2 direct.
DdcResult ddc(Ctx& c, const Csr& aff, const LabelMap& map, uint8_t* d_labels, double fraction,
              int64_t bins, int selection, double direct_alpha, bool convert);
// The whole PMISR-DDC split (weight mode 0) in seven sync-free passes over A
// (cfsplit.cu); labels bit-identical to strength -> pmisr -> extract -> ddc.
struct CfFused {
  int64_t s_nnz = 0, n_f_pre = 0, n_converted = 0;
  double max_theta = 0.0, alpha_diag = 0.0;
};
CfFused cf_split_fused(Ctx& c, const Csr& a, double alpha, uint64_t seed, bool ddc_enabled,
                       double fraction, int64_t bins, uint8_t* d_labels, uint8_t* d_labels_pre);
// The same split without the readback: the 8 report counters land in
// d_u_out (or stay in the context scratch when d_u_out is null; the pointer
// used is returned, null for an empty matrix without d_u_out); the finish
// step turns the host copy of the counters into the report and raises the
// zero-diagonal error. Lets several splits share one synchronisation.
// d_zeroed (optional, with d_u_out zeroed too): a region of
// cf_split_zero_bytes() bytes the caller has zeroed -- the split's counters,
// histogram, counts and marks live there and no zeroing kernel is launched
// (a batch zeroes every level's region with one memset).
const unsigned long long* cf_split_fused_enqueue(Ctx& c, const Csr& a, double alpha, uint64_t seed,
                                                 bool ddc_enabled, double fraction, int64_t bins,
                                                 uint8_t* d_labels, uint8_t* d_labels_pre,
                                                 unsigned long long* d_u_out, void* d_zeroed = nullptr);
size_t cf_split_zero_bytes(int64_t n, bool ddc_enabled, int64_t bins);
CfFused cf_split_fused_finish(Ctx& c, const unsigned long long* hu, bool ddc_enabled, const uint8_t* d_labels);
// coarsening.cpp:290-315 on device counters: d_out = {alpha_diag, max_theta}
void launch_ddc_select(Ctx& c, const unsigned long long* d_nf, const unsigned long long* d_hist, int64_t bins,
                       double fraction, const unsigned long long* d_maxbits, double* d_out);
// max theta only (theta_post, air.cpp:355); throws on a zero diagonal
double dominance_max(Ctx& c, const Csr& aff, int rb = 0);
double dominance_report(Ctx& c, const Csr& aff, int64_t bins, double* d_theta, int64_t* h_hist);  // rb: F rows of a slab

// poly.cu ---------------------------------------------------------------------
struct PolyFit {
  std::vector<double> coeffs;  // m values
  int64_t effective_order = 0;
};
struct RowSplit;  // rowsplit.cuh: row-partitioned setup work over ranks (nullable)
PolyFit poly_coefficients(Ctx& c, const Csr& a, int64_t m, uint64_t seed, const RowSplit* rs = nullptr);
void poly_assemble(Ctx& c, const Csr& a, const double* h_coeffs, int64_t ncoeffs, int64_t deg,
                   int64_t sparsity_order, Csr& out, const RowSplit* rs = nullptr);
double smoother_growth(Ctx& c, const Csr& a, const Csr& q, const RowSplit* rs = nullptr);
// pieces of the fit for a row-distributed operator (dsetup.cu): the power
// basis start (standard normals of global rows base..), one double-double
// SpMV of local rows, the Gram matrix of n local rows, the host fit
void poly_basis_fill(Ctx& c, int64_t n, int64_t base, uint64_t seed, double* hi, double* lo);
void poly_dd_spmv(Ctx& c, const Csr& a, const double* xh, const double* xl, double* yh, double* yl);
void poly_gram(Ctx& c, int64_t n, int nc, const double* kh, const double* kl, std::vector<dd>& G);
PolyFit poly_fit_gram(const std::vector<dd>& G, int nc, int64_t m, int64_t n);
// sparsity-1 assembly of rows rb..rb+n of a (pattern = row + diagonal, in
// a's column space; columns outside a's rows must not occur in the pattern)
void poly_assemble_rows(Ctx& c, const Csr& a, int rb, int n, const double* h_coeffs, int64_t ncoeffs,
                        int64_t deg, Csr& out);

// transfer.cu -----------------------------------------------------------------
// R rows of the C points of acf (coarse rows cb..; whole operator: cb = 0);
// bmap: row of ffinv holding each F column (gathered rows), null = identity
void build_restriction(Ctx& c, const Csr& acf, const Csr& ffinv, double drop, const LabelMap& map,
                       Csr& r, const int32_t* bmap = nullptr, int cb = 0, const RowSplit* rs = nullptr);
// R rows [Z | I] from the rows of Z = A_cf Aff^-1: Z's columns mapped by
// f2f (null: already fine indices), the identity at c2f[row]
void restriction_from_z(Ctx& c, const Csr& z, const int32_t* f2f, const int32_t* c2f, int64_t ncols, Csr& r);
// one-point map of the rows of a (row i = column i: own rows first in a
// local layout), label / f2s per column (f2s: coarse index of C columns)
void prolongation_map_fused(Ctx& c, const uint8_t* label, const int32_t* f2s, const Csr& a, double alpha,
                            int32_t* pmap);
// one-point P (air.cpp:191-238) as pmap[i] (coarse index or -1) and a CSR.
// one-point P of the slab rows rb.. of `a` (S of the same rows, global map)
void prolongation_map_rows(Ctx& c, const LabelMap& map, const Strength& g, const Csr& a, int rb,
                           int32_t* pmap);
// the n x nc CSR of a one-point map (-1 = empty row)
void prolongation_from_map(Ctx& c, const int32_t* pmap, int n, int nc, Csr& p);
void build_prolongation(Ctx& c, const LabelMap& map, const Strength& g, const Csr& a,
                        DBuf<int32_t>& pmap, Csr& p);
// the same P with the strength test re-applied to A's rows (no S)
void build_prolongation_fused(Ctx& c, const LabelMap& map, const Csr& a, double alpha, DBuf<int32_t>& pmap,
                              Csr& p);

}  // namespace airg
