// Row-partitioned setup work over P ranks (SURVEY §8e "setup collectives").
//
// The distributed setup keeps every level's operators replicated on every
// rank (180 GB of HBM holds C4 at 8 GPUs many times over) and splits the
// WORK: each heavy row kernel of the setup -- the SpGEMMs of Z = A_cf Aff^-1,
// A P and R (A P), the fixed-sparsity polynomial assembly, the power-basis
// and growth-estimate SpMVs -- runs on one contiguous row slab per rank, and
// the slabs are all-gathered (NCCL grouped broadcasts over NVLink; in the
// one-process emulation every "rank" writes its slab in place). Each row is
// computed by the same kernel with the same arithmetic as on one GPU, and
// every reduction (Gram matrix, norms) runs on the gathered, replicated
// vectors, so the distributed hierarchy is bit-identical to the one-GPU one
// for every P, in native mode included.
#pragma once

#include <nccl.h>

#include <vector>

#include "sparse.cuh"

namespace airg {

struct RowSplit {
  int P = 1;
  int me = -1;  // -1: emulate all P ranks in this process
  ncclComm_t comm = nullptr;
  bool mine(int r) const { return me < 0 || me == r; }
  // balanced contiguous slabs of n rows (starts, P + 1 entries)
  std::vector<int64_t> slabs(int64_t n) const;
  // make y[s[r]:s[r+1]] of every rank r present on every rank (doubles / ints / bytes)
  void gather_vec(Ctx& c, double* y, const std::vector<int64_t>& s) const;
  void gather_vec(Ctx& c, int32_t* y, const std::vector<int64_t>& s) const;
  void gather_vec(Ctx& c, uint8_t* y, const std::vector<int64_t>& s) const;
};

// Row slabs of one matrix for the ranks this process runs (emulation: all).
struct RowSlices {
  std::vector<int64_t> s;
  std::vector<Csr> part;  // part[r]: rows s[r]..s[r+1], global columns
  void build(Ctx& c, const RowSplit& rs, const Csr& a);
};

// y = A x with x and y full vectors on every rank: each rank computes its
// slab (exact SpMV kernel) and the slabs are gathered.
void split_spmv(Ctx& c, const RowSplit& rs, const RowSlices& a, const double* x, double* y);

// The rows of C = A B (optionally dropped, square rule) computed slab by
// slab and gathered into the full C on every rank.
void split_spgemm(Ctx& c, const RowSplit& rs, const Csr& a, const Csr& b, Csr& out, double drop_tol,
                  bool keep_diag);

// Gather per-rank row slabs (rows s[r]..s[r+1] in slab[r]) into one CSR with
// `ncols` columns on every rank.
void gather_csr(Ctx& c, const RowSplit& rs, const std::vector<int64_t>& s, std::vector<Csr>& slab,
                int64_t ncols, Csr& out);

// rows lo..hi of a (global columns)
void csr_slice(Ctx& c, const Csr& a, int64_t lo, int64_t hi, Csr& out);

}  // namespace airg
