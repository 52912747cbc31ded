// Row-slab distributed AIRG solve.
//
// Every level's index spaces (fine rows, F points) are split into contiguous
// slabs over the active ranks; each operator's rows live with the owner of
// its output rows and read its input vector through a per-rank halo (the
// remote entries its rows reference, grouped by owner). Row order and the
// order of entries inside a row are untouched, only column indices are
// remapped to the [owned | halo] local layout, so every row product is the
// same sequential, separately rounded sum as on one GPU: the distributed
// V-cycle is bit-identical to the single-GPU one (and to the reference).
//
// Active-GPU reduction follows the reference's replay rule
// (partition_model.cpp:77-112): level by level, when the mean local /
// non-local nnz ratio of the balanced partition drops below the threshold,
// the active ranks halve by merging adjacent slabs (rank 2k keeps both). The
// coarsest grid is gathered onto rank 0 for the polynomial coarse solve.
//
// Transport: kEmulate keeps all P ranks in one process on one GPU and runs
// them phase by phase (no kernel ever waits on another rank); the halo
// exchange is a gather kernel reading the owners' buffers. kNccl runs one
// rank per process/GPU and exchanges halos with grouped ncclSend/ncclRecv
// and reduces norms with ncclAllReduce. AIRG_TRANSPORT=p2p replaces the
// solve's halo exchanges by NVLink peer stores (halo_p2p.cuh): every rank's
// vector buffers live in one IPC-shared arena, owners push halo entries
// straight into the consumers' halo slots and signal per-slot counters; the
// same protocol runs in emulation with the "peers" on one GPU.
#pragma once

#include <nccl.h>

#include "hier.cuh"

namespace airg {

// ---- NVLink peer-store halo exchange (parameter block of halo_p2p.cu) ----
constexpr int kP2PMaxPeers = 32;
constexpr int kP2PMaxAcks = 64;
// One exchange of one vector on one rank, as ONE kernel: (1) hand back the
// halo slots this rank has finished reading since its last exchange
// ("consumed" acks to their owners), (2) wait until every receiver has
// consumed my previous push of this vector, store my entries of their halos
// into their buffers and signal "delivered", (3) wait for every owner's
// delivery into my halo. Emulation runs the phases as separate launches
// (all ranks share one stream).
struct P2PExch {
  int phases = 0;  // 1 acks, 2 push, 4 wait
  int nack = 0;
  unsigned long long* ack_out[kP2PMaxAcks] = {};
  // push
  int64_t ns = 0;
  const int32_t* idx = nullptr;  // owned local index per pushed entry
  double* const* dst = nullptr;  // destination per entry (a peer's halo slot)
  const double* src = nullptr;   // my [own | halo] buffer
  int npeer = 0;
  unsigned long long* remote_flag[kP2PMaxPeers] = {};  // "delivered" counter in each receiver's arena
  const unsigned long long* ack[kP2PMaxPeers] = {};    // "consumed" counter per receiver in my arena
  unsigned long long* sends = nullptr;                 // completed pushes of this vector
  unsigned* blocks = nullptr;                          // CTA arrivals (self-resetting)
  // wait
  int nsrc = 0;
  const unsigned long long* flag[kP2PMaxPeers] = {};   // "delivered" counters in my arena
  unsigned long long* recvs = nullptr;                 // deliveries consumed so far
};

struct Part {
  std::vector<int64_t> s;  // P + 1 starts
  int P() const { return (int)s.size() - 1; }
  int64_t lo(int r) const { return s[r]; }
  int64_t cnt(int r) const { return s[r + 1] - s[r]; }
  int owner(int64_t g) const;
};

// A vector over one partitioned index space, with a halo plan per rank.
struct DVec {
  Part part;
  int64_t N = 0;
  struct Rank {
    int64_t own = 0, lo = 0, nhalo = 0;
    DBuf<int32_t> halo;              // sorted global indices of the halo
    std::vector<int64_t> halo_host;  // same, host copy (plan building)
    DBuf<double> buf;                // [own | halo]
    // emulation: owner rank and owner-local index per halo entry
    DBuf<int32_t> src_rank, src_idx;
    // nccl: per-peer receive segments and send lists
    std::vector<int64_t> recv_off, recv_cnt, send_off, send_cnt;
    DBuf<int32_t> send_idx;
    DBuf<double> send_buf;
    // p2p: pushed entries (index, destination), the exchange parameter block
    // and the "consumed" counters of my owners to bump after reading
    DBuf<int32_t> p2p_idx;
    DBuf<double*> p2p_dst;
    P2PExch exch;
    std::vector<unsigned long long*> release_to;
  };
  std::vector<Rank> rk;
  DBuf<double*> bases;  // emulation: buf pointer per rank
  int slot = -1;        // p2p: index of this vector's counters (-1: not exchanged by p2p)
};

struct DLevel {
  Part fine, coarse_part, fpart;  // partitions of level l rows, level l+1 rows, F points
  int active = 1;
  double ratio_before = 0.0, ratio_after = 0.0;
  double share_before = 1.0, share_after = 1.0;  // local_share (partition_model.cpp:66-75)
  bool triggered = false;
  DVec B, X, RF;  // b_l (input of R_l), x_l (input of AF/AFFg and of P_{l-1}), r_F
  int64_t nnz_afp = 0, nnz_w = 0;  // fast V-cycle: global entries of A_F P and W_k
  struct Rank {
    Csr R, AF, AFFG, FINV;    // local rows, remapped columns
    Csr AFP, W;               // fast V-cycle: A_F P (-> X_{l+1} layout), W_k (-> RF layout); F rows
    DBuf<int32_t> pmap, f2f;  // prolongation map (-> X_{l+1} layout), F row -> local fine row
    DBuf<int32_t> c2f;        // fast V-cycle: the own C rows (local fine rows)
    int64_t nc_own = 0;
    DBuf<double> sc;
    int64_t nf_own = 0, n_own = 0;
  };
  std::vector<Rank> rk;
};

struct DHier {
  int P = 1;
  int me = -1;  // -1: emulate all ranks in this process
  ncclComm_t comm = nullptr;
  double threshold = 2.0;
  std::vector<DLevel> lv;
  int64_t fused_smooths = -1;  // up_f_smooths of the fast V-cycle's A_F P / W_k slabs (-1: none)
  int64_t coarse_e_its = -1;   // coarse_iterations the composed coarse solve was built for
  bool coarse_e_ok = false;    // ... and whether it is used
  Part cpart;            // coarsest rows (gathered on rank 0)
  DVec CB, CX, CR, XS;   // coarse b / e / r and the top solution vector
  struct Rank {
    Csr A0, AC, ACI;     // top operator (residual), coarse operator and its inverse
    Csr ACE;             // fast V-cycle: the composed coarse solve E_k (coarse owner)
    DBuf<double> rhs;    // owned part of b
  };
  std::vector<Rank> rk;
  DBuf<double> part;     // residual partial sums (all local ranks)
  DBuf<double> scal;
  std::vector<int> part_off;  // per local rank offset into part
  int nparts = 0;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_key = -1;
  uint64_t graph_kernels = 0;
  // outer GMRES (dist_gmres): the captured V-cycle alone, and per local rank
  // the Krylov basis V, Z = M V, w, x and the dot outputs
  cudaGraphExec_t graph_vc = nullptr;
  int64_t graph_vc_key = -1;
  uint64_t graph_vc_kernels = 0;
  struct GmRank {
    DBuf<double> V, Z, w, x, dots, part;
    // device-resident form (dist_gmres_dev): the GMRES state and scalars of
    // this rank (identical on every rank: the reductions are allreduced)
    DBuf<GmDev> st;
    DBuf<double> H, cs, sn, g, y, hb, G, hist, gpart, sc;
  };
  std::vector<GmRank> gm;
  int gm_m = 0;
  int* gm_flag = nullptr;  // pinned: the lagged "inner loop continues" flags of the device GMRES
  int64_t top_n = 0;
  // owned setup (dist_setup_owned): per-level reports, identical on every rank
  struct Summary {
    int64_t n = 0, nnz = 0, nf = 0, nc = 0, n_f_pre = 0, n_converted = 0;
    int64_t nnz_ff = 0, nnz_fc = 0, nnz_cf = 0, nnz_ffinv = 0, nnz_r = 0, nnz_p = 0;
    int64_t attempts = 1, eff = 0;
    double max_theta_pre = 0.0, alpha_diag = 0.0, max_theta_post = 0.0, growth = 0.0;
    std::vector<double> coeffs;
  };
  std::vector<Summary> summary;  // fine levels, then the coarse level (n, nnz, nnz_ffinv = |Ac^-1|, ...)
  bool owned = false;
  double setup_ms = 0.0, cf_ms = 0.0;  // owned setup: wall time, device time of the CF splits (this process)
  // p2p transport: one arena per rank (emulation: all allocated here; NCCL
  // ranks: mine allocated, the peers' opened from their IPC handles)
  struct P2PState {
    bool on = false;
    int nslots = 0;
    std::vector<void*> base;
    std::vector<char> owned;
    DBuf<unsigned long long> ctr;  // per local rank: [slot] sends | [slot] receives
    DBuf<unsigned> blocks;         // per local rank and slot: push CTA arrivals
    // per rank: acks recorded by release() and not yet emitted (enqueue time)
    std::vector<std::vector<unsigned long long*>> pending;
  } p2p;
  ~DHier();
  bool mine(int r) const { return me < 0 || me == r; }
};

// p2p transport (halo_p2p.cu): arenas, slot counters and parameter blocks for
// the solve's vectors; exchange / release of one vector
void p2p_setup(Ctx& c, DHier& d, const std::vector<DVec*>& vecs);
void p2p_exchange(Ctx& c, DHier& d, DVec& V);
void p2p_release(Ctx& c, DHier& d, DVec& V);
void p2p_flush(Ctx& c, DHier& d);  // emit every pending ack (end of a captured body)
void p2p_free(DHier& d);
bool p2p_requested();
// Host rule of the p2p push (also behind airg_p2p_push_plan_host for the CPU
// tests): the sender's entries of one receiver's sorted halo -- the sender's
// local index of each, and its position in the receiver's [own | halo]
// buffer (receiver own count + receive offset of the sender + k).
void p2p_push_plan(const std::vector<int64_t>& recv_halo, int64_t recv_own, int64_t recv_off,
                   int64_t send_lo, int64_t send_own, std::vector<int32_t>& src_idx,
                   std::vector<int64_t>& dst_pos);

#define NCCL_CHECK(x)                                                          \
  do {                                                                         \
    ncclResult_t r__ = (x);                                                    \
    if (r__ != ncclSuccess)                                                    \
      throw CudaError(std::string("NCCL error: ") + ncclGetErrorString(r__)); \
  } while (0)

// ---- partition and halo plumbing shared by the solve and the owned setup
// partition_rows (partition_model.cpp:8-22) on `active` logical ranks placed
// on every (P / active)-th physical rank; merged: adjacent logical pairs
// (partition_model.cpp:101-104); gathered: every row on rank 0
Part balanced(int64_t n, int active, int P);
Part merged(const Part& p, int active, int new_active);
Part gathered(int64_t n, int P);
// rows lo..hi of a (columns unchanged)
void slice(Ctx& c, const Csr& a, int64_t lo, int64_t hi, Csr& out);
// One rank's halo of a DVec from marks over the global index space.
struct Marks {
  DBuf<int32_t> m;
  int64_t N = 0;
  void init(Ctx& c, int64_t n);
  void cols(Ctx& c, const Csr& a, int64_t lo, int64_t hi);  // columns outside [lo, hi) (bit 31 ignored)
  void vals(Ctx& c, const int32_t* idx, int64_t n, int64_t lo, int64_t hi);
};
void set_halo(Ctx& c, DVec& V, int r, Marks& mk);
// buffers, emulation tables and NCCL send lists once the halos are set.
// peers_known: every rank's halo list is in V (all ranks planned here);
// otherwise (one rank per process, owned setup) each rank's requests travel
// to their owners over NCCL.
void finalize(Ctx& c, DVec& V, const DHier& d, bool peers_known = true);
// columns (global) -> V's [own | halo] layout of rank r
void remap(Ctx& c, Csr& a, const DVec& V, int r);
void exchange(Ctx& c, DHier& d, DVec& V);     // halo <- owners
void reverse_add(Ctx& c, DHier& d, DVec& V);  // owners += halo entries
void release(Ctx& c, DHier& d, DVec& V);

// Per-rank operator slices a distributed solve is built from (dist_build):
// rows of the ranks this process runs, global column indices.
struct DistPieces {
  struct LevelRank {
    Csr R;                    // rows of level l+1 owned here (coarse_part), fine columns
    Csr AF, AFFG, FINV;       // F rows owned here (fpart): A_F (bit 31 = C column), A_FF (fine columns), Aff^-1
    Csr AFP, W;               // fast V-cycle (optional): A_F P (global coarse columns), W_k (global F columns)
    DBuf<int32_t> pmap;       // own fine rows -> global coarse index (-1: empty row)
    DBuf<int32_t> f2f;        // own F rows -> global fine row
  };
  std::vector<std::vector<LevelRank>> lv;  // [level][rank]
  std::vector<Part> fpart;                 // F-point partition per level
  std::vector<int64_t> n, nf;              // global rows / F points per level
  std::vector<Csr> AC, ACI, A0;            // per rank: coarse rows (cpart), top rows (level-0 partition)
  int64_t coarse_n = 0;
  int64_t fused_smooths = -1;              // AFP / W present, built for this many F-smooths
  bool all_ranks = false;                  // pieces of every rank present (halo lists of peers known)
};
// The solve structures of d from pieces; d.P / me / comm / threshold and
// every level's partition (d.lv[l].fine, active, ratios) already set.
void dist_build(Ctx& c, DHier& d, DistPieces& pc);

void dist_create(Ctx& c, Hier& h, int P, int me, ncclComm_t comm, double threshold,
                 const int64_t* level0_starts, DHier& d);

// Owned-row distributed setup (dsetup.cu): every rank holds and builds only
// its rows of every level. a_rows[r]: rows starts[r].. of the fine operator
// with global columns (mine ranks). Setup summaries land in d.summary.
void dist_setup_owned(Ctx& c, std::vector<Csr>& a_rows, const std::vector<int64_t>& starts,
                      const airg_setup_config& cfg, const Injection* inj, int P, int me, ncclComm_t comm,
                      double threshold, DHier& d);
// halo bytes received by this process per V-cycle and per level-0 SpMV
void dist_halo_bytes(const DHier& d, const airg_solve_config& cfg, int64_t& vcycle, int64_t& spmv);
// d_b / d_x: global vectors in emulation mode, this rank's slab with NCCL
void dist_solve(Ctx& c, DHier& d, const airg_solve_config& cfg, const double* d_b, double* d_x,
                airg_solve_stats& st, std::vector<double>& history);

// Distributed PMISR-DDC CF split of a slab-partitioned operator (the paper's
// contribution at N GPUs): strength on own rows, |S^T| by a reverse halo sum,
// weights on the global row index, one forward exchange of halo weights, the
// "not minimal" marks of remote endpoints returned by a reverse exchange, and
// DDC with a global max / histogram (allreduce). Labels are bit-identical to
// the one-GPU split for every partition. d_labels: global (emulation) or
// this rank's slab (NCCL).
struct CfReport {
  int64_t n_f_pre = 0, n_f = 0, n_converted = 0, s_nnz = 0;
  double max_theta = 0.0, alpha_diag = 0.0;
};
void dist_cf_split(Ctx& c, const Csr& a_global, int P, int me, ncclComm_t comm,
                   const std::vector<int64_t>& starts, double alpha, int64_t max_loops, uint64_t seed,
                   bool ddc_enabled, double fraction, int64_t bins, uint8_t* d_labels,
                   CfReport& rep);

// The split on slabs whose halo plan V is finalized: loc[r] = rank r's rows
// with columns remapped to V's [own | halo] layout (mine ranks). On return
// labs[r] holds rank r's final labels (AIRG_F / AIRG_C as doubles) over
// [own | halo].
void cf_split_slabs(Ctx& c, DHier& d, DVec& V, std::vector<Csr>& loc, double alpha, uint64_t seed,
                    bool ddc_enabled, double fraction, int64_t bins, std::vector<DBuf<double>>& labs,
                    CfReport& rep);

// Host-side halo plan of one rank (same rule as the device build): the
// sorted distinct referenced indices outside the owned range, with the
// per-owner receive counts. Used by the CPU (gloo) tests of the N > 1 path.
void halo_plan_host(const std::vector<int64_t>& starts, int rank, const int64_t* cols,
                    int64_t ncols, std::vector<int64_t>& halo, std::vector<int64_t>& recv_cnt);

}  // namespace airg
