// Halo exchange by NVLink peer stores (AIRG_TRANSPORT=p2p; see dist.cuh).
//
// Each rank keeps ALL its exchanged vectors ([own | halo] buffers) and two
// counter tables in one cudaMalloc'd arena whose IPC handle the other ranks
// open, so every rank can address every peer's halo slots directly. The
// arena layout is a pure function of the halo plans, which every rank holds
// for every rank, so no address tables are exchanged -- only the handles.
//
// Per vector ("slot") and ordered pair (owner o -> consumer q):
//   F[slot][o] in q's arena  -- deliveries from o (o increments it remotely)
//   A[slot][q] in o's arena  -- deliveries q has consumed (q increments it)
// exchange(V) is ONE kernel per rank (k_p2p_exchange):
//   1. the acks this rank owes (slots it finished reading since its last
//      exchange) go out as release adds on the owners' A counters;
//   2. wait until A[slot][q] == my pushes of V so far for every receiver q
//      (q is done with the previous contents), store my entries of q's halo
//      into q's buffer, fence at system scope, and the last CTA bumps
//      F[slot][me] at every receiver with a release add;
//   3. CTA 0 spins (acquire) until F[slot][o] reaches its receive count + 1
//      for every owner o; the consuming kernel runs after this grid.
// release(V), after the consuming kernel, only records the acks; the next
// exchange (or the flush closing a captured body) emits them. Every rank
// issues the same exchange sequence and phase 1 never waits, so a wait only
// depends on pushes and acks its peers issue earlier in their own streams:
// no circular wait. Emulation (all ranks on one GPU, one stream) launches the
// phases separately: all acks, then all pushes, then all waits, so no wait
// ever blocks. The values moved are copies: the V-cycle stays bit-identical.
#include <cstring>

#include "dist.cuh"

namespace airg {

#define P2P_NCCL(x)                                                            \
  do {                                                                         \
    ncclResult_t r__ = (x);                                                    \
    if (r__ != ncclSuccess)                                                    \
      throw CudaError(std::string("NCCL error: ") + ncclGetErrorString(r__)); \
  } while (0)

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// bounded spin (a lost peer traps instead of hanging the device)
__device__ __forceinline__ void spin_geq(const unsigned long long* p, unsigned long long target) {
  unsigned ns = 32;
  unsigned long long it = 0;
  while (ld_acquire_sys(p) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (++it > (1ull << 26)) __trap();
  }
}

__global__ void k_p2p_exchange(const __grid_constant__ P2PExch E) {
  pdl_wait();
  if ((E.phases & 1) && blockIdx.x == 0)
    for (int t = threadIdx.x; t < E.nack; t += blockDim.x) red_release_sys_add(E.ack_out[t], 1ull);
  if (E.phases & 2) {
    const unsigned long long done = *E.sends;  // my pushes of this vector so far
    if ((int)threadIdx.x < E.npeer) spin_geq(E.ack[threadIdx.x], done);
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < E.ns;
         k += (int64_t)gridDim.x * blockDim.x)
      *E.dst[k] = E.src[E.idx[k]];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(E.blocks, 1u) == gridDim.x - 1) {  // last CTA
      __threadfence_system();
      *E.blocks = 0;
      for (int p = 0; p < E.npeer; ++p) red_release_sys_add(E.remote_flag[p], 1ull);
      *E.sends = done + 1;
    }
  }
  if ((E.phases & 4) && blockIdx.x == 0) {
    const unsigned long long target = *E.recvs + 1;
    if ((int)threadIdx.x < E.nsrc) spin_geq(E.flag[threadIdx.x], target);
    __syncthreads();
    if (threadIdx.x == 0) *E.recvs = target;
  }
  pdl_trigger();
}

void launch_exchange(Ctx& c, const P2PExch& E) {
  const unsigned grid =
      (E.phases & 2) ? (unsigned)std::min<int64_t>(blocks_for(E.ns, 256), 2 * c.num_sms) : 1u;
  LAUNCH_PDL(c, k_p2p_exchange, grid, 256, 0, E);
}

// phase-1 launches for the acks of rank r (in chunks of kP2PMaxAcks)
void emit_acks(Ctx& c, std::vector<unsigned long long*>& acks) {
  for (size_t i = 0; i < acks.size(); i += kP2PMaxAcks) {
    P2PExch E;
    E.phases = 1;
    E.nack = (int)std::min<size_t>(kP2PMaxAcks, acks.size() - i);
    for (int k = 0; k < E.nack; ++k) E.ack_out[k] = acks[i + k];
    launch_exchange(c, E);
  }
  acks.clear();
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// arena of rank r: every vector's [own | halo] buffer, then F and A tables
struct Layout {
  std::vector<size_t> buf;
  size_t f = 0, a = 0, bytes = 0;
};
Layout layout(const std::vector<DVec*>& vecs, int r, int P) {
  Layout L;
  size_t cur = 0;
  for (const DVec* V : vecs) {
    cur = align_up(cur);
    L.buf.push_back(cur);
    const DVec::Rank& R = V->rk[r];
    cur += sizeof(double) * (size_t)std::max<int64_t>(1, R.own + R.nhalo);
  }
  L.f = align_up(cur);
  L.a = L.f + sizeof(unsigned long long) * vecs.size() * (size_t)P;
  L.bytes = align_up(L.a + sizeof(unsigned long long) * vecs.size() * (size_t)P);
  return L;
}

}  // namespace

void p2p_push_plan(const std::vector<int64_t>& recv_halo, int64_t recv_own, int64_t recv_off,
                   int64_t send_lo, int64_t send_own, std::vector<int32_t>& src_idx,
                   std::vector<int64_t>& dst_pos) {
  src_idx.clear();
  dst_pos.clear();
  // the receiver's halo is sorted and the owners' slabs are contiguous, so my
  // entries form one run starting at its receive offset for me
  for (int64_t g : recv_halo) {
    if (g < send_lo || g >= send_lo + send_own) continue;
    dst_pos.push_back(recv_own + recv_off + (int64_t)src_idx.size());
    src_idx.push_back((int32_t)(g - send_lo));
  }
}

bool p2p_requested() {
  static const bool v = [] {
    const char* e = getenv("AIRG_TRANSPORT");
    return e && !strcmp(e, "p2p");
  }();
  return v;
}

void p2p_setup(Ctx& c, DHier& d, const std::vector<DVec*>& vecs) {
  const int P = d.P;
  if (P > kP2PMaxPeers) throw InvalidArgument("dist: the p2p transport handles at most 32 ranks");
  DHier::P2PState& S = d.p2p;
  S.on = true;
  S.nslots = (int)vecs.size();
  for (int i = 0; i < S.nslots; ++i) vecs[i]->slot = i;
  std::vector<Layout> lay;
  for (int r = 0; r < P; ++r) lay.push_back(layout(vecs, r, P));
  S.base.assign(P, nullptr);
  S.owned.assign(P, 0);
  for (int r = 0; r < P; ++r) {
    if (!d.mine(r)) continue;
    CUDA_CHECK(cudaMalloc(&S.base[r], lay[r].bytes));  // plain cudaMalloc: IPC-exportable
    S.owned[r] = 1;
    CUDA_CHECK(cudaMemsetAsync(S.base[r], 0, lay[r].bytes, c.stream));
  }
  if (d.me >= 0) {  // one process per GPU: exchange the arena handles, open the peers'
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    cudaIpcMemHandle_t mine;
    CUDA_CHECK(cudaIpcGetMemHandle(&mine, S.base[d.me]));
    DBuf<char> all(c, sizeof(cudaIpcMemHandle_t) * (size_t)P);
    to_device(c, all.p + sizeof(cudaIpcMemHandle_t) * d.me, reinterpret_cast<const char*>(&mine), sizeof mine);
    P2P_NCCL(ncclAllGather(all.p + sizeof(cudaIpcMemHandle_t) * d.me, all.p, sizeof(cudaIpcMemHandle_t),
                           ncclChar, d.comm, c.stream));
    std::vector<cudaIpcMemHandle_t> hs(P);
    to_host(c, reinterpret_cast<char*>(hs.data()), all.p, sizeof(cudaIpcMemHandle_t) * (size_t)P);
    for (int q = 0; q < P; ++q) {
      if (q == d.me) continue;
      CUDA_CHECK(cudaIpcOpenMemHandle(&S.base[q], hs[q], cudaIpcMemLazyEnablePeerAccess));
    }
  }  // emulation: every arena is local
  auto at = [&](int r, size_t off) { return static_cast<char*>(S.base[r]) + off; };
  auto F = [&](int r, int slot, int from) {
    return reinterpret_cast<unsigned long long*>(at(r, lay[r].f)) + (size_t)slot * P + from;
  };
  auto A = [&](int r, int slot, int by) {
    return reinterpret_cast<unsigned long long*>(at(r, lay[r].a)) + (size_t)slot * P + by;
  };
  // per local rank: [slot] sends then [slot] receives; CTA counters per slot
  S.pending.assign(P, {});
  S.ctr.alloc(c, (size_t)2 * S.nslots * P);
  S.ctr.zero(c);
  S.blocks.alloc(c, (size_t)S.nslots * P);
  S.blocks.zero(c);
  for (DVec* Vp : vecs) {
    DVec& V = *Vp;
    const int slot = V.slot;
    std::vector<double*> bases(P, nullptr);
    for (int r = 0; r < P; ++r) {
      DVec::Rank& R = V.rk[r];
      if (d.mine(r)) {
        R.buf.view(reinterpret_cast<double*>(at(r, lay[r].buf[slot])), (size_t)std::max<int64_t>(1, R.own + R.nhalo));
        bases[r] = R.buf.p;
      }
    }
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r)) continue;
      DVec::Rank& R = V.rk[r];
      // sender side: my entries of every peer's halo, in the peer's halo order
      std::vector<int32_t> idx;
      std::vector<double*> dst;
      P2PExch& E = R.exch;
      E = P2PExch();
      for (int q = 0; q < P; ++q) {
        if (q == r) continue;
        const DVec::Rank& Q = V.rk[q];
        const int64_t cnt = Q.recv_cnt.empty() ? 0 : Q.recv_cnt[r];
        if (!cnt) continue;
        double* qbuf = reinterpret_cast<double*>(at(q, lay[q].buf[slot]));
        std::vector<int32_t> si;
        std::vector<int64_t> pos;
        p2p_push_plan(Q.halo_host, Q.own, Q.recv_off[r], R.lo, R.own, si, pos);
        if ((int64_t)si.size() != cnt) throw RuntimeError("p2p: send list does not match the receiver's halo plan");
        for (size_t k = 0; k < si.size(); ++k) {
          idx.push_back(si[k]);
          dst.push_back(qbuf + pos[k]);
        }
        E.remote_flag[E.npeer] = F(q, slot, r);
        E.ack[E.npeer] = A(r, slot, q);
        E.npeer++;
      }
      R.p2p_idx.alloc(c, std::max<size_t>(1, idx.size()));
      R.p2p_dst.alloc(c, std::max<size_t>(1, dst.size()));
      to_device(c, R.p2p_idx.p, idx.data(), idx.size());
      to_device(c, R.p2p_dst.p, dst.data(), dst.size());
      E.ns = (int64_t)idx.size();
      E.idx = R.p2p_idx.p;
      E.dst = R.p2p_dst.p;
      E.src = R.buf.p;
      E.sends = S.ctr.p + (size_t)2 * S.nslots * r + slot;
      E.blocks = S.blocks.p + (size_t)S.nslots * r + slot;
      E.phases = (E.ns ? 2 : 0);
      // consumer side: every owner I receive from
      R.release_to.clear();
      for (int o = 0; o < P; ++o) {
        if (o == r || R.recv_cnt.empty() || !R.recv_cnt[o]) continue;
        E.flag[E.nsrc++] = F(r, slot, o);
        R.release_to.push_back(A(o, slot, r));
      }
      if (E.nsrc) E.phases |= 4;
      E.recvs = S.ctr.p + (size_t)2 * S.nslots * r + S.nslots + slot;
    }
    if (d.me < 0) {
      V.bases.alloc(c, (size_t)P);
      to_device(c, V.bases.p, bases.data(), (size_t)P);
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

void p2p_exchange(Ctx& c, DHier& d, DVec& V) {
  DHier::P2PState& S = d.p2p;
  if (d.me >= 0) {  // one process per GPU: the three phases in one kernel
    P2PExch E = V.rk[d.me].exch;
    std::vector<unsigned long long*>& acks = S.pending[d.me];
    if (acks.size() > (size_t)kP2PMaxAcks) emit_acks(c, acks);  // rare: many slots released
    E.nack = (int)acks.size();
    for (int k = 0; k < E.nack; ++k) E.ack_out[k] = acks[k];
    if (E.nack) E.phases |= 1;
    acks.clear();
    if (E.phases) launch_exchange(c, E);
    return;
  }
  // emulation: all acks, then all pushes, then all waits
  for (int r = 0; r < d.P; ++r) emit_acks(c, S.pending[r]);
  for (int r = 0; r < d.P; ++r) {
    P2PExch E = V.rk[r].exch;
    E.phases &= 2;
    if (E.phases) launch_exchange(c, E);
  }
  for (int r = 0; r < d.P; ++r) {
    P2PExch E = V.rk[r].exch;
    E.phases &= 4;
    if (E.phases) launch_exchange(c, E);
  }
}

void p2p_release(Ctx& c, DHier& d, DVec& V) {
  (void)c;
  for (int r = 0; r < d.P; ++r)
    if (d.mine(r)) {
      const std::vector<unsigned long long*>& to = V.rk[r].release_to;
      d.p2p.pending[r].insert(d.p2p.pending[r].end(), to.begin(), to.end());
    }
}

void p2p_flush(Ctx& c, DHier& d) {
  if (!d.p2p.on) return;
  for (int r = 0; r < d.P; ++r)
    if (d.mine(r)) emit_acks(c, d.p2p.pending[r]);
}

void p2p_free(DHier& d) {
  DHier::P2PState& S = d.p2p;
  for (size_t r = 0; r < S.base.size(); ++r) {
    if (!S.base[r]) continue;
    if (S.owned[r])
      cudaFree(S.base[r]);
    else
      cudaIpcCloseMemHandle(S.base[r]);
    S.base[r] = nullptr;
  }
}

DHier::~DHier() {
  if (gm_flag) cudaFreeHost(gm_flag);
  if (graph) cudaGraphExecDestroy(graph);
  if (graph_vc) cudaGraphExecDestroy(graph_vc);
  p2p_free(*this);
}

}  // namespace airg
