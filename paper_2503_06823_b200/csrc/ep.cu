// Expert parallelism over peer memory: the token dispatch is
// fused into the permute kernel (NVLink stores straight into the computing
// rank's receive buffer) and the return into GEMM2's epilogue (each expert
// output row stored straight into its source rank's own permuted layout), so
// the combine runs locally.  No all-to-all, no host synchronisation.
//
// Placement: every resident expert e is spread over a run of consecutive
// ranks with cumulative shares cum[e][q] (units of 2^-24; ep.plan_shares cuts
// the experts' expected loads, laid end to end in expert order, into one
// unit interval per rank).  Per forward, every rank derives from the
// replicated table of all ranks' counts the same split: e's rows, ordered by
// (source rank, local row), are cut at B_e(q) = pad * round(N_e/pad * cum[e][q]
// / 2^24) and rank q computes rows [B_e(q-1), B_e(q)).  A hot expert's rows
// are thereby shared by its ranks token by token (not source by source), so
// the busiest rank carries its share of the batch whatever the per-source
// skew.  Pieces are multiples of the segment padding, so every receive
// segment stays GEMM-tile aligned.
//
// Every rank allocates one symmetric region (same size everywhere) and maps
// every peer's region through CUDA IPC.  The layers of a stack share one
// region (emoe_ep_create's share_with), so the receive / expert-output / H
// buffers exist once per GPU, not once per layer:
//   flags    u64 [3 phases][kMaxPeers]   epoch written by each source rank
//   cnt      i32 [kMaxPeers][E]          real (unpadded) per-expert counts of every source
//   recv_x   bf16 [recv_cap][d]          rows dispatched to this rank
//   y_local  bf16 [rows_cap][d]          expert outputs of this rank's own rows,
//                                        in its local permuted layout
// One forward, all on the caller's stream:
//   K1 + K3a  route and scan locally (layer_route_scan)
//   bar0      publish this rank's counts to every peer, signal, wait for all
//             ranks, then derive from the replicated table the split, this
//             rank's receive segments (source, owned expert) with the row
//             shift of each back into its source's layout, and its send
//             pieces (per expert, per computing rank: local row end + shift)
//   K3b       permute_kernel<REMOTE>: rows -> computing rank's recv_x (peer stores)
//   bar1      signal + wait: every source finished writing to this rank
//   K4        grouped GEMMs over the (source, expert) segments of recv_x;
//             GEMM2's epilogue pushes each row to its source's y_local
//   bar2      signal + wait: every rank's pushes have landed
//   K5        combine_bf16_kernel over the local y_local (slot order)
// Every row meets the same GEMM arithmetic wherever it runs and the combine
// order is fixed at the source, so the output is bit-identical to EP=1.
// Buffer reuse across forwards (and across the layers sharing a region)
// needs no extra barrier: a source writes cnt / recv_x of forward n+1 only
// after its own bar2 of forward n, which every rank reaches only after its
// layout reads of forward n; GEMM2 of forward n+1 pushes into a source's
// y_local only after bar1 of n+1, i.e. after every rank finished its combine
// of forward n.  The epoch is per region, so consecutive layers' barriers
// never alias.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "capi_util.h"
#include "kernels.h"

namespace emoe {
namespace {

constexpr int kPhases = 3;
constexpr int kMaxE = 128;
constexpr int kShareBits = 24;  // cum shares are fixed point with 24 fraction bits
// stats: rows computed (padded), real rows sent to peers, real rows received
// from peers, real rows routed (this rank's tokens), real rows computed
constexpr int kStats = 5;

struct PeerSym {
  uint64_t* flags[kMaxPeers];
  int32_t* cnt[kMaxPeers];
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// signal this rank's arrival at `phase` on every peer, then wait for every
// peer's arrival on this rank (bounded: a peer that never arrives sets
// status = 1 after timeout_ns instead of hanging the GPU)
__device__ void barrier(const PeerSym& sym, int W, int rank, int phase, uint64_t epoch, uint64_t timeout_ns,
                        int* status) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < W; ++q) st_release_sys(sym.flags[q] + phase * kMaxPeers + rank, epoch);
  }
  if (threadIdx.x < W) {
    const uint64_t* f = sym.flags[rank] + phase * kMaxPeers + threadIdx.x;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(f) < epoch) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicExch(status, 1);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

struct LayoutArgs {
  const int32_t* counts;       // [E] this rank's real rows per expert
  const int64_t* seg_offsets;  // [E+1] this rank's padded local segments
  const int64_t* cum;          // [E][W] cumulative shares (-1: not resident)
  const int32_t* owned;        // [n_owned] experts this rank computes (ascending)
  int n_owned;
  int pad;
  int64_t recv_cap;
  int64_t* piece_end;    // [E][W] local row end of this rank's piece of e computed on rank q
  int64_t* piece_shift;  // [E][W] receive row on q = local row + shift
  int64_t* recv_segs;    // [W * n_owned + 1]
  int64_t* out_shift;    // [W * n_owned] receive row -> row in the source's layout
  int64_t* stats;        // [kStats]
};

// bar0: publish counts, barrier, then the split, the receive segments and the send pieces
__global__ void __launch_bounds__(256) ep_bar0_kernel(PeerSym sym, int W, int rank, int E, uint64_t epoch,
                                                      uint64_t timeout_ns, int* status, LayoutArgs a) {
  __shared__ int32_t cr[kMaxPeers][kMaxE];   // real counts [source][expert]
  __shared__ int64_t pre[kMaxPeers][kMaxE];  // rows of e held by earlier sources (padded)
  __shared__ int64_t loc[kMaxPeers][kMaxE];  // source's padded local segment offset of e
  __shared__ int64_t bnd[kMaxE][kMaxPeers];  // split ends B_e(q)
  __shared__ int64_t tot[kMaxPeers][kMaxPeers];  // [source][receiver] rows
  __shared__ unsigned long long st_sent, st_recv, st_routed;
  __shared__ int overflow;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int32_t v = a.counts[e];
    for (int q = 0; q < W; ++q) sym.cnt[q][rank * E + e] = v;
  }
  barrier(sym, W, rank, 0, epoch, timeout_ns, status);
  const int32_t* cnt = sym.cnt[rank];  // every source's counts, now local
  const int64_t pad = a.pad;
  for (int i = threadIdx.x; i < W * E; i += blockDim.x) cr[i / E][i % E] = cnt[i];
  if (threadIdx.x == 0) {
    overflow = 0;
    st_sent = st_recv = st_routed = 0;
  }
  __syncthreads();
  auto padded = [&](int s, int e) -> int64_t { return ((int64_t)cr[s][e] + pad - 1) / pad * pad; };
  // per expert: source prefixes and the split ends
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t n = 0;
    for (int s = 0; s < W; ++s) {
      pre[s][e] = n;
      n += padded(s, e);
    }
    const int64_t units = n / pad;
    for (int q = 0; q < W; ++q) {
      const int64_t c = a.cum[e * W + q];
      int64_t b = q == W - 1 || c < 0 ? n : pad * ((units * c + (1ll << (kShareBits - 1))) >> kShareBits);
      bnd[e][q] = b < n ? b : n;
    }
  }
  // per source: padded local offsets (its segments in expert order)
  for (int s = threadIdx.x; s < W; s += blockDim.x) {
    int64_t o = 0;
    for (int e = 0; e < E; ++e) {
      loc[s][e] = o;
      o += padded(s, e);
    }
  }
  __syncthreads();
  // rows of source s's segment e that rank q computes: [lo, hi) of e's global order
  auto piece = [&](int s, int e, int q, int64_t& lo, int64_t& hi) {
    const int64_t p0 = pre[s][e], p1 = p0 + padded(s, e);
    lo = max(p0, q > 0 ? bnd[e][q - 1] : (int64_t)0);
    hi = min(p1, bnd[e][q]);
    if (hi < lo) hi = lo;
  };
  if (threadIdx.x < W * W) {
    const int s = threadIdx.x / W, q = threadIdx.x % W;
    int64_t t = 0;
    for (int e = 0; e < E; ++e) {
      int64_t lo, hi;
      piece(s, e, q, lo, hi);
      t += hi - lo;
    }
    tot[s][q] = t;
  }
  __syncthreads();
  if (threadIdx.x < W) {
    int64_t t = 0;
    for (int s = 0; s < W; ++s) t += tot[s][threadIdx.x];
    if (t > a.recv_cap) overflow = 1;
  }
  __syncthreads();
  if (overflow) {  // every rank sees the same table: all drop the forward's rows and report status 2
    if (threadIdx.x == 0) atomicExch(status, 2);
    for (int i = threadIdx.x; i < E * W; i += blockDim.x) {
      a.piece_end[i] = a.seg_offsets[i / W];  // no row falls in any piece
      a.piece_shift[i] = 0;
    }
    for (int i = threadIdx.x; i <= W * a.n_owned; i += blockDim.x) a.recv_segs[i] = 0;
    if (threadIdx.x < kStats) a.stats[threadIdx.x] = 0;
    return;
  }
  // send pieces of this rank, one thread per computing rank q, experts in order
  if (threadIdx.x < W) {
    const int q = threadIdx.x;
    int64_t recv_off = 0;  // rows earlier sources send q, then this rank's earlier experts
    for (int s = 0; s < rank; ++s) recv_off += tot[s][q];
    for (int e = 0; e < E; ++e) {
      int64_t lo, hi;
      piece(rank, e, q, lo, hi);
      const int64_t p0 = pre[rank][e], seg = a.seg_offsets[e];
      const int64_t end_g = min(max(bnd[e][q], p0), p0 + padded(rank, e));
      a.piece_end[e * W + q] = seg + (end_g - p0);
      // local row r of the piece lands on receive row recv_off + (r - seg) - (lo - p0)
      a.piece_shift[e * W + q] = recv_off - seg - (lo - p0);
      recv_off += hi - lo;
      // real (unpadded) rows of the piece, for the exchange statistics
      const int64_t real = min(hi, p0 + (int64_t)cr[rank][e]) - lo;
      if (real > 0) {
        if (q != rank) atomicAdd(&st_sent, (unsigned long long)real);
        atomicAdd(&st_routed, (unsigned long long)real);
      }
    }
  }
  // receive segments of this rank: (source, owned expert) in order; the
  // return shift maps receive row r of segment (s, e) to row r + shift of
  // source s's layout
  if (threadIdx.x == 32) {
    int64_t off = 0;
    int i = 0;
    unsigned long long rr = 0, rc = 0;
    for (int s = 0; s < W; ++s)
      for (int j = 0; j < a.n_owned; ++j) {
        const int e = a.owned[j];
        int64_t lo, hi;
        piece(s, e, rank, lo, hi);
        a.recv_segs[i] = off;
        a.out_shift[i] = loc[s][e] + (lo - pre[s][e]) - off;
        ++i;
        off += hi - lo;
        const int64_t real = min(hi, pre[s][e] + (int64_t)cr[s][e]) - lo;
        if (real > 0) {
          if (s != rank) rr += (unsigned long long)real;
          rc += (unsigned long long)real;
        }
      }
    a.recv_segs[i] = off;
    a.stats[0] = off;
    a.stats[4] = (int64_t)rc;
    st_recv = rr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.stats[1] = (int64_t)st_sent;
    a.stats[2] = (int64_t)st_recv;
    a.stats[3] = (int64_t)st_routed;
  }
}


// NCCL chunk transport (ep.py NcclExpertParallelMoE): every (source,
// destination) pair owns a fixed chunk of `cap` rows in the send / receive /
// return buffers, so the all-to-all needs no host-side split sizes.  From the
// all-gathered count table (device), every rank derives the same split as
// ep_bar0_kernel, then: its send pieces into its send chunks (chunk q = rows
// [q cap, (q + 1) cap), pieces in expert order), and its receive segments
// (source, owned expert) in compact order with the shift of each into the
// receive chunks (which the return chunks mirror).  A pair over `cap` rows
// drops the forward's rows on every rank and sets status 2.
struct ChunkArgs {
  const int32_t* table;        // [W][E] real counts of every source (all-gathered)
  const int64_t* seg_offsets;  // [E+1] this rank's padded local segments
  const int64_t* cum;          // [E][W]
  const int32_t* owned;        // [n_owned]
  int n_owned, pad;
  int64_t cap;
  int64_t* piece_end;    // [E][W]
  int64_t* piece_shift;  // [E][W]: send-buffer row = local row + shift
  int64_t* recv_segs;    // [W * n_owned + 1] compact
  int64_t* a_shift;      // [W * n_owned]: receive-chunk row = compact row + shift
  int64_t* stats;        // [kStats]
  int* status;
};

__global__ void __launch_bounds__(256) epx_layout_kernel(int W, int rank, int E, ChunkArgs a) {
  __shared__ int32_t cr[kMaxPeers][kMaxE];
  __shared__ int64_t pre[kMaxPeers][kMaxE];
  __shared__ int64_t bnd[kMaxE][kMaxPeers];
  __shared__ int64_t tot[kMaxPeers][kMaxPeers];
  __shared__ int overflow;
  const int64_t pad = a.pad;
  for (int i = threadIdx.x; i < W * E; i += blockDim.x) cr[i / E][i % E] = a.table[i];
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  auto padded = [&](int s, int e) -> int64_t { return ((int64_t)cr[s][e] + pad - 1) / pad * pad; };
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t n = 0;
    for (int s = 0; s < W; ++s) {
      pre[s][e] = n;
      n += padded(s, e);
    }
    const int64_t units = n / pad;
    for (int q = 0; q < W; ++q) {
      const int64_t c = a.cum[e * W + q];
      int64_t b = q == W - 1 || c < 0 ? n : pad * ((units * c + (1ll << (kShareBits - 1))) >> kShareBits);
      bnd[e][q] = b < n ? b : n;
    }
  }
  __syncthreads();
  auto piece = [&](int s, int e, int q, int64_t& lo, int64_t& hi) {
    const int64_t p0 = pre[s][e], p1 = p0 + padded(s, e);
    lo = max(p0, q > 0 ? bnd[e][q - 1] : (int64_t)0);
    hi = min(p1, bnd[e][q]);
    if (hi < lo) hi = lo;
  };
  if (threadIdx.x < W * W) {
    const int s = threadIdx.x / W, q = threadIdx.x % W;
    int64_t t = 0;
    for (int e = 0; e < E; ++e) {
      int64_t lo, hi;
      piece(s, e, q, lo, hi);
      t += hi - lo;
    }
    tot[s][q] = t;
    if (t > a.cap) overflow = 1;  // benign race: every writer stores 1
  }
  __syncthreads();
  if (overflow) {
    if (threadIdx.x == 0) atomicExch(a.status, 2);
    for (int i = threadIdx.x; i < E * W; i += blockDim.x) {
      a.piece_end[i] = a.seg_offsets[i / W];
      a.piece_shift[i] = 0;
    }
    for (int i = threadIdx.x; i <= W * a.n_owned; i += blockDim.x) a.recv_segs[i] = 0;
    if (threadIdx.x < kStats) a.stats[threadIdx.x] = 0;
    return;
  }
  if (threadIdx.x < W) {  // send pieces into this rank's chunk for q
    const int q = threadIdx.x;
    int64_t off = 0;  // rows already placed in chunk q
    for (int e = 0; e < E; ++e) {
      int64_t lo, hi;
      piece(rank, e, q, lo, hi);
      const int64_t p0 = pre[rank][e], seg = a.seg_offsets[e];
      const int64_t end_g = min(max(bnd[e][q], p0), p0 + padded(rank, e));
      a.piece_end[e * W + q] = seg + (end_g - p0);
      a.piece_shift[e * W + q] = (int64_t)q * a.cap + off - seg - (lo - p0);
      off += hi - lo;
    }
  }
  if (threadIdx.x == 32) {  // receive segments: (source, owned expert), compact, shifted into chunk s
    int64_t off = 0;
    int i = 0;
    for (int s = 0; s < W; ++s) {
      int64_t in_chunk = 0;
      int j = 0;
      for (int e = 0; e < E; ++e) {
        int64_t lo, hi;
        piece(s, e, rank, lo, hi);
        if (j < a.n_owned && a.owned[j] == e) {
          a.recv_segs[i] = off;
          a.a_shift[i] = (int64_t)s * a.cap + in_chunk - off;
          ++i;
          ++j;
          off += hi - lo;
        }
        in_chunk += hi - lo;  // a non-owned expert has no rows for this rank
      }
    }
    a.recv_segs[i] = off;
    a.stats[0] = off;
  }
}

__global__ void ep_bar_kernel(PeerSym sym, int W, int rank, int phase, uint64_t epoch, uint64_t timeout_ns,
                              int* status) {
  barrier(sym, W, rank, phase, epoch, timeout_ns, status);
}

template <typename T>
T* dmalloc(size_t count) {
  T* p = nullptr;
  if (count) EMOE_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// The per-GPU symmetric region (shared by the layers of a stack).
struct EpRegion {
  int W = 1, rank = 0, E = 0, d = 0, f = 0, elem = 2;
  int64_t recv_cap = 0, rows_cap = 0;
  uint64_t epoch = 0, timeout_ns = 0;
  uint8_t* sym = nullptr;
  size_t sym_bytes = 0, off_cnt = 0, off_x = 0, off_y = 0;
  uint8_t* peer[kMaxPeers] = {};
  bool opened = false;
  void* h = nullptr;  // [recv_cap][f] GEMM1 output of the received rows
  int* status = nullptr;

  PeerSym peer_sym() const {
    PeerSym p{};
    for (int q = 0; q < W; ++q) {
      p.flags[q] = reinterpret_cast<uint64_t*>(peer[q]);
      p.cnt[q] = reinterpret_cast<int32_t*>(peer[q] + off_cnt);
    }
    return p;
  }
  ~EpRegion() {
    cudaDeviceSynchronize();
    for (int q = 0; q < W; ++q)
      if (peer[q] && peer[q] != sym) cudaIpcCloseMemHandle(peer[q]);
    for (void* p : {(void*)sym, h, (void*)status})
      if (p) cudaFree(p);
  }
};

}  // namespace
}  // namespace emoe

using namespace emoe;

struct emoe_ep {
  emoe_layer* layer = nullptr;
  LayerView v{};
  std::shared_ptr<EpRegion> R;
  std::vector<int64_t> cum;  // [E][W]
  std::vector<int32_t> owned;

  int64_t* cum_dev = nullptr;
  int32_t* owned_dev = nullptr;
  int64_t* piece_end = nullptr;
  int64_t* piece_shift = nullptr;
  int64_t* recv_segs = nullptr;
  int32_t* seg_expert = nullptr;  // [W * n_owned]
  int32_t* seg_rank = nullptr;    // [W * n_owned] source rank of each receive segment
  int64_t* out_shift = nullptr;   // [W * n_owned]
  int64_t* stats = nullptr;       // [kStats]

  // stage events: route, count exchange (bar0), dispatch (remote permute),
  // dispatch wait (bar1), gemm1, gemm2 + return pushes, return wait (bar2), combine
  static constexpr int kEv = 9;
  bool profiling = false;
  std::vector<std::array<cudaEvent_t, kEv>> ev_pool;
  size_t ev_used = 0;
  void mark(int i, cudaStream_t s) {
    if (!profiling) return;
    if (i == 0 && ev_used == ev_pool.size()) {
      std::array<cudaEvent_t, kEv> set;
      for (cudaEvent_t& e : set) EMOE_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(set);
    }
    EMOE_CUDA(cudaEventRecord(ev_pool[ev_used][i], s));
    if (i == kEv - 1) ++ev_used;
  }

  void forward(const void* x, const float* logits_in, void* y, int64_t T, cudaStream_t s) {
    EpRegion& g = *R;
    EMOE_REQUIRE(g.opened, "ep_forward: peers not opened (emoe_ep_open_peers)");
    const int W = g.W;
    ++g.epoch;
    mark(0, s);
    layer_route_scan(layer, x, logits_in, T, s);
    if (T == 0) {  // nothing routed: publish zero counts so peers' layouts stay consistent
      EMOE_CUDA(cudaMemsetAsync(const_cast<int64_t*>(v.seg_offsets), 0, sizeof(int64_t) * (v.E + 1), s));
      EMOE_CUDA(cudaMemsetAsync(const_cast<int32_t*>(v.counts), 0, sizeof(int32_t) * v.E, s));
    }
    mark(1, s);
    const int n_owned = (int)owned.size();
    LayoutArgs a{v.counts, v.seg_offsets, cum_dev, owned_dev, n_owned, v.seg_pad, g.recv_cap,
                 piece_end, piece_shift, recv_segs, out_shift, stats};
    const PeerSym ps = g.peer_sym();
    ep_bar0_kernel<<<1, 256, 0, s>>>(ps, W, g.rank, v.E, g.epoch, g.timeout_ns, g.status, a);
    EMOE_CUDA(cudaGetLastError());
    mark(2, s);
    PeerRows pr{};
    for (int q = 0; q < W; ++q) pr.base[q] = g.peer[q] + g.off_x;
    pr.piece_end = piece_end;
    pr.piece_shift = piece_shift;
    pr.W = W;
    pr.cap = g.recv_cap;
    launch_permute_remote(x, v.elem, T, v.d, v.E, v.k, v.served_idx, v.seg_offsets, v.block_base, pr, v.pos, s);
    mark(3, s);
    ep_bar_kernel<<<1, 32, 0, s>>>(ps, W, g.rank, 1, g.epoch, g.timeout_ns, g.status);
    EMOE_CUDA(cudaGetLastError());
    mark(4, s);
    cudaEvent_t mid = profiling ? ev_pool[ev_used][5] : nullptr;
    if (n_owned > 0) {
      PeerOut po{};
      for (int q = 0; q < W; ++q) po.base[q] = g.peer[q] + g.off_y;
      po.seg_rank = seg_rank;
      po.seg_shift = out_shift;
      layer_ffn_rows(layer, g.sym + g.off_x, g.recv_cap, recv_segs, seg_expert, W * n_owned, g.h, g.sym + g.off_y,
                     s, &po, mid);
    } else if (mid) {
      EMOE_CUDA(cudaEventRecord(mid, s));
    }
    mark(6, s);
    ep_bar_kernel<<<1, 32, 0, s>>>(ps, W, g.rank, 2, g.epoch, g.timeout_ns, g.status);
    EMOE_CUDA(cudaGetLastError());
    count_launch(3);
    mark(7, s);
    launch_combine(g.sym + g.off_y, DT_BF16, T, v.d, v.k, v.pos, v.served_w, y, s);
    mark(8, s);
  }

  void destroy() {
    cudaDeviceSynchronize();
    for (void* p : {(void*)cum_dev, (void*)owned_dev, (void*)piece_end, (void*)piece_shift, (void*)recv_segs,
                    (void*)seg_expert, (void*)seg_rank, (void*)out_shift, (void*)stats})
      if (p) cudaFree(p);
    for (auto& set : ev_pool)
      for (cudaEvent_t e : set) cudaEventDestroy(e);
    R.reset();
  }
};

extern "C" {

int emoe_ep_create(emoe_layer* layer, int world, int rank, const int64_t* cum_shares, int64_t recv_rows_cap,
                   emoe_ep* share_with, emoe_ep** out) {
  return guard([&] {
    EMOE_REQUIRE(layer && cum_shares && out, "ep_create: null argument");
    EMOE_REQUIRE(world >= 1 && world <= kMaxPeers, "ep_create: world must be in [1, 8]");
    EMOE_REQUIRE(rank >= 0 && rank < world, "ep_create: rank out of range");
    const LayerView v = layer_view(layer);
    EMOE_REQUIRE(v.dtype == DT_BF16, "ep_create: expert parallelism runs the bf16 path");
    const int E = v.E;
    EMOE_REQUIRE(E <= kMaxE, "ep_create: at most 128 experts");
    const int64_t one = 1ll << kShareBits;
    std::vector<int64_t> cum(cum_shares, cum_shares + (size_t)world * E);
    std::vector<int32_t> owned;
    for (int e = 0; e < E; ++e) {
      const int64_t* c = cum.data() + (size_t)e * world;
      if (c[0] < 0) {  // not resident
        for (int q = 0; q < world; ++q) EMOE_REQUIRE(c[q] < 0, "ep_create: cum_shares row mixes -1 and shares");
        continue;
      }
      for (int q = 0; q < world; ++q) {
        EMOE_REQUIRE(c[q] >= 0 && c[q] <= one, "ep_create: cum_shares must lie in [0, 2^24]");
        EMOE_REQUIRE(q == 0 || c[q] >= c[q - 1], "ep_create: cum_shares must be non-decreasing over ranks");
      }
      EMOE_REQUIRE(c[world - 1] == one, "ep_create: cum_shares must end at 2^24");
      if (c[rank] > (rank > 0 ? c[rank - 1] : 0)) owned.push_back(e);
    }
    EMOE_REQUIRE((int64_t)world * (int64_t)owned.size() <= 256, "ep_create: more than 256 receive segments");
    auto* ep = new emoe_ep();
    try {
      ep->layer = layer;
      ep->v = v;
      ep->cum = cum;
      ep->owned = owned;
      if (share_with) {
        const EpRegion& g = *share_with->R;
        EMOE_REQUIRE(g.W == world && g.rank == rank, "ep_create: share_with has another world or rank");
        EMOE_REQUIRE(g.E == E && g.d == v.d && g.f == v.f && g.elem == v.elem && v.rows_cap <= g.rows_cap,
                     "ep_create: share_with's region does not fit this layer's shape");
        EMOE_REQUIRE(recv_rows_cap <= 0 || recv_rows_cap <= g.recv_cap,
                     "ep_create: recv_rows_cap exceeds the shared region's");
        ep->R = share_with->R;
      } else {
        auto g = std::make_shared<EpRegion>();
        g->W = world;
        g->rank = rank;
        g->E = E;
        g->d = v.d;
        g->f = v.f;
        g->elem = v.elem;
        g->rows_cap = v.rows_cap;
        // default: the worst case (every source sends this rank all of its rows)
        g->recv_cap = recv_rows_cap > 0 ? ceil_div(recv_rows_cap, v.seg_pad) * v.seg_pad
                                        : (int64_t)world * v.rows_cap;
        const char* to = getenv("EMOE_EP_TIMEOUT_S");
        g->timeout_ns = (uint64_t)((to ? atof(to) : 60.0) * 1e9);
        const size_t row = (size_t)v.d * v.elem;
        g->off_cnt = align256(sizeof(uint64_t) * kPhases * kMaxPeers);
        g->off_x = align256(g->off_cnt + sizeof(int32_t) * kMaxPeers * E);
        g->off_y = align256(g->off_x + (size_t)g->recv_cap * row);
        g->sym_bytes = align256(g->off_y + (size_t)v.rows_cap * row);
        g->sym = dmalloc<uint8_t>(g->sym_bytes);
        EMOE_CUDA(cudaMemset(g->sym, 0, g->sym_bytes));
        g->status = dmalloc<int>(1);
        EMOE_CUDA(cudaMemset(g->status, 0, sizeof(int)));
        g->h = dmalloc<uint8_t>((size_t)g->recv_cap * v.f * v.elem);
        EMOE_CUDA(cudaMemset(g->h, 0, (size_t)g->recv_cap * v.f * v.elem));
        g->peer[rank] = g->sym;
        if (world == 1) g->opened = true;
        ep->R = g;
      }
      ep->cum_dev = dmalloc<int64_t>(cum.size());
      EMOE_CUDA(cudaMemcpy(ep->cum_dev, cum.data(), cum.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      ep->owned_dev = dmalloc<int32_t>(std::max<size_t>(1, owned.size()));
      if (!owned.empty())
        EMOE_CUDA(cudaMemcpy(ep->owned_dev, owned.data(), owned.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      ep->piece_end = dmalloc<int64_t>((size_t)E * world);
      ep->piece_shift = dmalloc<int64_t>((size_t)E * world);
      const int n_seg = world * (int)owned.size();
      ep->recv_segs = dmalloc<int64_t>(n_seg + 1);
      ep->seg_expert = dmalloc<int32_t>(std::max(1, n_seg));
      ep->seg_rank = dmalloc<int32_t>(std::max(1, n_seg));
      ep->out_shift = dmalloc<int64_t>(std::max(1, n_seg));
      ep->stats = dmalloc<int64_t>(kStats);
      EMOE_CUDA(cudaMemset(ep->stats, 0, sizeof(int64_t) * kStats));
      std::vector<int32_t> se, sr;
      for (int s = 0; s < world; ++s) {
        se.insert(se.end(), owned.begin(), owned.end());
        sr.insert(sr.end(), owned.size(), s);
      }
      if (n_seg) {
        EMOE_CUDA(cudaMemcpy(ep->seg_expert, se.data(), se.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        EMOE_CUDA(cudaMemcpy(ep->seg_rank, sr.data(), sr.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      }
      EMOE_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      ep->destroy();
      delete ep;
      throw;
    }
    *out = ep;
  });
}

int emoe_ep_ipc_handle(emoe_ep* ep, void* handle_out) {
  return guard([&] {
    EMOE_REQUIRE(ep && handle_out, "ep_ipc_handle: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == EMOE_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t hdl;
    EMOE_CUDA(cudaIpcGetMemHandle(&hdl, ep->R->sym));
    std::memcpy(handle_out, &hdl, sizeof(hdl));
  });
}

int emoe_ep_open_peers(emoe_ep* ep, const void* handles) {
  return guard([&] {
    EMOE_REQUIRE(ep && handles, "ep_open_peers: null argument");
    EpRegion& g = *ep->R;
    EMOE_REQUIRE(!g.opened || g.W == 1, "ep_open_peers: already opened (a shared region opens once)");
    const uint8_t* h = static_cast<const uint8_t*>(handles);
    for (int q = 0; q < g.W; ++q) {
      if (q == g.rank) continue;
      cudaIpcMemHandle_t hdl;
      std::memcpy(&hdl, h + (size_t)q * EMOE_IPC_HANDLE_BYTES, sizeof(hdl));
      void* p = nullptr;
      EMOE_CUDA(cudaIpcOpenMemHandle(&p, hdl, cudaIpcMemLazyEnablePeerAccess));
      g.peer[q] = static_cast<uint8_t*>(p);
    }
    g.opened = true;
  });
}

int emoe_ep_forward(emoe_ep* ep, const void* x, const float* logits_in, void* y, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(ep && x && y, "ep_forward: null argument");
    EMOE_REQUIRE(T >= 0 && T <= ep->v.max_tokens, "ep_forward: T exceeds the layer's max_tokens");
    ep->forward(x, logits_in, y, T, static_cast<cudaStream_t>(stream));
  });
}

int emoe_ep_status(emoe_ep* ep, void* stream, int* status, int64_t* recv_rows) {
  return guard([&] {
    EMOE_REQUIRE(ep, "ep_status: null handle");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int st = 0;
    int64_t rr = 0;
    EMOE_CUDA(cudaMemcpyAsync(&st, ep->R->status, sizeof(int), cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaMemcpyAsync(&rr, ep->stats, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
    if (status) *status = st;
    if (recv_rows) *recv_rows = rr;
  });
}

int emoe_ep_stats(emoe_ep* ep, void* stream, int64_t* out) {
  return guard([&] {
    EMOE_REQUIRE(ep && out, "ep_stats: null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EMOE_CUDA(cudaMemcpyAsync(out, ep->stats, sizeof(int64_t) * kStats, cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
  });
}

int emoe_ep_layout(emoe_ep* ep, void* stream, int64_t* piece_end, int64_t* piece_shift, int64_t* recv_segs,
                   int64_t* out_shift) {
  return guard([&] {
    EMOE_REQUIRE(ep, "ep_layout: null handle");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t ew = (size_t)ep->v.E * ep->R->W, ns = (size_t)ep->R->W * ep->owned.size();
    if (piece_end) EMOE_CUDA(cudaMemcpyAsync(piece_end, ep->piece_end, ew * 8, cudaMemcpyDeviceToHost, s));
    if (piece_shift) EMOE_CUDA(cudaMemcpyAsync(piece_shift, ep->piece_shift, ew * 8, cudaMemcpyDeviceToHost, s));
    if (recv_segs) EMOE_CUDA(cudaMemcpyAsync(recv_segs, ep->recv_segs, (ns + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (out_shift && ns) EMOE_CUDA(cudaMemcpyAsync(out_shift, ep->out_shift, ns * 8, cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
  });
}

int emoe_ep_set_profiling(emoe_ep* ep, int enable) {
  return guard([&] {
    EMOE_REQUIRE(ep, "ep_set_profiling: null handle");
    ep->profiling = enable != 0;
    ep->ev_used = 0;
  });
}

int emoe_ep_stage_times(emoe_ep* ep, float* ms) {
  return guard([&] {
    EMOE_REQUIRE(ep && ms, "ep_stage_times: null argument");
    EMOE_REQUIRE(ep->ev_used > 0, "ep_stage_times: no profiled forward since the last call");
    constexpr int n = emoe_ep::kEv - 1;
    for (int i = 0; i < n; ++i) ms[i] = 0.0f;
    for (size_t u = 0; u < ep->ev_used; ++u) {
      auto& set = ep->ev_pool[u];
      EMOE_CUDA(cudaEventSynchronize(set[n]));
      for (int i = 0; i < n; ++i) {
        float t = 0;
        EMOE_CUDA(cudaEventElapsedTime(&t, set[i], set[i + 1]));
        ms[i] += t / (float)ep->ev_used;
      }
    }
    ep->ev_used = 0;
  });
}

int emoe_ep_destroy(emoe_ep* ep) {
  return guard([&] {
    if (!ep) return;
    ep->destroy();
    delete ep;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// NCCL chunk transport: the device halves (the collectives are the caller's)
// ---------------------------------------------------------------------------
struct emoe_epx {
  emoe_layer* layer = nullptr;
  LayerView v{};
  int W = 1, rank = 0;
  int64_t cap = 0;
  std::vector<int32_t> owned;
  int64_t* cum_dev = nullptr;
  int32_t* owned_dev = nullptr;
  int64_t* piece_end = nullptr;
  int64_t* piece_shift = nullptr;
  int64_t* recv_segs = nullptr;
  int64_t* a_shift = nullptr;
  int32_t* seg_expert = nullptr;
  int64_t* stats = nullptr;
  int* status = nullptr;
  void* h = nullptr;  // [W * cap][f] GEMM1 output, compact
  void destroy() {
    cudaDeviceSynchronize();
    for (void* p : {(void*)cum_dev, (void*)owned_dev, (void*)piece_end, (void*)piece_shift, (void*)recv_segs,
                    (void*)a_shift, (void*)seg_expert, (void*)stats, (void*)status, h})
      if (p) cudaFree(p);
  }
};

extern "C" {

int emoe_epx_create(emoe_layer* layer, int world, int rank, const int64_t* cum_shares, int64_t cap_rows,
                    emoe_epx** out) {
  return guard([&] {
    EMOE_REQUIRE(layer && cum_shares && out, "epx_create: null argument");
    EMOE_REQUIRE(world >= 1 && world <= kMaxPeers && rank >= 0 && rank < world, "epx_create: bad world / rank");
    const LayerView v = layer_view(layer);
    EMOE_REQUIRE(v.dtype == DT_BF16 && v.E <= kMaxE, "epx_create: bf16, E <= 128");
    const int E = v.E;
    std::vector<int32_t> owned;
    for (int e = 0; e < E; ++e) {
      const int64_t* c = cum_shares + (size_t)e * world;
      if (c[0] >= 0 && c[rank] > (rank > 0 ? c[rank - 1] : 0)) owned.push_back(e);
    }
    EMOE_REQUIRE((int64_t)world * (int64_t)owned.size() <= 256, "epx_create: more than 256 receive segments");
    auto* x = new emoe_epx();
    try {
      x->layer = layer;
      x->v = v;
      x->W = world;
      x->rank = rank;
      x->owned = owned;
      x->cap = ceil_div(cap_rows > 0 ? cap_rows : v.rows_cap, v.seg_pad) * v.seg_pad;
      const size_t ew = (size_t)E * world, ns = (size_t)world * owned.size();
      x->cum_dev = dmalloc<int64_t>(ew);
      EMOE_CUDA(cudaMemcpy(x->cum_dev, cum_shares, ew * 8, cudaMemcpyHostToDevice));
      x->owned_dev = dmalloc<int32_t>(std::max<size_t>(1, owned.size()));
      if (!owned.empty())
        EMOE_CUDA(cudaMemcpy(x->owned_dev, owned.data(), owned.size() * 4, cudaMemcpyHostToDevice));
      x->piece_end = dmalloc<int64_t>(ew);
      x->piece_shift = dmalloc<int64_t>(ew);
      x->recv_segs = dmalloc<int64_t>(ns + 1);
      x->a_shift = dmalloc<int64_t>(std::max<size_t>(1, ns));
      x->seg_expert = dmalloc<int32_t>(std::max<size_t>(1, ns));
      std::vector<int32_t> se;
      for (int s = 0; s < world; ++s) se.insert(se.end(), owned.begin(), owned.end());
      if (ns) EMOE_CUDA(cudaMemcpy(x->seg_expert, se.data(), ns * 4, cudaMemcpyHostToDevice));
      x->stats = dmalloc<int64_t>(kStats);
      EMOE_CUDA(cudaMemset(x->stats, 0, sizeof(int64_t) * kStats));
      x->status = dmalloc<int>(1);
      EMOE_CUDA(cudaMemset(x->status, 0, sizeof(int)));
      x->h = dmalloc<uint8_t>((size_t)world * x->cap * v.f * v.elem);
      EMOE_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      x->destroy();
      delete x;
      throw;
    }
    *out = x;
  });
}

int emoe_epx_cap_rows(const emoe_epx* x, int64_t* cap) {
  return guard([&] {
    EMOE_REQUIRE(x && cap, "epx_cap_rows: null argument");
    *cap = x->cap;
  });
}

int emoe_epx_route(emoe_epx* x, const void* xin, const float* logits_in, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(x && xin, "epx_route: null argument");
    EMOE_REQUIRE(T >= 0 && T <= x->v.max_tokens, "epx_route: T exceeds the layer's max_tokens");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    layer_route_scan(x->layer, xin, logits_in, T, s);
    if (T == 0) EMOE_CUDA(cudaMemsetAsync(const_cast<int32_t*>(x->v.counts), 0, sizeof(int32_t) * x->v.E, s));
  });
}

int emoe_epx_dispatch(emoe_epx* x, const int32_t* table_dev, const void* xin, int64_t T, void* send_chunks,
                      void* stream) {
  return guard([&] {
    EMOE_REQUIRE(x && table_dev && send_chunks, "epx_dispatch: null argument");
    EMOE_REQUIRE(T == 0 || xin, "epx_dispatch: null x");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ChunkArgs a{table_dev,   x->v.seg_offsets, x->cum_dev,   x->owned_dev, (int)x->owned.size(), x->v.seg_pad,
                x->cap,      x->piece_end,     x->piece_shift, x->recv_segs, x->a_shift,           x->stats,
                x->status};
    epx_layout_kernel<<<1, 256, 0, s>>>(x->W, x->rank, x->v.E, a);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    if (T == 0) return;
    PeerRows pr{};
    for (int q = 0; q < x->W; ++q) pr.base[q] = static_cast<uint8_t*>(send_chunks);
    pr.piece_end = x->piece_end;
    pr.piece_shift = x->piece_shift;
    pr.W = x->W;
    pr.cap = (int64_t)x->W * x->cap;
    pr.pos_remote = 1;
    launch_permute_remote(xin, x->v.elem, T, x->v.d, x->v.E, x->v.k, x->v.served_idx, x->v.seg_offsets,
                          x->v.block_base, pr, x->v.pos, s);
  });
}

int emoe_epx_ffn(emoe_epx* x, const void* recv_chunks, void* return_chunks, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(x && recv_chunks && return_chunks, "epx_ffn: null argument");
    const int n_seg = x->W * (int)x->owned.size();
    if (n_seg == 0) return;
    const int64_t rows = (int64_t)x->W * x->cap;
    layer_ffn_chunks(x->layer, recv_chunks, rows, x->recv_segs, x->seg_expert, n_seg, x->a_shift, x->h, rows,
                     return_chunks, rows, static_cast<cudaStream_t>(stream));
  });
}

int emoe_epx_combine(emoe_epx* x, const void* returned_chunks, void* y, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(x && returned_chunks && y, "epx_combine: null argument");
    launch_combine(returned_chunks, DT_BF16, T, x->v.d, x->v.k, x->v.pos, x->v.served_w, y,
                   static_cast<cudaStream_t>(stream));
  });
}

int emoe_epx_status(emoe_epx* x, void* stream, int* status, int64_t* rows) {
  return guard([&] {
    EMOE_REQUIRE(x, "epx_status: null handle");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int st = 0;
    int64_t rr = 0;
    EMOE_CUDA(cudaMemcpyAsync(&st, x->status, sizeof(int), cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaMemcpyAsync(&rr, x->stats, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
    if (status) *status = st;
    if (rows) *rows = rr;
  });
}

int emoe_epx_destroy(emoe_epx* x) {
  return guard([&] {
    if (!x) return;
    x->destroy();
    delete x;
  });
}

}  // extern "C"
