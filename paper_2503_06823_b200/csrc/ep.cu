// Expert parallelism over peer memory: the token dispatch is
// fused into the permute kernel (NVLink stores straight into the owning
// rank's receive buffer) and the return into GEMM2's epilogue (each expert
// output row stored straight into its source rank's own permuted layout), so
// the combine runs locally.  No all-to-all, no host synchronisation.
//
// Every rank allocates one symmetric region (same size everywhere) and maps
// every peer's region through CUDA IPC:
//   flags    u64 [3 phases][kMaxPeers]   epoch written by each source rank
//   cnt      i32 [kMaxPeers][E]          padded segment sizes of every source
//   recv_x   bf16 [recv_cap][d]          rows dispatched to this rank
//   y_local  bf16 [rows_cap][d]          expert outputs of this rank's own rows,
//                                        in its local permuted layout
// One forward, all on the caller's stream:
//   K1 + K3a  route and scan locally (layer_route_scan)
//   bar0      publish this rank's padded counts to every peer, signal, wait
//             for all ranks, then derive from the replicated count table the
//             receive segments, per local expert the row shift into its
//             owner's receive buffer, and per receive segment the row shift
//             back into its source's layout
//   K3b       permute_kernel<REMOTE>: rows -> owner's recv_x (peer stores)
//   bar1      signal + wait: every source finished writing to this rank
//   K4        grouped GEMMs over the (source, expert) segments of recv_x;
//             GEMM2's epilogue pushes each row to its source's y_local
//   bar2      signal + wait: every rank's pushes have landed
//   K5        combine_bf16_kernel over the local y_local (slot order)
// Receive layout on rank q: segments ordered by (source rank, expert), the
// same order the NCCL path (ep.py) uses; every row meets the same GEMM
// arithmetic and the combine order is fixed at the source, so the output is
// bit-identical to EP=1.
// Buffer reuse across forwards needs no extra barrier: a source writes cnt /
// recv_x of forward n+1 only after its own bar2 of forward n, which every
// rank reaches only after its layout reads of forward n; GEMM2 of forward
// n+1 pushes into a source's y_local only after bar1 of n+1, i.e. after every
// rank finished its combine of forward n.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "capi_util.h"
#include "kernels.h"

namespace emoe {
namespace {

constexpr int kPhases = 3;

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
  const int64_t* seg_offsets;  // [E+1] this rank's padded local segments
  const int32_t* dest;         // [W][E]
  const int32_t* owned;        // [n_owned] experts this rank computes (ascending)
  int n_owned;
  int64_t recv_cap;
  int64_t* recv_segs;  // [W * n_owned + 1]
  int64_t* row_shift;  // [E]
  int64_t* out_shift;  // [W * n_owned] receive row -> row in the source's layout
  int64_t* recv_rows;  // [1]
};

// bar0: publish counts, barrier, then the receive segments and the send shifts
__global__ void __launch_bounds__(256) ep_bar0_kernel(PeerSym sym, int W, int rank, int E, uint64_t epoch,
                                                      uint64_t timeout_ns, int* status, LayoutArgs a) {
  __shared__ int64_t tot[kMaxPeers][kMaxPeers];  // [source][receiver] rows
  __shared__ int overflow;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int32_t v = (int32_t)(a.seg_offsets[e + 1] - a.seg_offsets[e]);
    for (int q = 0; q < W; ++q) sym.cnt[q][rank * E + e] = v;
  }
  barrier(sym, W, rank, 0, epoch, timeout_ns, status);
  const int32_t* cnt = sym.cnt[rank];  // every source's counts, now local
  if (threadIdx.x < W * W) {
    const int s = threadIdx.x / W, q = threadIdx.x % W;
    int64_t t = 0;
    for (int e = 0; e < E; ++e)
      if (a.dest[s * E + e] == q) t += cnt[s * E + e];
    tot[s][q] = t;
  }
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  if (threadIdx.x < W) {
    int64_t t = 0;
    for (int s = 0; s < W; ++s) t += tot[s][threadIdx.x];
    if (t > a.recv_cap) overflow = 1;
  }
  __syncthreads();
  if (overflow) {
    if (threadIdx.x == 0) atomicExch(status, 2);
    for (int e = threadIdx.x; e < E; e += blockDim.x) a.row_shift[e] = a.recv_cap;  // every row out of range
    for (int i = threadIdx.x; i <= W * a.n_owned; i += blockDim.x) a.recv_segs[i] = 0;
    if (threadIdx.x == 0) *a.recv_rows = 0;
    return;
  }
  // send shifts: segment e goes to q = dest[rank][e] after every earlier
  // source's rows for q and this rank's rows of earlier experts for q
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int q = a.dest[rank * E + e];
    if (q < 0) {
      a.row_shift[e] = 0;
      continue;
    }
    int64_t base = 0;
    for (int s = 0; s < rank; ++s) base += tot[s][q];
    for (int e2 = 0; e2 < e; ++e2)
      if (a.dest[rank * E + e2] == q) base += cnt[rank * E + e2];
    a.row_shift[e] = base - a.seg_offsets[e];
  }
  // receive segments: (source, owned expert) in order; the return shift maps
  // receive row r of segment (s, e) to row r + shift of source s's layout
  // (its padded segment e starts at the exclusive prefix of its counts)
  if (threadIdx.x == 0) {
    int64_t off = 0;
    int i = 0;
    for (int s = 0; s < W; ++s)
      for (int j = 0; j < a.n_owned; ++j) {
        const int e = a.owned[j];
        int64_t src_off = 0;
        for (int e2 = 0; e2 < e; ++e2) src_off += cnt[s * E + e2];
        a.recv_segs[i] = off;
        a.out_shift[i] = src_off - off;
        ++i;
        if (a.dest[s * E + e] == rank) off += cnt[s * E + e];
      }
    a.recv_segs[i] = off;
    *a.recv_rows = off;
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

}  // namespace
}  // namespace emoe

using namespace emoe;

struct emoe_ep {
  emoe_layer* layer = nullptr;
  LayerView v{};
  int W = 1, rank = 0;
  int64_t recv_cap = 0;
  std::vector<int32_t> dest;  // [W][E]
  std::vector<int32_t> owned;
  uint64_t epoch = 0;
  uint64_t timeout_ns = 0;

  uint8_t* sym = nullptr;  // own symmetric region
  size_t sym_bytes = 0, off_cnt = 0, off_x = 0, off_y = 0;  // off_y: y_local
  uint8_t* peer[kMaxPeers] = {};  // symmetric regions of every rank (own = sym)
  bool opened = false;

  int32_t* dest_dev = nullptr;
  int32_t* owned_dev = nullptr;
  int64_t* row_shift = nullptr;
  int64_t* recv_segs = nullptr;
  int32_t* seg_expert = nullptr;  // [W * n_owned]
  int32_t* seg_rank = nullptr;    // [W * n_owned] source rank of each receive segment
  int64_t* out_shift = nullptr;   // [W * n_owned]
  int64_t* recv_rows = nullptr;
  int* status = nullptr;
  void* h = nullptr;

  PeerSym peer_sym() const {
    PeerSym p{};
    for (int q = 0; q < W; ++q) {
      p.flags[q] = reinterpret_cast<uint64_t*>(peer[q]);
      p.cnt[q] = reinterpret_cast<int32_t*>(peer[q] + off_cnt);
    }
    return p;
  }
  PeerRows rows(size_t off) const {
    PeerRows r{};
    for (int q = 0; q < W; ++q) r.base[q] = peer[q] + off;
    r.dest = dest_dev + (size_t)rank * v.E;
    r.row_shift = row_shift;
    r.cap = recv_cap;
    return r;
  }

  void forward(const void* x, const float* logits_in, void* y, int64_t T, cudaStream_t s) {
    EMOE_REQUIRE(opened, "ep_forward: peers not opened (emoe_ep_open_peers)");
    ++epoch;
    layer_route_scan(layer, x, logits_in, T, s);
    if (T == 0) {  // nothing routed: publish zero counts so peers' layouts stay consistent
      EMOE_CUDA(cudaMemsetAsync(const_cast<int64_t*>(v.seg_offsets), 0, sizeof(int64_t) * (v.E + 1), s));
    }
    const int n_owned = (int)owned.size();
    LayoutArgs a{v.seg_offsets, dest_dev, owned_dev, n_owned, recv_cap, recv_segs, row_shift, out_shift, recv_rows};
    const PeerSym ps = peer_sym();
    ep_bar0_kernel<<<1, 256, 0, s>>>(ps, W, rank, v.E, epoch, timeout_ns, status, a);
    EMOE_CUDA(cudaGetLastError());
    launch_permute_remote(x, v.elem, T, v.d, v.E, v.k, v.served_idx, v.seg_offsets, v.block_base, rows(off_x),
                          v.pos, s);
    ep_bar_kernel<<<1, 32, 0, s>>>(ps, W, rank, 1, epoch, timeout_ns, status);
    EMOE_CUDA(cudaGetLastError());
    if (n_owned > 0) {
      PeerOut po{};
      for (int q = 0; q < W; ++q) po.base[q] = peer[q] + off_y;
      po.seg_rank = seg_rank;
      po.seg_shift = out_shift;
      layer_ffn_rows(layer, sym + off_x, recv_cap, recv_segs, seg_expert, W * n_owned, h, sym + off_y, s, &po);
    }
    ep_bar_kernel<<<1, 32, 0, s>>>(ps, W, rank, 2, epoch, timeout_ns, status);
    EMOE_CUDA(cudaGetLastError());
    count_launch(3);
    launch_combine(sym + off_y, DT_BF16, T, v.d, v.k, v.pos, v.served_w, y, s);
  }

  void destroy() {
    for (int q = 0; q < W; ++q)
      if (peer[q] && peer[q] != sym) cudaIpcCloseMemHandle(peer[q]);
    for (void* p : {(void*)sym, (void*)dest_dev, (void*)owned_dev, (void*)row_shift, (void*)recv_segs,
                    (void*)seg_expert, (void*)seg_rank, (void*)out_shift, (void*)recv_rows, (void*)status, h})
      if (p) cudaFree(p);
  }
};

extern "C" {

int emoe_ep_create(emoe_layer* layer, int world, int rank, const int32_t* dest, int64_t recv_rows_cap,
                   emoe_ep** out) {
  return guard([&] {
    EMOE_REQUIRE(layer && dest && out, "ep_create: null argument");
    EMOE_REQUIRE(world >= 1 && world <= kMaxPeers, "ep_create: world must be in [1, 8]");
    EMOE_REQUIRE(rank >= 0 && rank < world, "ep_create: rank out of range");
    const LayerView v = layer_view(layer);
    EMOE_REQUIRE(v.dtype == DT_BF16, "ep_create: expert parallelism runs the bf16 path");
    const int E = v.E;
    std::vector<int32_t> dv(dest, dest + (size_t)world * E);
    std::vector<int32_t> owned;
    for (int e = 0; e < E; ++e) {
      bool mine = false;
      for (int s = 0; s < world; ++s) {
        EMOE_REQUIRE(dv[(size_t)s * E + e] >= -1 && dv[(size_t)s * E + e] < world, "ep_create: dest out of range");
        mine |= dv[(size_t)s * E + e] == rank;
      }
      if (mine) owned.push_back(e);
    }
    EMOE_REQUIRE((int64_t)world * (int64_t)owned.size() <= 256, "ep_create: more than 256 receive segments");
    auto* ep = new emoe_ep();
    try {
      ep->layer = layer;
      ep->v = v;
      ep->W = world;
      ep->rank = rank;
      ep->dest = dv;
      ep->owned = owned;
      // default: the worst case (every source sends this rank all of its rows)
      ep->recv_cap = recv_rows_cap > 0 ? ceil_div(recv_rows_cap, v.seg_pad) * v.seg_pad : (int64_t)world * v.rows_cap;
      const char* to = getenv("EMOE_EP_TIMEOUT_S");
      ep->timeout_ns = (uint64_t)((to ? atof(to) : 60.0) * 1e9);
      const size_t row = (size_t)v.d * v.elem;
      ep->off_cnt = align256(sizeof(uint64_t) * kPhases * kMaxPeers);
      ep->off_x = align256(ep->off_cnt + sizeof(int32_t) * kMaxPeers * E);
      ep->off_y = align256(ep->off_x + (size_t)ep->recv_cap * row);
      ep->sym_bytes = align256(ep->off_y + (size_t)v.rows_cap * row);
      ep->sym = dmalloc<uint8_t>(ep->sym_bytes);
      EMOE_CUDA(cudaMemset(ep->sym, 0, ep->sym_bytes));
      ep->dest_dev = dmalloc<int32_t>(dv.size());
      EMOE_CUDA(cudaMemcpy(ep->dest_dev, dv.data(), dv.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      ep->owned_dev = dmalloc<int32_t>(std::max<size_t>(1, owned.size()));
      if (!owned.empty())
        EMOE_CUDA(cudaMemcpy(ep->owned_dev, owned.data(), owned.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      ep->row_shift = dmalloc<int64_t>(E);
      const int n_seg = world * (int)owned.size();
      ep->recv_segs = dmalloc<int64_t>(n_seg + 1);
      ep->seg_expert = dmalloc<int32_t>(std::max(1, n_seg));
      ep->seg_rank = dmalloc<int32_t>(std::max(1, n_seg));
      ep->out_shift = dmalloc<int64_t>(std::max(1, n_seg));
      std::vector<int32_t> se, sr;
      for (int s = 0; s < world; ++s) {
        se.insert(se.end(), owned.begin(), owned.end());
        sr.insert(sr.end(), owned.size(), s);
      }
      if (n_seg) {
        EMOE_CUDA(cudaMemcpy(ep->seg_expert, se.data(), se.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        EMOE_CUDA(cudaMemcpy(ep->seg_rank, sr.data(), sr.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      }
      ep->recv_rows = dmalloc<int64_t>(1);
      ep->status = dmalloc<int>(1);
      EMOE_CUDA(cudaMemset(ep->status, 0, sizeof(int)));
      ep->h = dmalloc<uint8_t>((size_t)ep->recv_cap * v.f * v.elem);
      EMOE_CUDA(cudaMemset(ep->h, 0, (size_t)ep->recv_cap * v.f * v.elem));
      ep->peer[rank] = ep->sym;
      if (world == 1) ep->opened = true;
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
    EMOE_CUDA(cudaIpcGetMemHandle(&hdl, ep->sym));
    std::memcpy(handle_out, &hdl, sizeof(hdl));
  });
}

int emoe_ep_open_peers(emoe_ep* ep, const void* handles) {
  return guard([&] {
    EMOE_REQUIRE(ep && handles, "ep_open_peers: null argument");
    EMOE_REQUIRE(!ep->opened || ep->W == 1, "ep_open_peers: already opened");
    const uint8_t* h = static_cast<const uint8_t*>(handles);
    for (int q = 0; q < ep->W; ++q) {
      if (q == ep->rank) continue;
      cudaIpcMemHandle_t hdl;
      std::memcpy(&hdl, h + (size_t)q * EMOE_IPC_HANDLE_BYTES, sizeof(hdl));
      void* p = nullptr;
      EMOE_CUDA(cudaIpcOpenMemHandle(&p, hdl, cudaIpcMemLazyEnablePeerAccess));
      ep->peer[q] = static_cast<uint8_t*>(p);
    }
    ep->opened = true;
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
    EMOE_CUDA(cudaMemcpyAsync(&st, ep->status, sizeof(int), cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaMemcpyAsync(&rr, ep->recv_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
    if (status) *status = st;
    if (recv_rows) *recv_rows = rr;
  });
}

int emoe_ep_destroy(emoe_ep* ep) {
  return guard([&] {
    if (!ep) return;
    cudaDeviceSynchronize();
    ep->destroy();
    delete ep;
  });
}

}  // extern "C"
