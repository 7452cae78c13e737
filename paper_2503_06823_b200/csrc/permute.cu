// K3 (scan + stable permute/gather) and K5 (gate-weighted combine).
//
// Permutation contract (builder-defined, restated in
// oracle_permute): expert e owns rows [off_e, off_e + pad_up(n_e)) of X_perm;
// the served pair (t, e) lands at off_e + #{t' < t : e in served(t')}, i.e. the
// segment is stable in token order.  No atomics decide positions, so the
// layout is bit-reproducible and identical to the CPU oracle.
//
// Data movement: x is read once (one warp per token, 16-byte vectors) and
// written to each of its <= k destinations; the combine reads each served row
// of Y once and writes y once, accumulating in fp32 in slot order.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace emoe {

namespace {

constexpr int RT = kRouteBlockTokens;

// K3a: one block per expert scans its per-block counts (block order) into
// per-block bases and the expert total; the last block to finish (a device
// counter, reset by that block for the next launch) turns the totals into the
// padded segment offsets and marks the padding rows of every segment as
// sourceless (row_token = -1; rows past seg_offsets[E] are never read).  One
// launch instead of scan + offsets kernels and a row_token memset.
constexpr int SCAN_T = 256;
__global__ void __launch_bounds__(SCAN_T) scan_kernel(const int32_t* __restrict__ block_counts, int nblocks, int E,
                                                   int pad, int64_t* __restrict__ block_base,
                                                   int32_t* __restrict__ counts, int64_t* __restrict__ seg_offsets,
                                                   int32_t* __restrict__ row_token, int32_t* __restrict__ done) {
  __shared__ int64_t warp_tot[SCAN_T / 32];
  __shared__ int64_t carry;
  __shared__ int is_last;
  __shared__ int32_t pad_beg[1024], pad_len[1024];
  const int e = blockIdx.x, lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  if (threadIdx.x == 0) carry = 0;
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  for (int b0 = 0; b0 < nblocks; b0 += SCAN_T) {
    const int b = b0 + threadIdx.x;
    const int64_t v = b < nblocks ? block_counts[(int64_t)b * E + e] : 0;
    int64_t incl = v;  // inclusive warp scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t n = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += n;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int64_t before = carry;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    if (b < nblocks) block_base[(int64_t)b * E + e] = before + incl - v;
    __syncthreads();
    if (threadIdx.x == SCAN_T - 1) carry = before + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[e] = (int32_t)carry;
    __threadfence();
    is_last = atomicAdd(done, 1) == E - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // the padded segment offsets: exclusive scan over E in chunks of SCAN_T
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int e0 = 0; e0 < E; e0 += SCAN_T) {
    const int i = e0 + threadIdx.x;
    const int64_t n = i < E ? (int64_t)__ldcg(counts + i) : 0;
    const int64_t v = (n + pad - 1) / pad * pad;
    int64_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += u;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int64_t before = carry;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    const int64_t off_i = before + incl - v;
    if (i < E) {
      seg_offsets[i] = off_i;
      if (i == E - 1) seg_offsets[E] = off_i + v;
      pad_beg[i] = (int32_t)(off_i + n);  // this segment's padding rows [off + n, off + pad(n))
      pad_len[i] = (int32_t)(v - n);
    }
    __syncthreads();
    if (threadIdx.x == SCAN_T - 1) carry = before + incl;
    __syncthreads();
  }
  // one thread per segment walks its padding rows (independent stores; an
  // expert-by-expert loop over the block measured 12 vs 7 us at E = 128)
  if (row_token)
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      for (int r = 0; r < pad_len[e]; ++r) row_token[pad_beg[e] + r] = -1;
  if (threadIdx.x == 0) *done = 0;
}

// K3b.  Block = 128 tokens (the route kernel's blocks).  Warps 0-3 rank their
// 32 tokens per expert with ballots (stable token order, no atomics); then
// all 8 warps gather rows, each lane keeping 8 16-byte loads in flight.
constexpr int PERMUTE_THREADS = 256;
constexpr int GATHER_UNROLL = 8;

// REMOTE (expert-parallel dispatch over peer memory): local row d of segment
// e is written to the receive buffer of the rank computing its piece
// (peers.base[q], mapped through CUDA IPC) at row d + piece_shift[e][q];
// pos[t][j] keeps d, the local row the pushed output returns to.  The per-block tail fence makes the NVLink
// stores visible system-wide before the host-ordered signal kernel runs.
// SPLIT (fp32 rows of a 3xTF32 layer): also write each row's tf32 hi / lo
// parts to x_hi / x_lo (a separate instantiation, so the other layers' permute
// carries none of it)
// Small batches (few token blocks): K3a folded into K3b.  Every block derives
// the segment offsets and its own per-expert bases from the block counts
// (nblocks x E values, read through L2), and block (0, 0) stores the counts,
// the padded offsets (read by the GEMMs) and the padding rows of row_token --
// one launch instead of two where the scan's latency is most of its cost.
struct SmallScan {
  const int32_t* block_counts = nullptr;  // null: offsets / bases come from scan_kernel
  int nblocks = 0;
  int pad = 0;
  int32_t* counts = nullptr;
  int64_t* seg_offsets = nullptr;
};
constexpr int SMALL_SCAN_BLOCKS = 32;  // token blocks (4,096 tokens) up to which the scan is folded in
constexpr int SMALL_SCAN_E = 128;

template <bool REMOTE, bool SPLIT = false>
__global__ void __launch_bounds__(PERMUTE_THREADS) permute_kernel(
    const uint8_t* __restrict__ x, int row_bytes, int64_t T, int E, int k, const int32_t* __restrict__ served_idx,
    const int64_t* __restrict__ seg_offsets, const int64_t* __restrict__ block_base, uint8_t* __restrict__ x_perm,
    int32_t* __restrict__ pos, int32_t* __restrict__ row_token, PeerRows peers, float* __restrict__ x_hi,
    float* __restrict__ x_lo, SmallScan ss) {
  extern __shared__ int32_t sh[];
  __shared__ int64_t s_off[SMALL_SCAN_E + 1], s_base[SMALL_SCAN_E];
  int32_t* warp_counts = sh;          // [4][E]
  int32_t* dst_s = sh + 4 * E;        // [RT][k]
  // REMOTE: destination row pointer per (token, slot), 8-B aligned after dst_s
  uint8_t** dptr_s = reinterpret_cast<uint8_t**>(sh + 4 * E + ((RT * k + 1) & ~1));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t0 = (int64_t)blockIdx.x * RT;
  pdl_wait();
  pdl_trigger();
  const bool small_scan = !REMOTE && ss.block_counts != nullptr;
  if (small_scan) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      int64_t tot = 0, base = 0;
      for (int b = 0; b < ss.nblocks; ++b) {
        if (b == (int)blockIdx.x) base = tot;
        tot += __ldcg(ss.block_counts + (int64_t)b * E + e);
      }
      s_base[e] = base;
      s_off[e] = tot;  // the total, until the scan below
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // padded exclusive scan over the experts (E <= 128)
      int64_t run = 0;
      for (int e = 0; e < E; ++e) {
        const int64_t n = s_off[e];
        s_off[e] = run;
        run += (n + ss.pad - 1) / ss.pad * ss.pad;
      }
      s_off[E] = run;
    }
    __syncthreads();
    if (blockIdx.x == 0 && blockIdx.y == 0) {
      for (int e = threadIdx.x; e <= E; e += blockDim.x) ss.seg_offsets[e] = s_off[e];
      for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int64_t tot = 0;
        for (int b = 0; b < ss.nblocks; ++b) tot += __ldcg(ss.block_counts + (int64_t)b * E + e);
        ss.counts[e] = (int32_t)tot;
        if (row_token)  // this segment's padding rows
          for (int64_t r = s_off[e] + tot; r < s_off[e + 1]; ++r) row_token[r] = -1;
      }
    }
  }
  int my[8];
  int rank[8];
  if (warp < 4) {
    const int64_t t = t0 + threadIdx.x;
    const bool valid = t < T;
    for (int j = 0; j < k; ++j) {
      my[j] = valid ? served_idx[t * k + j] : -1;
      rank[j] = 0;
    }
    const uint32_t lt = (1u << lane) - 1u;
    if (k == 1) {  // one served slot: lanes with the same expert form one match group
      for (int e = lane; e < E; e += 32) warp_counts[warp * E + e] = 0;
      __syncwarp();
      const uint32_t m = __match_any_sync(0xffffffffu, my[0]);
      if (my[0] >= 0) {
        rank[0] = __popc(m & lt);
        if (rank[0] == 0) warp_counts[warp * E + my[0]] = __popc(m);
      }
    } else {
      // per expert: lanes (tokens) that serve it; a token serves an expert at most once
      for (int e = 0; e < E; ++e) {
        bool has = false;
        for (int j = 0; j < k; ++j) has |= (my[j] == e);
        const uint32_t m = __ballot_sync(0xffffffffu, has);
        if (lane == 0) warp_counts[warp * E + e] = __popc(m);
        if (has)
          for (int j = 0; j < k; ++j)
            if (my[j] == e) rank[j] = __popc(m & lt);
      }
    }
  }
  __syncthreads();
  if (warp < 4) {
    const int64_t t = t0 + threadIdx.x;
    for (int j = 0; j < k; ++j) {
      const int e = my[j];
      int32_t d = -1;
      if (e >= 0) {
        int64_t base = small_scan ? s_off[e] + s_base[e] : seg_offsets[e] + block_base[(int64_t)blockIdx.x * E + e];
        for (int w = 0; w < warp; ++w) base += warp_counts[w * E + e];
        d = (int32_t)(base + rank[j]);
      }
      dst_s[threadIdx.x * k + j] = d;
      if (blockIdx.y != 0) continue;  // column-split blocks: block row 0 writes the positions
      if (REMOTE) {
        uint8_t* ptr = nullptr;
        int64_t dst_row = -1;
        if (e >= 0) {
          for (int q = 0; q < peers.W; ++q)  // the piece of segment e holding local row d
            if (d < peers.piece_end[e * peers.W + q]) {
              const int64_t r = d + peers.piece_shift[e * peers.W + q];
              if (r >= 0 && r < peers.cap) {
                ptr = peers.base[q] + r * row_bytes;
                dst_row = r;
              }
              break;
            }  // no piece: the receivers overflowed (status 2), the row is dropped
        }
        dptr_s[threadIdx.x * k + j] = ptr;
        // outputs return to this local row (peer memory), or to the same row
        // of the return chunks (NCCL chunk transport)
        if (t < T) pos[t * k + j] = ptr ? (peers.pos_remote ? (int32_t)dst_row : d) : -1;
      } else if (t < T) {
        if (pos) pos[t * k + j] = d;
        if (row_token && d >= 0) row_token[d] = (int32_t)t;
      }
    }
  }
  __syncthreads();
  // gather: the block's rows x (row_bytes / 16) chunks as one flat index space
  // (consecutive threads -> consecutive 16-B chunks of the contiguous x rows),
  // GATHER_UNROLL independent loads in flight per thread whatever d is
  // (small T: gridDim.y blocks share a token block, each gathering one column slice)
  const int nvec_all = row_bytes / 16;
  const int v0 = (int)((int64_t)nvec_all * blockIdx.y / gridDim.y);
  const int nvec = (int)((int64_t)nvec_all * (blockIdx.y + 1) / gridDim.y) - v0;
  const int rows = (int)min((int64_t)RT, T - t0);
  const int total = rows * nvec;
  const uint4* src = reinterpret_cast<const uint4*>(x + t0 * row_bytes);
  for (int base = threadIdx.x; base < total; base += PERMUTE_THREADS * GATHER_UNROLL) {
    uint4 val[GATHER_UNROLL];
    int tok[GATHER_UNROLL];
#pragma unroll
    for (int u = 0; u < GATHER_UNROLL; ++u) {
      const int i = base + u * PERMUTE_THREADS;
      tok[u] = i < total ? i / nvec : -1;
      if (tok[u] >= 0 && dst_s[tok[u] * k] < 0) tok[u] = -1;  // token served nowhere
      if (tok[u] >= 0) val[u] = __ldg(src + (int64_t)tok[u] * nvec_all + v0 + (i - tok[u] * nvec));
    }
#pragma unroll
    for (int u = 0; u < GATHER_UNROLL; ++u) {
      if (tok[u] < 0) continue;
      const int v = v0 + base + u * PERMUTE_THREADS - tok[u] * nvec;
      for (int j = 0; j < k; ++j) {
        const int32_t d = dst_s[tok[u] * k + j];
        if (d < 0) break;  // served slots are compacted to the front
        uint8_t* row = REMOTE ? dptr_s[tok[u] * k + j] : x_perm + (int64_t)d * row_bytes;
        if (REMOTE && !row) continue;
        reinterpret_cast<uint4*>(row)[v] = val[u];
        if (SPLIT) {  // fp32 rows of a 3xTF32 layer: the hi / lo split as well
          const float4 f = *reinterpret_cast<const float4*>(&val[u]);
          const float4 h = make_float4(round_tf32(f.x), round_tf32(f.y), round_tf32(f.z), round_tf32(f.w));
          reinterpret_cast<float4*>(x_hi + (int64_t)d * (row_bytes / 4))[v] = h;
          reinterpret_cast<float4*>(x_lo + (int64_t)d * (row_bytes / 4))[v] =
              make_float4(f.x - h.x, f.y - h.y, f.z - h.z, f.w - h.w);
        }
      }
    }
  }
  if (REMOTE) __threadfence_system();
}

// K3b on the TMA engine (large batches, local rows, no tf32 split): the
// same ranking as permute_kernel (one thread per token, warp ballots), then
// lane 0 of every warp moves its 32 tokens' rows with bulk copies: one
// cp.async.bulk global -> shared per row into a 3-slot ring (two loads in
// flight while a third row is being stored), one cp.async.bulk shared ->
// global per destination.  Rows move as whole 16-B-aligned byte ranges, so
// the SMs issue 1 + k instructions per row instead of row_bytes / 16 loads
// and stores per copy.
constexpr int PB_WARPS = 4;
constexpr int PB_SLOTS = 3;

__global__ void __launch_bounds__(PB_WARPS * 32) permute_bulk_kernel(
    const uint8_t* __restrict__ x, int row_bytes, int64_t T, int E, int k, const int32_t* __restrict__ served_idx,
    const int64_t* __restrict__ seg_offsets, const int64_t* __restrict__ block_base, uint8_t* __restrict__ x_perm,
    int32_t* __restrict__ pos, int32_t* __restrict__ row_token) {
  extern __shared__ __align__(128) uint8_t smb[];
  uint8_t* ring = smb;                                                            // [warps][slots][row_bytes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smb + PB_WARPS * PB_SLOTS * row_bytes);  // [warps][slots]
  int32_t* warp_counts = reinterpret_cast<int32_t*>(bars + PB_WARPS * PB_SLOTS);      // [4][E]
  int32_t* dst_s = warp_counts + 4 * E;                                              // [RT][k]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t0 = (int64_t)blockIdx.x * RT;
  const int64_t t = t0 + threadIdx.x;
  const bool valid = t < T;
  pdl_wait();
  pdl_trigger();
  int my[8], rank[8];
  for (int j = 0; j < k; ++j) {
    my[j] = valid ? served_idx[t * k + j] : -1;
    rank[j] = 0;
  }
  if (lane < PB_SLOTS) mbar_init(&bars[warp * PB_SLOTS + lane], 1);
  const uint32_t lt = (1u << lane) - 1u;
  if (k == 1) {
    for (int e = lane; e < E; e += 32) warp_counts[warp * E + e] = 0;
    __syncwarp();
    const uint32_t m = __match_any_sync(0xffffffffu, my[0]);
    if (my[0] >= 0) {
      rank[0] = __popc(m & lt);
      if (rank[0] == 0) warp_counts[warp * E + my[0]] = __popc(m);
    }
  } else {
    for (int e = 0; e < E; ++e) {
      bool has = false;
      for (int j = 0; j < k; ++j) has |= (my[j] == e);
      const uint32_t m = __ballot_sync(0xffffffffu, has);
      if (lane == 0) warp_counts[warp * E + e] = __popc(m);
      if (has)
        for (int j = 0; j < k; ++j)
          if (my[j] == e) rank[j] = __popc(m & lt);
    }
  }
  fence_barrier_init();
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const int e = my[j];
    int32_t d = -1;
    if (e >= 0) {
      int64_t base = seg_offsets[e] + block_base[(int64_t)blockIdx.x * E + e];
      for (int w = 0; w < warp; ++w) base += warp_counts[w * E + e];
      d = (int32_t)(base + rank[j]);
    }
    dst_s[threadIdx.x * k + j] = d;
    if (valid) {
      pos[t * k + j] = d;
      if (row_token && d >= 0) row_token[d] = (int32_t)t;
    }
  }
  __syncwarp();
  if (lane != 0) return;
  // this warp's served tokens, in order
  int list[32];
  int n = 0;
  for (int i = 0; i < 32; ++i) {
    const int r = warp * 32 + i;
    if (t0 + r < T && dst_s[r * k] >= 0) list[n++] = r;
  }
  uint8_t* slots = ring + (size_t)warp * PB_SLOTS * row_bytes;
  uint64_t* bar = bars + warp * PB_SLOTS;
  auto issue = [&](int q) {
    const int sl = q % PB_SLOTS;
    mbar_arrive_expect_tx(&bar[sl], (uint32_t)row_bytes);
    bulk_load_g2s(slots + (size_t)sl * row_bytes, x + (t0 + list[q]) * (int64_t)row_bytes, (uint32_t)row_bytes,
                  &bar[sl]);
  };
  for (int q = 0; q < PB_SLOTS - 1 && q < n; ++q) issue(q);
  for (int i = 0; i < n; ++i) {
    const int sl = i % PB_SLOTS;
    mbar_wait(&bar[sl], (uint32_t)((i / PB_SLOTS) & 1));
    const int r = list[i];
    for (int j = 0; j < k; ++j) {
      const int32_t d = dst_s[r * k + j];
      if (d < 0) break;  // served slots are compacted to the front
      bulk_store_s2g(x_perm + (int64_t)d * row_bytes, slots + (size_t)sl * row_bytes, (uint32_t)row_bytes);
    }
    bulk_commit_group();
    const int q = i + PB_SLOTS - 1;  // its slot last held row i - 1
    if (q < n) {
      bulk_wait_group_read<1>();  // row i - 1's stores have read their slot
      issue(q);
    }
  }
  bulk_wait_group_all();
}

// One warp per token; lanes own 16-byte column chunks.
__global__ void __launch_bounds__(256) combine_bf16_kernel(const __nv_bfloat16* __restrict__ Y, int64_t T, int d,
                                                           int k, const int32_t* __restrict__ pos,
                                                           const float* __restrict__ served_w,
                                                           __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  if (t >= T) return;
  int32_t p[8];
  float w[8];
  for (int j = 0; j < k; ++j) {
    p[j] = pos[t * k + j];
    w[j] = served_w[t * k + j];
  }
  const int nvec = d / 8;  // gridDim.y blocks share a token group, each a column slice (small T)
  const int v1 = (int)((int64_t)nvec * (blockIdx.y + 1) / gridDim.y);
  for (int v = (int)((int64_t)nvec * blockIdx.y / gridDim.y) + lane; v < v1; v += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < k; ++j) {
      if (p[j] < 0) continue;
      const uint4 r = __ldg(reinterpret_cast<const uint4*>(Y + (int64_t)p[j] * d) + v);
      const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[2 * q] += w[j] * bf16_lo(u[q]);
        acc[2 * q + 1] += w[j] * bf16_hi(u[q]);
      }
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    reinterpret_cast<uint4*>(y + t * d)[v] = o;
  }
}

__global__ void __launch_bounds__(256) combine_f32_kernel(const float* __restrict__ Y, int64_t T, int d, int k,
                                                          const int32_t* __restrict__ pos,
                                                          const float* __restrict__ served_w, float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  if (t >= T) return;
  int32_t p[8];
  float w[8];
  for (int j = 0; j < k; ++j) {
    p[j] = pos[t * k + j];
    w[j] = served_w[t * k + j];
  }
  const int nvec = d / 4;
  const int v1 = (int)((int64_t)nvec * (blockIdx.y + 1) / gridDim.y);
  for (int v = (int)((int64_t)nvec * blockIdx.y / gridDim.y) + lane; v < v1; v += 32) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int j = 0; j < k; ++j) {
      if (p[j] < 0) continue;
      const float4 r = __ldg(reinterpret_cast<const float4*>(Y + (int64_t)p[j] * d) + v);
      acc.x += w[j] * r.x;
      acc.y += w[j] * r.y;
      acc.z += w[j] * r.z;
      acc.w += w[j] * r.w;
    }
    reinterpret_cast<float4*>(y + t * d)[v] = acc;
  }
}

// EMOE_BULK_COPY=0 keeps the LDG/STG permute (A/B runs); the bulk kernel
// needs enough token blocks to fill the GPU
int bulk_min_blocks() {
  static const int v = [] {
    const char* e = getenv("EMOE_BULK_COPY");
    return e && e[0] == '0' ? (1 << 30) : 2 * 148;
  }();
  return v;
}

}  // namespace

void launch_scan(const int32_t* block_counts, int nblocks, int E, int pad, int32_t* counts, int64_t* seg_offsets,
                 int64_t* block_base, int32_t* row_token, int32_t* done, cudaStream_t s) {
  EMOE_REQUIRE(E >= 1 && E <= 1024, "scan: expert count out of range");
  EMOE_CUDA(launch_pdl(scan_kernel, dim3(E), dim3(SCAN_T), 0, s, 1, block_counts, nblocks, E, pad, block_base, counts,
                       seg_offsets, row_token, done));
  count_launch();
}

static void launch_permute_ss(const void* x, int elem_bytes, int64_t T, int d, int E, int k,
                              const int32_t* served_idx, const int64_t* seg_offsets, const int64_t* block_base,
                              void* x_perm, int32_t* pos, int32_t* row_token, cudaStream_t s, float* x_hi,
                              float* x_lo, const SmallScan& ss);

void launch_permute(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                    const int64_t* seg_offsets, const int64_t* block_base, void* x_perm, int32_t* pos,
                    int32_t* row_token, cudaStream_t s, float* x_hi, float* x_lo) {
  launch_permute_ss(x, elem_bytes, T, d, E, k, served_idx, seg_offsets, block_base, x_perm, pos, row_token, s, x_hi,
                    x_lo, SmallScan{});
}

void launch_scan_permute(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                         const int32_t* block_counts, int pad, int32_t* counts, int64_t* seg_offsets,
                         int64_t* block_base, void* x_perm, int32_t* pos, int32_t* row_token, int32_t* done,
                         cudaStream_t s, float* x_hi, float* x_lo) {
  static const bool fold = [] {  // EMOE_SMALL_SCAN=0 keeps the separate scan launch (A/B runs)
    const char* v = getenv("EMOE_SMALL_SCAN");
    return !(v && v[0] == '0');
  }();
  const int nblocks = (int)ceil_div(T, RT);
  if (fold && nblocks >= 1 && nblocks <= SMALL_SCAN_BLOCKS && E <= SMALL_SCAN_E) {
    SmallScan ss;
    ss.block_counts = block_counts;
    ss.nblocks = nblocks;
    ss.pad = pad;
    ss.counts = counts;
    ss.seg_offsets = seg_offsets;
    launch_permute_ss(x, elem_bytes, T, d, E, k, served_idx, seg_offsets, block_base, x_perm, pos, row_token, s, x_hi,
                      x_lo, ss);
    return;
  }
  launch_scan(block_counts, nblocks, E, pad, counts, seg_offsets, block_base, row_token, done, s);
  launch_permute(x, elem_bytes, T, d, E, k, served_idx, seg_offsets, block_base, x_perm, pos, row_token, s, x_hi,
                 x_lo);
}

static void launch_permute_ss(const void* x, int elem_bytes, int64_t T, int d, int E, int k,
                              const int32_t* served_idx, const int64_t* seg_offsets, const int64_t* block_base,
                              void* x_perm, int32_t* pos, int32_t* row_token, cudaStream_t s, float* x_hi,
                              float* x_lo, const SmallScan& ss) {
  EMOE_REQUIRE(!x_hi || (elem_bytes == 4 && x_lo), "permute: the tf32 split needs fp32 rows and both outputs");
  const int row_bytes = d * elem_bytes;
  EMOE_REQUIRE(row_bytes % 16 == 0, "permute: row bytes must be a multiple of 16");
  const int nblocks = (int)ceil_div(T, RT);
  if (nblocks == 0) return;
  const size_t smem = (4 * (size_t)E + (size_t)RT * k) * sizeof(int32_t);
  // few token blocks (small T): split each block's rows by columns over
  // gridDim.y blocks so the gather still spans the GPU (>= 8 x 16 B per row slice)
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int ny = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * sms, nblocks), row_bytes / 16 / 8));
  // large batches of long rows (>= 4 KB): rows moved by the TMA engine.
  // Shorter rows (Switch shape, 1.5 KB) stay on LDG/STG: 44 vs 35 us at
  // T = 65,536 -- one bulk copy in flight per 1.5 KB row is too little
  // parallelism (profiles/r02_bulk_copy_ab.txt)
  if (!x_hi && nblocks >= bulk_min_blocks() && row_bytes >= 4096) {
    const size_t bsmem = (size_t)PB_WARPS * PB_SLOTS * row_bytes + (size_t)PB_WARPS * PB_SLOTS * 8 +
                         (4 * (size_t)E + (size_t)RT * k) * sizeof(int32_t);
    if (bsmem <= 200 * 1024) {
      if (bsmem > 48 * 1024) ensure_max_dynamic_smem(reinterpret_cast<const void*>(permute_bulk_kernel), (int)bsmem);
      EMOE_CUDA(launch_pdl(permute_bulk_kernel, dim3(nblocks), dim3(PB_WARPS * 32), bsmem, s, 1,
                           static_cast<const uint8_t*>(x), row_bytes, T, E, k, served_idx, seg_offsets, block_base,
                           static_cast<uint8_t*>(x_perm), pos, row_token));
      count_launch();
      return;
    }
  }
  auto kernel = x_hi ? permute_kernel<false, true> : permute_kernel<false, false>;
  EMOE_CUDA(launch_pdl(kernel, dim3(nblocks, ny), dim3(PERMUTE_THREADS), smem, s, 1,
                       static_cast<const uint8_t*>(x), row_bytes, T, E, k, served_idx, seg_offsets, block_base,
                       static_cast<uint8_t*>(x_perm), pos, row_token, PeerRows{}, x_hi, x_lo, ss));
  count_launch();
}

void launch_permute_remote(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                           const int64_t* seg_offsets, const int64_t* block_base, const PeerRows& peers,
                           int32_t* pos, cudaStream_t s) {
  const int row_bytes = d * elem_bytes;
  EMOE_REQUIRE(row_bytes % 16 == 0, "permute: row bytes must be a multiple of 16");
  const int nblocks = (int)ceil_div(T, RT);
  if (nblocks == 0) return;
  const size_t smem = (4 * (size_t)E + (size_t)((RT * k + 1) & ~1)) * sizeof(int32_t) + (size_t)RT * k * 8;
  permute_kernel<true><<<nblocks, PERMUTE_THREADS, smem, s>>>(static_cast<const uint8_t*>(x), row_bytes, T, E, k,
                                                              served_idx, seg_offsets, block_base, nullptr, pos,
                                                              nullptr, peers, nullptr, nullptr, SmallScan{});
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

void launch_combine(const void* Y, int dtype, int64_t T, int d, int k, const int32_t* pos, const float* served_w,
                    void* y, cudaStream_t s) {
  const int nblocks = (int)ceil_div(T, 8);
  if (nblocks == 0) return;
  // few token groups (small T): split the columns over gridDim.y blocks so
  // the combine still spans the GPU (>= 32 vectors per slice)
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int nvec = dtype == DT_F32 ? d / 4 : d / 8;
  const int ny = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * sms, nblocks), nvec / 32));
  if (dtype == DT_F32) {
    EMOE_REQUIRE(d % 4 == 0, "combine: d must be a multiple of 4");
    EMOE_CUDA(launch_pdl(combine_f32_kernel, dim3(nblocks, ny), dim3(256), 0, s, 1, static_cast<const float*>(Y), T,
                         d, k, pos, served_w, static_cast<float*>(y)));
  } else {
    EMOE_REQUIRE(d % 8 == 0, "combine: d must be a multiple of 8");
    EMOE_CUDA(launch_pdl(combine_bf16_kernel, dim3(nblocks, ny), dim3(256), 0, s, 1,
                         static_cast<const __nv_bfloat16*>(Y), T, d, k, pos, served_w, static_cast<__nv_bfloat16*>(y)));
  }
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace emoe
