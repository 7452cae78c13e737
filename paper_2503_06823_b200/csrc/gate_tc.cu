// K1 for many experts (E in {32, 64, 96, 128}, bf16): the gate GEMM on
// tcgen05 with the routing fused into its epilogue, so x is read once and
// the fp32 logits never round-trip through HBM.
//
// Tile = 128 tokens x all E experts (UMMA N = E, K = 16 per instruction,
// fp32 accumulators in TMEM).  TMEM lane = token: every epilogue thread reads
// its own token's logits row from TMEM in 32-column chunks and routes it in
// registers -- a running top-k in one pass, and for the full-softmax weight
// mode a second pass for the denominator -- with the operations, and the
// order, of routing::route_one_token + route_tail (route_tail.cuh), so the
// results are bit-identical to routing the stored logits.
//
// Two forms, both persistent with NG = 4 epilogue warp groups (TMEM holds
// four accumulator buffers; group g routes the tiles with it % 4 == g, so four
// tiles are routed concurrently while the next ones load -- the per-token
// routing is a long dependent chain and one warp per SM sub-partition could
// not hide it):
//   pair    (default where it fits) CTA pairs, tcgen05.mma.cta_group::2,
//           M = 256 tokens: each CTA keeps its half of W_g resident in shared
//           memory for the whole kernel (E/2 x d x 2 bytes, 96 KB at E = 128,
//           d = 768), so only x streams from HBM, through a ring of up to 8
//           16-KB stages
//   stream  each CTA streams its x tile and the gate k-blocks; a cluster of
//           CN CTAs shares every gate k-block by TMA multicast (CN = 2
//           default), and every CTA's MMA commit releases the stage in all of
//           them (the rings run in lockstep; a CTA past the end computes a
//           zero-filled tile and stores nothing)
// warp 0 = TMA producer, warp 1 = MMA issuer (one thread), warps 2.. = the
// epilogue groups.  Per-tile expert counts (block_counts, the permutation's
// input) are tallied per group in shared memory.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "route_tail.cuh"

namespace emoe {
namespace gatetc {

constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int NG = 4;   // epilogue warp groups = TMEM accumulator buffers
constexpr int NUM_THREADS = 64 + 128 * NG;
constexpr int A_BYTES = 128 * BK * 2;
constexpr int MAX_STAGES = 8;
constexpr int BAR_BYTES = 1024;  // mbarriers and the TMEM slot
constexpr int SMEM_LIMIT = 227 * 1024 - 4096;  // dynamic bytes: static shared state and alignment slack stay free

struct Params {
  RouteArgs a;
  RouteOut o;
  int64_t ntiles;
  int k_blocks;
  int stages;
  int store_logits;
};

__device__ __forceinline__ void group_sync(int g) {  // the 4 warps of epilogue group g
  asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
}

// One 32-column chunk of this thread's logits row (+ the caller's bias).
__device__ __forceinline__ void load_chunk(uint32_t taddr, int c, int64_t t, bool live, const RouteArgs& a, int NE,
                                           float (&v)[32]) {
  uint32_t r[32];
  tmem_ld_32x32b_x32(taddr + c * 32, r);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (live && a.bias) {
    const float4* b4 = reinterpret_cast<const float4*>(a.bias + t * NE + c * 32);
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 bb = __ldg(b4 + j / 4);
      v[j] += bb.x;
      v[j + 1] += bb.y;
      v[j + 2] += bb.z;
      v[j + 3] += bb.w;
    }
  }
}

// Route this thread's token (TMEM lane) of the tile at taddr.  Top-k by a
// running insertion with strict comparisons in index order (a value displaces
// an entry only when larger, so ties keep the lower index: the order of
// route_one_token's repeated argmax); then route_tail's remap, served set
// and weights.  Every TMEM read is done when it returns.
template <int NE>
__device__ __forceinline__ void route_from_tmem(uint32_t taddr, int64_t t, bool live, const Params& p,
                                                const routing::SharedRouteState& st, int* counts) {
  const RouteArgs& a = p.a;
  const RouteOut& o = p.o;
  const int k = a.k;
  float tv[8];
  int ti[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    tv[r] = 0.0f;
    ti[r] = -1;
  }
  int n = 0;
#pragma unroll 1
  for (int c = 0; c < NE / 32; ++c) {
    float v[32];
    load_chunk(taddr, c, t, live, a, NE, v);
    if (live && p.store_logits && o.logits) {
      float4* dst = reinterpret_cast<float4*>(o.logits + t * NE + c * 32);
#pragma unroll
      for (int j = 0; j < 32; j += 4) dst[j / 4] = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
    if (k == 1) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (ti[0] < 0 || v[j] > tv[0]) {
          tv[0] = v[j];
          ti[0] = c * 32 + j;
        }
    } else if (k == 2) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int e = c * 32 + j;
        if (ti[0] < 0 || v[j] > tv[0]) {
          tv[1] = tv[0];
          ti[1] = ti[0];
          tv[0] = v[j];
          ti[0] = e;
        } else if (ti[1] < 0 || v[j] > tv[1]) {
          tv[1] = v[j];
          ti[1] = e;
        }
      }
    } else {
#pragma unroll 1
      for (int j = 0; j < 32; ++j) {
        const float x = v[j];
        if (n == k && !(x > tv[k - 1])) continue;
        int pos = n < k ? n : k - 1;
        while (pos > 0 && x > tv[pos - 1]) {
          tv[pos] = tv[pos - 1];
          ti[pos] = ti[pos - 1];
          --pos;
        }
        tv[pos] = x;
        ti[pos] = c * 32 + j;
        if (n < k) ++n;
      }
    }
  }
  // route_token remap (expert_store.cpp:206-220, engine.cpp:533-537)
  int ex = -1, rk = -1, hit = 0;
  if (live) {
    if (st.n_res == 0) {
      ex = ti[0];
      if (!a.forced_miss) atomicExch(a.error_flag, 3);
    } else {
      for (int r = 0; r < k; ++r)
        if (st.resident[ti[r]]) {
          ex = ti[r];
          rk = r;
          hit = r == 0;
          break;
        }
      if (rk < 0) ex = st.fallback;
    }
  }
  // full-softmax weights: the denominator over every logit in index order
  // (route_tail's serial sum), and the fallback expert's logit
  float den1 = 0.0f, vex = 0.0f;
  if (a.weight_mode != 0) {
    const float mx = tv[0];
#pragma unroll 1
    for (int c = 0; c < NE / 32; ++c) {
      float v[32];
      load_chunk(taddr, c, t, live, a, NE, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        den1 += expf(v[j] - mx);
        if (c * 32 + j == ex) vex = v[j];
      }
    }
  }
  if (!live) return;
  if (o.topk_idx)
    for (int r = 0; r < k; ++r) o.topk_idx[t * k + r] = ti[r];
  if (o.route_expert) o.route_expert[t] = ex;
  if (o.route_rank) o.route_rank[t] = rk;
  if (o.route_hit) o.route_hit[t] = (uint8_t)hit;
  int si[8];
  float sv[8];  // the served experts' logits
  int ns = 0;
  if (st.n_res > 0) {
    if (rk >= 0) {
      for (int r = 0; r < k; ++r)
        if (st.resident[ti[r]]) {
          sv[ns] = tv[r];
          si[ns++] = ti[r];
        }
    } else {
      sv[ns] = a.weight_mode == 0 ? 0.0f : vex;  // mode 0: a lone served expert's weight is expf(0) / expf(0)
      si[ns++] = ex;
    }
  }
  float w[8];
  if (a.weight_mode == 0) {
    if (ns > 0) {
      const float mx = sv[0];
      float den = 0.0f;
      for (int j = 0; j < ns; ++j) {
        w[j] = expf(sv[j] - mx);
        den += w[j];
      }
      for (int j = 0; j < ns; ++j) w[j] = w[j] / den;
    }
  } else {
    const float mx = tv[0];
    for (int j = 0; j < ns; ++j) w[j] = expf(sv[j] - mx) / den1;
  }
  for (int j = 0; j < k; ++j) {
    o.served_idx[t * k + j] = j < ns ? si[j] : -1;
    o.served_w[t * k + j] = j < ns ? w[j] : 0.0f;
  }
  for (int j = 0; j < ns; ++j) atomicAdd(&counts[si[j]], 1);
}

// The epilogue of one tile for epilogue group g: route, release the TMEM
// buffer, flush the tile's expert counts.
template <int NE>
__device__ __forceinline__ void epilogue_tile(uint32_t taddr, int64_t tile, int quarter, int lane, int g,
                                              const Params& p, const routing::SharedRouteState& st, int* counts,
                                              uint64_t* tempty, bool to_leader) {
  const int64_t t = tile * 128 + quarter * 32 + lane;
  const bool live = tile < p.ntiles && t < p.a.T;
  route_from_tmem<NE>(taddr, t, live, p, st, counts);
  tc_fence_before();
  if (lane == 0) {
    if (to_leader)
      mbar_arrive_leader_relaxed(tempty);
    else
      mbar_arrive_relaxed(tempty);
  }
  if (tile < p.ntiles) {
    group_sync(g);  // every token of the tile counted
    const int tg = (threadIdx.x - 64) % 128;
    if (p.o.block_counts)
      for (int e = tg; e < p.a.E; e += 128) {
        p.o.block_counts[tile * p.a.E + e] = counts[e];
        counts[e] = 0;
      }
    group_sync(g);
  }
}

template <int NE>
constexpr int tmem_cols() {
  return NG * NE <= 128 ? 128 : (NG * NE <= 256 ? 256 : 512);
}

// ---------------------------------------------------------------------------
// stream form
// ---------------------------------------------------------------------------
template <int NE, int CN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gate_route_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_g,
                         Params p) {
  constexpr int B_BYTES = NE * BK * 2;
  constexpr int SLICE_ROWS = NE / CN;
  constexpr int SLICE_BYTES = SLICE_ROWS * BK * 2;
  constexpr int TMEM_COLS = tmem_cols<NE>();
  constexpr uint16_t MASK = (uint16_t)((1u << CN) - 1u);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_b + S * B_BYTES);
  uint64_t* empty_bar = full_bar + MAX_STAGES;
  uint64_t* tfull_bar = empty_bar + MAX_STAGES;  // [NG]
  uint64_t* tempty_bar = tfull_bar + NG;         // [NG]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + NG);
  int* g_counts = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full_bar) + BAR_BYTES);  // [NG][NE]
  __shared__ routing::SharedRouteState st;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = CN > 1 ? cluster_ctarank() : 0;
  const int64_t cluster_id = blockIdx.x / CN, n_clusters = gridDim.x / CN;
  // every CTA of a cluster walks the same number of tile slots
  const int64_t n_iter = (ceil_div(p.ntiles, CN) + n_clusters - 1 - cluster_id) / n_clusters;

  for (int i = threadIdx.x; i < NG * NE; i += NUM_THREADS) g_counts[i] = 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_g);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CN);  // one MMA commit from every CTA of the cluster
    }
    for (int b = 0; b < NG; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  // barriers, TMEM and descriptors are set up: from here on the kernel reads
  // what preceding kernels wrote (x, the residency tables)
  pdl_wait();
  pdl_trigger();
  routing::load_route_state(st, p.a);
  tc_fence_before();
  if (CN > 1)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0; it < n_iter; ++it) {
        const int64_t tile = (cluster_id + it * n_clusters) * CN + rank;  // >= ntiles: zero-filled rows
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], A_BYTES + B_BYTES);
          tma_load_2d(&tmap_x, &full_bar[stage], smem_a + stage * A_BYTES, kb * BK, (int32_t)(tile * 128),
                      kCacheEvictFirst);
          uint8_t* bdst = smem_b + stage * B_BYTES + rank * SLICE_BYTES;
          if (CN > 1)
            tma_load_2d_mcast(&tmap_g, &full_bar[stage], bdst, kb * BK, (int32_t)(rank * SLICE_ROWS), MASK,
                              kCacheEvictLast);
          else
            tma_load_2d(&tmap_g, &full_bar[stage], bdst, kb * BK, 0, kCacheEvictLast);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // tail: every peer's last commits to this CTA's empty barriers have landed
      for (int i = 0; i < S; ++i) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, NE);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0; it < n_iter; ++it) {
        const int buf = (int)(it % NG);
        mbar_wait(&tempty_bar[buf], (uint32_t)((it / NG) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * NE;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = umma_desc_sw128(smem_a + stage * A_BYTES);
          const uint64_t b_desc = umma_desc_sw128(smem_b + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(tmem_d, a_desc + (uint64_t)(kk * 2), b_desc + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          if (CN > 1)
            umma_commit_mcast(&empty_bar[stage], MASK);
          else
            umma_commit(&empty_bar[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[buf]);
      }
    }
  } else {
    const int g = (warp - 2) / 4, quarter = warp & 3;
    for (int64_t it = g; it < n_iter; it += NG) {
      const int64_t tile = (cluster_id + it * n_clusters) * CN + rank;
      mbar_wait(&tfull_bar[g], (uint32_t)((it / NG) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + g * NE;
      epilogue_tile<NE>(taddr, tile, quarter, lane, g, p, st, g_counts + g * NE, &tempty_bar[g], false);
    }
  }

  if (CN > 1)
    cluster_sync_all();
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// pair form: the gate resident in shared memory, cta_group::2
// ---------------------------------------------------------------------------
template <int NE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gate_route_tc2_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_g,
                          Params p) {
  constexpr int BH = NE / 2;             // gate rows this CTA holds
  constexpr int KB_BYTES = BH * BK * 2;  // one resident k-block
  constexpr int TMEM_COLS = tmem_cols<NE>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* smem_a = smem;               // [S][A_BYTES]
  uint8_t* b_res = smem + S * A_BYTES;  // [k_blocks][KB_BYTES]
  uint8_t* bar_area = b_res + (size_t)p.k_blocks * KB_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty_bar = full_bar + MAX_STAGES;
  uint64_t* tfull_bar = empty_bar + MAX_STAGES;  // [NG]
  uint64_t* tempty_bar = tfull_bar + NG;         // [NG]
  uint64_t* bres_bar = tempty_bar + NG;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_bar + 1);
  int* g_counts = reinterpret_cast<int*>(bar_area + BAR_BYTES);  // [NG][NE]
  __shared__ routing::SharedRouteState st;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t pair_id = blockIdx.x / 2, n_pairs = gridDim.x / 2;
  const int64_t ntiles2 = ceil_div(p.ntiles, 2);  // 256-token pair tiles
  const int64_t n_iter = (ntiles2 + n_pairs - 1 - pair_id) / n_pairs;

  for (int i = threadIdx.x; i < NG * NE; i += NUM_THREADS) g_counts[i] = 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_g);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < NG; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 8);  // 4 epilogue warps x 2 CTAs (the leader's copy counts)
    }
    mbar_init(bres_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  pdl_wait();
  pdl_trigger();
  routing::load_route_state(st, p.a);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // the resident gate half, once; completion bytes to the leader's barrier
      if (leader) mbar_arrive_expect_tx(bres_bar, 2u * p.k_blocks * KB_BYTES);
      for (int kb = 0; kb < p.k_blocks; ++kb)
        tma_load_2d_pair(&tmap_g, bres_bar, b_res + kb * KB_BYTES, kb * BK, (int32_t)(rank * BH), kCacheEvictLast);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0; it < n_iter; ++it) {
        const int64_t tile2 = pair_id + it * n_pairs;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * A_BYTES);
          tma_load_2d_pair(&tmap_x, &full_bar[stage], smem_a + stage * A_BYTES, kb * BK,
                           (int32_t)(tile2 * 256 + rank * 128), kCacheEvictFirst);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      for (int i = 0; i < S; ++i) {  // the leader's last commits to this CTA have landed
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, NE);
      mbar_wait(bres_bar, 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0; it < n_iter; ++it) {
        const int buf = (int)(it % NG);
        mbar_wait(&tempty_bar[buf], (uint32_t)((it / NG) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * NE;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = umma_desc_sw128(smem_a + stage * A_BYTES);
          const uint64_t b_desc = umma_desc_sw128(b_res + kb * KB_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_pair(tmem_d, a_desc + (uint64_t)(kk * 2), b_desc + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          umma_commit_pair(&empty_bar[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull_bar[buf]);
      }
    }
  } else {
    const int g = (warp - 2) / 4, quarter = warp & 3;
    for (int64_t it = g; it < n_iter; it += NG) {
      const int64_t tile = (pair_id + it * n_pairs) * 2 + rank;  // this CTA's 128-token block
      mbar_wait(&tfull_bar[g], (uint32_t)((it / NG) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + g * NE;
      epilogue_tile<NE>(taddr, tile, quarter, lane, g, p, st, g_counts + g * NE, &tempty_bar[g], !leader);
    }
  }

  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

// shared memory of the two forms at `stages` ring stages
int smem_bytes(bool pair, int E, int k_blocks, int stages) {
  const int fixed = 1024 + BAR_BYTES + NG * E * 4;
  return pair ? fixed + stages * A_BYTES + k_blocks * (E / 2) * BK * 2 : fixed + stages * (A_BYTES + E * BK * 2);
}
int max_stages(bool pair, int E, int k_blocks) {
  int s = MAX_STAGES;
  while (s > 2 && smem_bytes(pair, E, k_blocks, s) > SMEM_LIMIT) --s;
  return s;
}

template <typename K>
void launch(K kernel, int cluster, int grid, int smem, const CUtensorMap& tx, const CUtensorMap& tg, const Params& p,
            cudaStream_t s) {
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
  EMOE_CUDA(launch_pdl(kernel, dim3(grid), dim3(NUM_THREADS), (size_t)smem, s, cluster, tx, tg, p));
  count_launch();
}

template <int NE>
void launch_pair(const CUtensorMap& tx, const CUtensorMap& tg, Params p, int num_sms, cudaStream_t s) {
  p.stages = max_stages(true, NE, p.k_blocks);
  const int grid = (int)std::min<int64_t>(num_sms / 2 * 2, ceil_div(p.ntiles, 2) * 2);
  launch(gate_route_tc2_kernel<NE>, 2, grid, smem_bytes(true, NE, p.k_blocks, p.stages), tx, tg, p, s);
}

template <int NE, int CN>
void launch_stream(const CUtensorMap& tx, const CUtensorMap& tg, Params p, int num_sms, cudaStream_t s) {
  p.stages = max_stages(false, NE, p.k_blocks);
  const int grid = (int)std::min<int64_t>(num_sms / CN * CN, ceil_div(p.ntiles, CN) * CN);
  launch(gate_route_tc_kernel<NE, CN>, CN, grid, smem_bytes(false, NE, p.k_blocks, p.stages), tx, tg, p, s);
}

}  // namespace gatetc

// Which form runs (EMOE_GATE_TC=pair|stream overrides for A/B runs): the
// pair form whenever the gate half fits in shared memory next to a ring of
// at least 4 stages, else the stream form with the gate k-blocks multicast
// over a cluster of EMOE_GATE_CLUSTER (default 2) CTAs.
static bool gate_tc_pair(int E, int d) {
  static const int force = [] {
    const char* v = getenv("EMOE_GATE_TC");
    return v ? (std::strcmp(v, "pair") == 0 ? 1 : std::strcmp(v, "stream") == 0 ? 0 : -1) : -1;
  }();
  const int kb = d / gatetc::BK;
  const bool fits = gatetc::smem_bytes(true, E, kb, 4) <= gatetc::SMEM_LIMIT;
  return force == 0 ? false : fits;
}

static int gate_tc_cluster() {
  static const int cn = [] {  // EMOE_GATE_CLUSTER: 1, 2 or 4 CTAs sharing the gate k-blocks (A/B runs)
    const char* v = getenv("EMOE_GATE_CLUSTER");
    const int c = v ? atoi(v) : 2;
    return c == 1 || c == 4 ? c : 2;
  }();
  return cn;
}

int gate_tc_box_rows(int E, int d) { return gate_tc_pair(E, d) ? E / 2 : E / gate_tc_cluster(); }

void launch_gate_route_tc(const CUtensorMap& tmap_x, const CUtensorMap& tmap_gate_slice, const RouteArgs& a,
                          const RouteOut& o, bool store_logits, int num_sms, cudaStream_t s) {
  EMOE_REQUIRE(a.E >= 32 && a.E <= 128 && a.E % 32 == 0, "gate_tc: E must be 32, 64, 96 or 128");
  EMOE_REQUIRE(a.d % gatetc::BK == 0, "gate_tc: d_model must be a multiple of 64");
  EMOE_REQUIRE(a.k >= 1 && a.k <= 8 && a.k <= a.E, "gate_tc: top_k must be in [1, min(8, E)]");
  gatetc::Params p;
  p.a = a;
  p.o = o;
  p.ntiles = ceil_div(a.T, 128);
  p.k_blocks = a.d / gatetc::BK;
  p.stages = 0;
  p.store_logits = store_logits ? 1 : 0;
  if (p.ntiles == 0) return;
  if (gate_tc_pair(a.E, a.d)) {
    switch (a.E) {
      case 32: gatetc::launch_pair<32>(tmap_x, tmap_gate_slice, p, num_sms, s); break;
      case 64: gatetc::launch_pair<64>(tmap_x, tmap_gate_slice, p, num_sms, s); break;
      case 96: gatetc::launch_pair<96>(tmap_x, tmap_gate_slice, p, num_sms, s); break;
      default: gatetc::launch_pair<128>(tmap_x, tmap_gate_slice, p, num_sms, s); break;
    }
    return;
  }
  const int cn = gate_tc_cluster();
  EMOE_REQUIRE(gatetc::smem_bytes(false, a.E, p.k_blocks, 2) <= gatetc::SMEM_LIMIT, "gate_tc: tile too large");
  switch (a.E) {
#define EMOE_GATE_CASE(NEV)                                                        \
  case NEV:                                                                        \
    if (cn == 1)                                                                   \
      gatetc::launch_stream<NEV, 1>(tmap_x, tmap_gate_slice, p, num_sms, s);       \
    else if (cn == 2)                                                              \
      gatetc::launch_stream<NEV, 2>(tmap_x, tmap_gate_slice, p, num_sms, s);       \
    else                                                                           \
      gatetc::launch_stream<NEV, 4>(tmap_x, tmap_gate_slice, p, num_sms, s);       \
    break;
    EMOE_GATE_CASE(32)
    EMOE_GATE_CASE(64)
    EMOE_GATE_CASE(96)
    EMOE_GATE_CASE(128)
#undef EMOE_GATE_CASE
  }
}

}  // namespace emoe
