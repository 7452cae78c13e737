// K1 for many experts (E in {32, 64, 96, 128}, bf16): the gate GEMM on
// tcgen05 with the routing fused into its epilogue, so x is read once and
// the fp32 logits never round-trip through HBM.
//
// Tile = 128 tokens x all E experts (UMMA M=128, N=E, K=16 per instruction,
// fp32 accumulators in TMEM).  TMEM lane = token: after the accumulator is
// read (tcgen05.ld 32x32b), every epilogue thread holds its token's whole
// logits row in registers and routes it exactly as the per-thread reference
// restatement does (route.cu route_one_token + route_tail: top-k descending
// with ascending index on ties, route_token remap, served set and weights,
// with the same operation order, so results are bit-identical to routing the
// stored logits).
//
// Hardware mapping (persistent, one CTA per SM, clusters of CN CTAs):
//   warp 0      TMA producer: its own 128 x 64 x-tile per k-block, plus a
//               1/CN slice of the gate's k-block multicast to every CTA of
//               the cluster (the gate is the same for every tile, so a
//               cluster shares each B k-block: L2 -> SM traffic for W_g drops
//               CN-fold; at E = 128 the gate's reads would otherwise equal x's)
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1 per k-block, commit
//               multicast to the stage's empty barrier of every cluster CTA
//               (a stage is refilled only when all CN CTAs consumed it)
//   warps 2..5  epilogue: TMEM double-buffered (2 x E columns) so tile i is
//               routed while tile i+1's loads and MMAs run; per-tile expert
//               counts in shared memory for the permutation (block_counts)
// Every CTA of a cluster walks the same number of tiles (a CTA past the end
// computes a zero-filled tile and stores nothing) so the multicast ring stays
// in lockstep.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "route_tail.cuh"

namespace emoe {
namespace gatetc {

constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int STAGES = 4;
constexpr int NUM_THREADS = 192;
constexpr int A_BYTES = 128 * BK * 2;
constexpr int BAR_BYTES = 1024;  // mbarriers and the TMEM slot, before the epilogue rows

struct Params {
  RouteArgs a;
  RouteOut o;
  int64_t ntiles;
  int k_blocks;
  int store_logits;
};

__device__ __forceinline__ void epi_sync() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <int NE, int CN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gate_route_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_g,
                         Params p) {
  constexpr int B_BYTES = NE * BK * 2;
  constexpr int SLICE_ROWS = NE / CN;
  constexpr int SLICE_BYTES = SLICE_ROWS * BK * 2;
  constexpr int TMEM_COLS = 2 * NE <= 64 ? 64 : (2 * NE <= 128 ? 128 : 256);
  constexpr uint16_t MASK = (uint16_t)((1u << CN) - 1u);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_b + STAGES * B_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  // the epilogue's logits rows, one per token: [128][NE + 1] fp32 (the pitch
  // puts a warp's per-thread row accesses on 32 distinct banks)
  float* s_rows = reinterpret_cast<float*>(smem_b + STAGES * B_BYTES + BAR_BYTES);
  __shared__ routing::SharedRouteState st;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = CN > 1 ? cluster_ctarank() : 0;
  const int64_t cluster_id = blockIdx.x / CN, n_clusters = gridDim.x / CN;
  // every CTA of a cluster walks the same number of tile slots
  const int64_t n_iter = (ceil_div(p.ntiles, CN) + n_clusters - 1 - cluster_id) / n_clusters;
  const RouteArgs& a = p.a;
  const int E = a.E;

  routing::load_route_state(st, a);  // residency, scores, the token-independent fallback (all threads)
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_g);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CN);  // one MMA commit from every CTA of the cluster
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
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
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // tail: every peer's last commits to this CTA's empty barriers have landed
      for (int i = 0; i < STAGES; ++i) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == STAGES) {
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
        const int buf = (int)(it & 1);
        mbar_wait(&tempty_bar[buf], (uint32_t)((it >> 1) & 1) ^ 1);
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
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[buf]);
      }
    }
  } else {
    // epilogue: TMEM lane = token; each thread moves its row to shared memory
    // (adding the bias / storing the logits on the way) and routes it
    const int quarter = warp & 3;
    const RouteOut& o = p.o;
    float* row = s_rows + (quarter * 32 + lane) * (NE + 1);
    for (int64_t it = 0; it < n_iter; ++it) {
      const int buf = (int)(it & 1);
      const int64_t tile = (cluster_id + it * n_clusters) * CN + rank;
      const int64_t t = tile * 128 + quarter * 32 + lane;
      const bool live = tile < p.ntiles && t < a.T;
      mbar_wait(&tfull_bar[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * NE;
#pragma unroll 1
      for (int c = 0; c < NE / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        float v[32];
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
        if (live && p.store_logits && o.logits) {
          float4* dst = reinterpret_cast<float4*>(o.logits + t * NE + c * 32);
#pragma unroll
          for (int j = 0; j < 32; j += 4) dst[j / 4] = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) row[c * 32 + j] = v[j];
      }
      tc_fence_before();
      if (lane == 0) mbar_arrive_relaxed(&tempty_bar[buf]);  // the MMAs of tile i+2 may start
      if (tile < p.ntiles) {
        if (live) routing::route_one_token(row, t, a, o, st);
        epi_sync();  // every token of the tile counted
        if (o.block_counts)
          for (int e = threadIdx.x - 64; e < E; e += 128) {
            o.block_counts[tile * E + e] = st.counts[e];
            st.counts[e] = 0;
          }
        epi_sync();
      }
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
// CTA-pair form with the gate resident in shared memory (E/2 x d x 2 bytes
// per CTA fits next to the x ring, e.g. 96 KB at E = 128, d = 768): each pair
// computes 256 tokens x E per tile with tcgen05.mma.cta_group::2 (M = 256; A =
// each CTA's own 128 token rows, B = each CTA's resident half of W_g), so only
// x streams from HBM -- no per-tile reload of W_g into shared memory, half the
// L2 -> SM bytes of the streaming form.  Each CTA's TMEM holds its own 128
// tokens x all E experts, so the epilogue is the streaming form's.
// ---------------------------------------------------------------------------
constexpr int PAIR_STAGES = 3;

template <int NE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gate_route_tc2_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_g,
                          Params p) {
  constexpr int BH = NE / 2;             // gate rows this CTA holds
  constexpr int KB_BYTES = BH * BK * 2;  // one resident k-block
  constexpr int TMEM_COLS = 2 * NE <= 64 ? 64 : (2 * NE <= 128 ? 128 : 256);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;                                        // [PAIR_STAGES][A_BYTES]
  uint8_t* b_res = smem + PAIR_STAGES * A_BYTES;                 // [k_blocks][KB_BYTES]
  uint8_t* bar_area = b_res + (size_t)p.k_blocks * KB_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty_bar = full_bar + PAIR_STAGES;
  uint64_t* tfull_bar = empty_bar + PAIR_STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;           // [2]
  uint64_t* bres_bar = tempty_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_bar + 1);
  float* s_rows = reinterpret_cast<float*>(bar_area + BAR_BYTES);  // [128][NE + 1]
  __shared__ routing::SharedRouteState st;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t pair_id = blockIdx.x / 2, n_pairs = gridDim.x / 2;
  const int64_t ntiles2 = ceil_div(p.ntiles, 2);  // 256-token pair tiles
  const int64_t n_iter = (ntiles2 + n_pairs - 1 - pair_id) / n_pairs;
  const RouteArgs& a = p.a;
  const int E = a.E;

  routing::load_route_state(st, a);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_g);
    for (int s = 0; s < PAIR_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
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
          if (++stage == PAIR_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      for (int i = 0; i < PAIR_STAGES; ++i) {  // the leader's last commits to this CTA have landed
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == PAIR_STAGES) {
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
        const int buf = (int)(it & 1);
        mbar_wait(&tempty_bar[buf], (uint32_t)((it >> 1) & 1) ^ 1);
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
          if (++stage == PAIR_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull_bar[buf]);
      }
    }
  } else {
    const int quarter = warp & 3;
    const RouteOut& o = p.o;
    float* row = s_rows + (quarter * 32 + lane) * (NE + 1);
    for (int64_t it = 0; it < n_iter; ++it) {
      const int buf = (int)(it & 1);
      const int64_t tile = (pair_id + it * n_pairs) * 2 + rank;  // this CTA's 128-token block
      const int64_t t = tile * 128 + quarter * 32 + lane;
      const bool live = tile < p.ntiles && t < a.T;
      mbar_wait(&tfull_bar[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * NE;
#pragma unroll 1
      for (int c = 0; c < NE / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        float v[32];
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
        if (live && p.store_logits && o.logits) {
          float4* dst = reinterpret_cast<float4*>(o.logits + t * NE + c * 32);
#pragma unroll
          for (int j = 0; j < 32; j += 4) dst[j / 4] = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) row[c * 32 + j] = v[j];
      }
      tc_fence_before();
      if (lane == 0) {
        if (leader)
          mbar_arrive_relaxed(&tempty_bar[buf]);
        else
          mbar_arrive_leader_relaxed(&tempty_bar[buf]);
      }
      if (tile < p.ntiles) {
        if (live) routing::route_one_token(row, t, a, o, st);
        epi_sync();
        if (o.block_counts)
          for (int e = threadIdx.x - 64; e < E; e += 128) {
            o.block_counts[tile * E + e] = st.counts[e];
            st.counts[e] = 0;
          }
        epi_sync();
      }
    }
  }

  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

template <int NE>
int pair_smem_bytes(int k_blocks) {
  return 1024 + PAIR_STAGES * A_BYTES + k_blocks * (NE / 2) * BK * 2 + BAR_BYTES + 128 * (NE + 1) * 4;
}

template <int NE>
void launch_pair(const CUtensorMap& tx, const CUtensorMap& tg, const Params& p, int num_sms, cudaStream_t s) {
  auto kernel = gate_route_tc2_kernel<NE>;
  const int smem = pair_smem_bytes<NE>(p.k_blocks);
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
  const int grid = (int)std::min<int64_t>(num_sms / 2 * 2, ceil_div(p.ntiles, 2) * 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  EMOE_CUDA(cudaLaunchKernelEx(&cfg, kernel, tx, tg, p));
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

template <int NE, int CN>
void launch_one(const CUtensorMap& tx, const CUtensorMap& tg, const Params& p, int num_sms, cudaStream_t s) {
  auto kernel = gate_route_tc_kernel<NE, CN>;
  const int smem = 1024 + STAGES * (A_BYTES + NE * BK * 2) + BAR_BYTES + 128 * (NE + 1) * 4;
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
  const int grid = (int)std::min<int64_t>(num_sms / CN * CN, ceil_div(p.ntiles, CN) * CN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CN;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  EMOE_CUDA(cudaLaunchKernelEx(&cfg, kernel, tx, tg, p));
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace gatetc

// Which form runs (EMOE_GATE_TC=pair|stream overrides for A/B runs): the
// CTA-pair form whenever the gate half fits in shared memory next to the x
// ring, else the streaming form with the gate k-blocks multicast over a
// cluster of EMOE_GATE_CLUSTER (default 2) CTAs.
static bool gate_tc_pair(int E, int d) {
  static const int force = [] {
    const char* v = getenv("EMOE_GATE_TC");
    return v ? (std::strcmp(v, "pair") == 0 ? 1 : std::strcmp(v, "stream") == 0 ? 0 : -1) : -1;
  }();
  const int k_blocks = d / gatetc::BK;
  const int smem = 1024 + gatetc::PAIR_STAGES * gatetc::A_BYTES + k_blocks * (E / 2) * gatetc::BK * 2 +
                   gatetc::BAR_BYTES + 128 * (E + 1) * 4;
  const bool fits = smem <= 227 * 1024;
  return force == 1 ? fits : (force == 0 ? false : fits);
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
  switch (a.E) {
#define EMOE_GATE_CASE(NEV)                                                    \
  case NEV:                                                                    \
    if (cn == 1)                                                               \
      gatetc::launch_one<NEV, 1>(tmap_x, tmap_gate_slice, p, num_sms, s);      \
    else if (cn == 2)                                                          \
      gatetc::launch_one<NEV, 2>(tmap_x, tmap_gate_slice, p, num_sms, s);      \
    else                                                                       \
      gatetc::launch_one<NEV, 4>(tmap_x, tmap_gate_slice, p, num_sms, s);      \
    break;
    EMOE_GATE_CASE(32)
    EMOE_GATE_CASE(64)
    EMOE_GATE_CASE(96)
    EMOE_GATE_CASE(128)
#undef EMOE_GATE_CASE
  }
}

}  // namespace emoe
