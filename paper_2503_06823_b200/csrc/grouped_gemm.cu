// K4: grouped expert FFN GEMM on 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel computes, for every resident expert
// e with rows X[off_e : off_e + n_e) of the permuted activations,
//     out[rows, n-block] = epilogue( X_rows . W_e[n-block rows]^T )
// with four epilogues:
//   EPI_SWIGLU  B tile = 128 rows of W1 + the same 128 rows of W3,
//               H = silu(X W1^T) * (X W3^T) -> bf16  (GEMM1, Mixtral / synthetic)
//   EPI_RELU    B tile = 256 rows of W1, H = relu(X W1^T) -> bf16  (GEMM1, Switch)
//   EPI_STORE   B tile = 256 rows of W2, Y = H W2^T -> bf16          (GEMM2); or
//               with the top-1 combine fused (rows scattered to y[t], scaled
//               by the token's weight), or with each row pushed into its
//               source rank's layout over peer memory (expert parallelism)
//   EPI_F32     fp32 accumulators out (the dense gate GEMM, E >= 32)
//
// Hardware mapping (B200, one CTA per SM, 6 warps), CG = CTAs per MMA:
//   CG = 1  tile 128 x 256: each CTA loads A 128x64 + B 256x64 per k-block
//           (48 KB, 4-stage ring) and issues tcgen05.mma.cta_group::1 M=128.
//   CG = 2  tile 256 x 256 on a CTA pair (cluster of 2 on one TPC): each CTA
//           loads its own 128 rows of A and half of B (128x64 + 128x64 = 32 KB,
//           6-stage ring); the leader issues tcgen05.mma.cta_group::2 M=256 that
//           reads both CTAs' shared memory and writes each CTA's 128 accumulator
//           rows to its own TMEM.  Per-SM shared-memory fill per MMA k-block drops
//           from 48 KB to 32 KB (B is split across the pair).
//   warp 0      TMA producer (128-B swizzle, L2 256-B promotion)
//   warp 1      MMA issuer (one elected lane; tcgen05.commit -> mbarriers)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> activation -> bf16
//               -> global; TMEM accumulators double-buffered (2 x 256 of 512
//               columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
// Segments are padded to the tile M (128 / 256 rows) by the permute kernel, so
// every tile row block belongs to exactly one expert and no load or store
// crosses a segment.  Tiles are walked in a grouped raster: `group_m` row
// blocks x all n blocks, sized on the host so the A panel (group_m x M x K x 2
// bytes) stays L2-resident while the weight tiles stream past it; long-K
// GEMM2s walk column panels of `group_n` weight n-blocks instead (weights
// evict-last, rows evict-first), see npanel_for().
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace emoe {
namespace gemm {

constexpr int BN = 256;  // UMMA N / accumulator columns per tile
constexpr int BK = 64;   // one 128-byte swizzle row of bf16
constexpr int MAX_EXPERTS = 256;
constexpr int TMEM_COLS = 512;
// epilogue output staging for the TMA store: one 32-row x 64-column bf16 box
// (128-B swizzled rows) per epilogue warp
constexpr int OUT_BOX_COLS = 64;
constexpr int OUT_BOX_BYTES = 32 * OUT_BOX_COLS * 2;
// mbarriers, TMEM slot, segment offsets (int32), weight slots (int16) and
// the segments' A / output row shifts (int32)
constexpr int BAR_AREA_BYTES = 4096;

// CG = CTAs per MMA (1 or 2), EW = epilogue warps (4: one per TMEM lane
// quarter; 8: two per quarter, each draining half of the accumulator columns,
// for short-K tiles whose MMAs finish faster than 4 warps can drain TMEM)
template <int CG, int EW, int MC = 1>
struct Cfg {
  static constexpr int TILE_M = 128 * CG * MC;  // rows one tile (a CTA pair's or a multicast cluster's) covers
  static constexpr int B_ROWS = BN / CG;  // B rows held by one CTA
#ifndef EMOE_CG1_STAGES
#define EMOE_CG1_STAGES 4
#endif
#ifndef EMOE_CG2_STAGES
#define EMOE_CG2_STAGES 6
#endif
  static constexpr int STAGES = CG == 1 ? EMOE_CG1_STAGES : EMOE_CG2_STAGES;
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int OUT_STAGE_BYTES = EW * OUT_BOX_BYTES;
  static constexpr int NUM_THREADS = 64 + 32 * EW;
  static constexpr int SMEM_BYTES = 1024 /*align*/ + STAGES * STAGE_BYTES + OUT_STAGE_BYTES + BAR_AREA_BYTES;
  static_assert(SMEM_BYTES <= 232448, "shared memory over the sm_100 per-block limit");
  static_assert(2 * STAGES * 8 + 4 * 8 + 16 + 4 * (MAX_EXPERTS + 1) + 2 * MAX_EXPERTS + 8 * MAX_EXPERTS <=
                    BAR_AREA_BYTES,
                "barrier area");
};

struct Params {
  const int64_t* seg_offsets;     // [E+1], multiples of TILE_M
  const int32_t* slot_of_expert;  // [E]
  int num_experts;
  int K;                // reduction length (multiple of BK)
  int n_blocks;         // output column blocks
  int out_block_cols;   // 128 (SwiGLU) or 256
  int b_rows_per_slot;  // rows of one expert in the B pool
  const int32_t* seg_expert;  // [segments] expert of each segment, null = segment i is expert i
  int group_m;          // raster group (row blocks)
  __nv_bfloat16* out;
  float* out_f32;       // EPI_F32 output
  int64_t row_limit;    // EPI_F32: rows >= row_limit not stored
  int col_limit;        // EPI_F32: columns >= col_limit not stored (multiple of 32)
  int64_t single_rows;  // > 0: one segment [0, single_rows) instead of seg_offsets
  int64_t ldo;
  int tma_store;        // bf16 epilogues: 1 = stage in smem + TMA bulk store, 0 = direct st.global
  // EPI_STORE with the top-1 combine fused (K5 for k = 1): row r's output goes
  // to scatter_out[scatter_tok[r]] scaled by scatter_w[token] (skipped when the
  // token is -1, i.e. a padding row); null = store the permuted rows
  const int32_t* scatter_tok;
  const float* scatter_w;
  __nv_bfloat16* scatter_out;
  // top-2 combine fused: pos [T][2] and per-(token, n-block, column half)
  // arrival counters; the second of a token's two rows to reach the
  // epilogue combines both (see the EPI_STORE branch)
  int scatter_k;
  const int32_t* scatter_pos;
  int32_t* scatter_arrive;
  // EPI_STORE pushing each segment's rows to its source rank's buffer
  // (expert parallelism over peer memory); null = local output
  const int32_t* seg_out_rank;
  const int64_t* seg_out_shift;
  uint8_t* out_peer[kMaxPeers];
  // L2 policies of the operand loads: the raster keeps an A panel resident
  // while the weight tiles stream past it
  uint64_t hint_a, hint_b;
  int group_n;  // column panel width in n-blocks (>= n_blocks: whole width)
  uint64_t hint_out;  // L2 policy of the TMA output stores (0: none)
  // per-segment row shifts (null = none): segment i's A rows are read from
  // row r + seg_a_shift[i] and its outputs stored to row r + seg_o_shift[i]
  // (r = the compact padded row); the NCCL expert-parallel transport reads
  // the received rows straight out of its all-to-all chunks and writes Y
  // back into the return chunks (ep.py NcclExpertParallelMoE)
  const int64_t* seg_a_shift;
  const int64_t* seg_o_shift;
};

struct TileCoord {
  int mb, nb, expert;
};

// Tile order: column panels of group_n n-blocks (group_n >= n_blocks: one
// panel) walked one after another; inside a panel, groups of group_m row
// blocks, each sweeping the panel's n-blocks with the row block fastest.
__device__ __forceinline__ TileCoord decode_tile(int t, int total_mb, int n_blocks, int group_m, int tile_m,
                                                 const int32_t* offs, int num_experts, int group_n) {
  const int ng = t / (total_mb * group_n);  // column panel
  const int n0 = ng * group_n;
  const int gn = min(group_n, n_blocks - n0);
  t -= ng * total_mb * group_n;
  const int per_group = group_m * gn;
  const int g = t / per_group;
  const int local = t - g * per_group;
  const int rows_in_group = min(group_m, total_mb - g * group_m);
  TileCoord c;
  c.nb = n0 + local / rows_in_group;
  c.mb = g * group_m + (local - (c.nb - n0) * rows_in_group);
  const int32_t row = c.mb * tile_m;
  // last segment starting at or before `row` (binary search: E = 128 made the
  // linear scan a ~2K-cycle per-tile stall of the producer warp)
  int e = 0, hi = num_experts - 1;
  while (e < hi) {
    const int mid = (e + hi + 1) >> 1;
    if (offs[mid] <= row)
      e = mid;
    else
      hi = mid - 1;
  }
  c.expert = e;
  return c;
}

// ---- TMA bulk store of the epilogue boxes ----
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* desc, const void* smem_src, int32_t c0,
                                                  int32_t c1, uint64_t hint) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "l"(hint)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* desc, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One warp's 32 rows x 64 bf16 columns (lane = row, packed[32] = its 128 B)
// to global.  TMA path: the warp's staging box (128-B rows, SWIZZLE_128B:
// 16-B chunk c of row r sits at chunk c ^ (r & 7), which also makes the
// 8-lane store phases bank-conflict free), then one bulk tensor store issued
// by lane 0.  The box is reused by the warp's next store (wait_group.read 0
// first — by then the previous chunk's TMEM loads and math have hidden it).
__device__ __forceinline__ void store_box(const Params& p, const CUtensorMap* tmap_out, uint8_t* stage_box,
                                          __nv_bfloat16* orow, const uint32_t (&packed)[32], int lane, int col,
                                          int64_t row0) {
  if (p.tma_store) {
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
    const int sw = lane & 7;
#pragma unroll
    for (int v = 0; v < 8; ++v)
      *reinterpret_cast<uint4*>(stage_box + lane * 128 + ((v ^ sw) << 4)) =
          make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      if (p.hint_out)
        tma_store_2d_hint(tmap_out, stage_box, col, (int32_t)row0, p.hint_out);
      else
        tma_store_2d(tmap_out, stage_box, col, (int32_t)row0);
      bulk_commit();
    }
  } else {
    uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
    for (int v = 0; v < 8; ++v)
      dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
  }
}

template <int EPI, int CG, int EW, int MC>
__global__ void __launch_bounds__(Cfg<CG, EW, MC>::NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const __grid_constant__ CUtensorMap tmap_b2, const __grid_constant__ CUtensorMap tmap_out,
                        Params p) {
  using C = Cfg<CG, EW, MC>;
  static_assert(MC == 1 || CG == 1, "multicast clusters pair with the 1-CTA MMA");
  constexpr bool CLUSTER = CG * MC > 1;
  constexpr uint16_t MC_MASK = (uint16_t)((1u << MC) - 1u);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::STAGES * C::A_BYTES;
  uint8_t* out_stage = smem + C::STAGES * C::STAGE_BYTES;  // 1024-B aligned
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(out_stage + C::OUT_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int32_t* s_offs = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int16_t* s_slot = reinterpret_cast<int16_t*>(s_offs + MAX_EXPERTS + 1);  // weight slot of each segment
                                                                            // (the producer's per-tile lookup)
  int32_t* s_ashift = reinterpret_cast<int32_t*>(s_slot + MAX_EXPERTS);     // [MAX_EXPERTS]
  int32_t* s_oshift = s_ashift + MAX_EXPERTS;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int E = p.num_experts;
  const uint32_t rank = CLUSTER ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const bool own_mma = MC > 1 || leader;  // CTAs that issue (and expect bytes for) their own MMAs
  const int cluster_id = blockIdx.x / (CG * MC);
  const int num_clusters = gridDim.x / (CG * MC);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    if (EPI == EPI_SWIGLU) tma_prefetch_desc(&tmap_b2);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], MC);  // MC > 1: one commit from the MMA of every cluster CTA
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], EW * CG);  // one arrival per epilogue warp of every CTA
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 1) {
      tmem_alloc(tmem_slot, TMEM_COLS);
      tmem_relinquish();
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  // set-up done: the segment table and rows come from preceding kernels
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i <= E; i += C::NUM_THREADS)
    s_offs[i] = (int32_t)(p.single_rows > 0 ? (i == 0 ? 0 : p.single_rows) : p.seg_offsets[i]);
  for (int i = threadIdx.x; i < E; i += C::NUM_THREADS)
    s_slot[i] = (int16_t)p.slot_of_expert[p.seg_expert ? p.seg_expert[i] : i];
  for (int i = threadIdx.x; i < E; i += C::NUM_THREADS) {
    s_ashift[i] = p.seg_a_shift ? (int32_t)p.seg_a_shift[i] : 0;
    s_oshift[i] = p.seg_o_shift ? (int32_t)p.seg_o_shift[i] : 0;
  }
  tc_fence_before();
  if (CLUSTER)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total_mb = s_offs[E] / C::TILE_M;
  const int total_tiles = total_mb * p.n_blocks;
  const int k_blocks = p.K / BK;

  if (warp == 0) {
    // ===================== TMA producer (every CTA) =====================
    // warp-uniform walk (as the MMA issuer), one elected lane issues the copies
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster_id; t < total_tiles; t += num_clusters) {
        const TileCoord c = decode_tile(t, total_mb, p.n_blocks, p.group_m, C::TILE_M, s_offs, E, p.group_n);
        const int slot = s_slot[c.expert];
        const int a_row = c.mb * C::TILE_M + (int)rank * 128 + s_ashift[c.expert];
        int b_row;
        const CUtensorMap* tb = &tmap_b;
        if (EPI == EPI_SWIGLU) {
          b_row = slot * p.b_rows_per_slot + c.nb * (BN / 2);
          if (CG == 2 && rank == 1) tb = &tmap_b2;  // pair: CTA0 holds the W1 half, CTA1 the W3 half
        } else {
          b_row = slot * p.b_rows_per_slot + c.nb * BN + (CG == 2 ? (int)rank * C::B_ROWS : 0);
        }
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          const int kc = kb * BK;
          uint8_t* adst = smem_a + stage * C::A_BYTES;
          uint8_t* bdst = smem_b + stage * C::B_BYTES;
          if (elect_one()) {
            if (MC > 1) {
              if (own_mma) mbar_arrive_expect_tx(&full_bar[stage], CG * C::STAGE_BYTES);
              // own A rows; this CTA's half of the weight tile to both CTAs
              // (SwiGLU: CTA0 the W1 rows, CTA1 the W3 rows; else 128 rows each)
              tma_load_2d(&tmap_a, &full_bar[stage], adst, kc, a_row, p.hint_a);
              if (EPI == EPI_SWIGLU)
                tma_load_2d_mcast(rank == 0 ? &tmap_b : &tmap_b2, &full_bar[stage], bdst + rank * (C::B_BYTES / 2), kc,
                                  b_row, MC_MASK, p.hint_b);
              else
                tma_load_2d_mcast(&tmap_b, &full_bar[stage], bdst + rank * (C::B_BYTES / MC), kc,
                                  b_row + (int)rank * (BN / MC), MC_MASK, p.hint_b);
            } else if (CG == 1) {
              mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
              tma_load_2d(&tmap_a, &full_bar[stage], adst, kc, a_row, p.hint_a);
              if (EPI == EPI_SWIGLU) {
                tma_load_2d(&tmap_b, &full_bar[stage], bdst, kc, b_row, p.hint_b);
                tma_load_2d(&tmap_b2, &full_bar[stage], bdst + C::B_BYTES / 2, kc, b_row, p.hint_b);
              } else {
                tma_load_2d(&tmap_b, &full_bar[stage], bdst, kc, b_row, p.hint_b);
              }
            } else {
              if (own_mma) mbar_arrive_expect_tx(&full_bar[stage], CG * C::STAGE_BYTES);
              tma_load_2d_pair(&tmap_a, &full_bar[stage], adst, kc, a_row, p.hint_a);
              tma_load_2d_pair(tb, &full_bar[stage], bdst, kc, b_row, p.hint_b);
            }
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (CLUSTER) {
        // producer tail: every stage released, i.e. the last multicast
        // commits to this CTA's barriers have landed before exit
        for (int i = 0; i < C::STAGES; ++i) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    // The whole warp walks the tile schedule (barrier waits and descriptors
    // stay warp-uniform, in uniform registers) and one elected lane issues
    // the MMAs and commits; from a single-lane branch every tcgen05.mma
    // needed a waterfall loop to move its operands to uniform registers.
    if (own_mma) {
      constexpr uint32_t idesc = umma_idesc_bf16(128 * CG, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = cluster_id; t < total_tiles; t += num_clusters, ++local) {
        const int buf = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[buf], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = umma_desc_sw128(smem_a + stage * C::A_BYTES);
          const uint64_t b_desc = umma_desc_sw128(smem_b + stage * C::B_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              // advance 16 bf16 = 32 B inside the 128-B swizzle row
              const uint32_t acc = (kb | kk) != 0 ? 1u : 0u;
              if (CG == 1)
                umma_bf16(tmem_d, a_desc + (uint64_t)(kk * 2), b_desc + (uint64_t)(kk * 2), idesc, acc);
              else
                umma_bf16_pair(tmem_d, a_desc + (uint64_t)(kk * 2), b_desc + (uint64_t)(kk * 2), idesc, acc);
            }
            if (MC > 1)
              umma_commit_mcast(&empty_bar[stage], MC_MASK);
            else if (CG == 1)
              umma_commit(&empty_bar[stage]);
            else
              umma_commit_pair(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if (CG == 1)
            umma_commit(&tfull_bar[buf]);
          else
            umma_commit_pair(&tfull_bar[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== epilogue (warps 2..5, every CTA) =====================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 2;
    uint8_t* my_stage = out_stage + ew * OUT_BOX_BYTES;
    // column share of this warp: all of the tile (EW = 4) or one half (EW = 8)
    constexpr int OUT_COLS = EPI == EPI_SWIGLU ? BN / 2 : BN;
    constexpr int SPAN = OUT_COLS / (EW / 4);
    const int c_lo = (ew / 4) * SPAN;
    int local = 0;
    for (int t = cluster_id; t < total_tiles; t += num_clusters, ++local) {
      const TileCoord c = decode_tile(t, total_mb, p.n_blocks, p.group_m, C::TILE_M, s_offs, E, p.group_n);
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      const int64_t row0 = (int64_t)c.mb * C::TILE_M + rank * 128 + quarter * 32;
      const int64_t row = row0 + lane;
      const int64_t orow0 = row0 + s_oshift[c.expert];  // output row of this warp's first row
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * BN;
      const int col0 = c.nb * p.out_block_cols;
      __nv_bfloat16* orow = p.out + (orow0 + lane) * p.ldo + col0;
      int combine_partner = -1, combine_slot = 0, combine_tok = -1;  // fused top-2 combine, after the TMEM release
      float combine_w0 = 0.0f, combine_w1 = 0.0f;
      if (EPI == EPI_SWIGLU) {
#pragma unroll 1
        for (int cc = c_lo; cc < c_lo + SPAN; cc += OUT_BOX_COLS) {
          uint32_t g0[32], g1[32], u0[32], u1[32];
          tmem_ld_32x32b_x32(taddr + cc, g0);
          tmem_ld_32x32b_x32(taddr + cc + 32, g1);
          tmem_ld_32x32b_x32(taddr + BN / 2 + cc, u0);
          tmem_ld_32x32b_x32(taddr + BN / 2 + cc + 32, u1);
          tmem_ld_wait();
          uint32_t packed[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const bool hi = j >= 16;
            const int q = 2 * (j & 15);
            const float ga = __uint_as_float(hi ? g1[q] : g0[q]), gb = __uint_as_float(hi ? g1[q + 1] : g0[q + 1]);
            const float ua = __uint_as_float(hi ? u1[q] : u0[q]), ub = __uint_as_float(hi ? u1[q + 1] : u0[q + 1]);
            const float h0 = ga / (1.0f + __expf(-ga)) * ua;
            const float h1 = gb / (1.0f + __expf(-gb)) * ub;
            packed[j] = pack_bf16x2(h0, h1);
          }
          store_box(p, &tmap_out, my_stage, orow + cc, packed, lane, col0 + cc, orow0);
        }
      } else if (EPI == EPI_F32) {
        // fp32 accumulators straight out (dense gate GEMM): rows >= row_limit
        // and columns >= col_limit are not stored
        float* frow = p.out_f32 + row * p.ldo;
        const bool row_ok = row < p.row_limit;
#pragma unroll 1
        for (int cc = c_lo; cc < c_lo + SPAN; cc += 32) {
          uint32_t a[32];
          tmem_ld_32x32b_x32(taddr + cc, a);
          tmem_ld_wait();
          if (row_ok && cc < p.col_limit) {
            uint4* dst = reinterpret_cast<uint4*>(frow + cc);
#pragma unroll
            for (int v = 0; v < 8; ++v) dst[v] = make_uint4(a[4 * v], a[4 * v + 1], a[4 * v + 2], a[4 * v + 3]);
          }
        }
      } else if (EPI == EPI_STORE && p.seg_out_rank != nullptr) {
        // expert parallelism: the tile's rows belong to one (source, expert)
        // segment; write them into the source rank's permuted layout over
        // NVLink (each lane's 128-B row chunk, posted stores)
        __nv_bfloat16* prow = reinterpret_cast<__nv_bfloat16*>(p.out_peer[p.seg_out_rank[c.expert]]) +
                              (row + p.seg_out_shift[c.expert]) * p.ldo + col0;
#pragma unroll 1
        for (int cc = c_lo; cc < c_lo + SPAN; cc += OUT_BOX_COLS) {
          uint32_t a0[32], a1[32];
          tmem_ld_32x32b_x32(taddr + cc, a0);
          tmem_ld_32x32b_x32(taddr + cc + 32, a1);
          tmem_ld_wait();
          uint4* dst = reinterpret_cast<uint4*>(prow + cc);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            uint32_t q4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = 4 * v + u, q = 2 * (j & 15);
              q4[u] = pack_bf16x2(__uint_as_float(j < 16 ? a0[q] : a1[q]), __uint_as_float(j < 16 ? a0[q + 1] : a1[q + 1]));
            }
            dst[v] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
          }
        }
      } else if (EPI == EPI_STORE && p.scatter_tok != nullptr && p.scatter_k == 2) {
        // top-2 combine fused: y[t] = bf16(fma(w1, Y1, fma(w0, Y0, 0))) with
        // Y_j = bf16(row of slot j) -- the separate combine's operations in
        // its slot order, so bit-identical.  The two rows of a token sit in
        // different experts' tiles.  Each stores its bf16 row chunk into
        // Y_perm, then (after the TMEM buffer is released) arrives on the
        // token's (n-block, column half) counter with one acq_rel atomic:
        // the second to arrive finds the partner's chunk complete and
        // visible, combines both from L2 into y[t] and re-zeroes the counter.
        // Nobody waits, so no lane can stall a warp-collective TMEM load.
        // Single-served tokens write y[t] directly from the accumulators.
        const int tok = p.scatter_tok[row];
        int partner = -1, slot = 0;
        float w0 = 0.0f, w1 = 0.0f;
        if (tok >= 0) {
          const int p0 = p.scatter_pos[2 * tok], p1 = p.scatter_pos[2 * tok + 1];
          slot = p0 == (int)row ? 0 : 1;
          partner = slot == 0 ? p1 : p0;
          w0 = p.scatter_w[2 * tok];
          w1 = p.scatter_w[2 * tok + 1];
        }
        __nv_bfloat16* yrow = p.scatter_out + (int64_t)(tok < 0 ? 0 : tok) * p.ldo + col0;
        __nv_bfloat16* own = p.out + row * p.ldo + col0;
#pragma unroll 1
        for (int cc = c_lo; cc < c_lo + SPAN; cc += OUT_BOX_COLS) {
          uint32_t a0[32], a1[32];
          tmem_ld_32x32b_x32(taddr + cc, a0);
          tmem_ld_32x32b_x32(taddr + cc + 32, a1);
          tmem_ld_wait();
          if (tok < 0) continue;
          uint32_t mine[32];
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int q = 2 * (jj & 15);
            mine[jj] = pack_bf16x2(__uint_as_float(jj < 16 ? a0[q] : a1[q]),
                                   __uint_as_float(jj < 16 ? a0[q + 1] : a1[q + 1]));
          }
          uint4* dst = reinterpret_cast<uint4*>((partner >= 0 ? own : yrow) + cc);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            if (partner >= 0) {
              dst[v] = make_uint4(mine[4 * v], mine[4 * v + 1], mine[4 * v + 2], mine[4 * v + 3]);
            } else {
              uint32_t q4[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint32_t y0 = mine[4 * v + u];
                q4[u] = pack_bf16x2(fmaf(w0, bf16_lo(y0), 0.0f), fmaf(w0, bf16_hi(y0), 0.0f));
              }
              dst[v] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
            }
          }
        }
        combine_partner = partner;
        combine_slot = slot;
        combine_tok = tok;
        combine_w0 = w0;
        combine_w1 = w1;
      } else if (EPI == EPI_STORE && p.scatter_tok != nullptr) {
        // top-1 combine fused: y[t] = w_t * bf16(Y_row), the same two roundings
        // as the separate combine (bit-identical), each lane's 128-B row
        // chunk stored straight into its token's row
        const int tok = p.scatter_tok[row];
        const float w = tok >= 0 ? p.scatter_w[tok] : 0.0f;
        __nv_bfloat16* yrow = p.scatter_out + (int64_t)(tok < 0 ? 0 : tok) * p.ldo + col0;
#pragma unroll 1
        for (int cc = c_lo; cc < c_lo + SPAN; cc += OUT_BOX_COLS) {
          uint32_t a0[32], a1[32];
          tmem_ld_32x32b_x32(taddr + cc, a0);
          tmem_ld_32x32b_x32(taddr + cc + 32, a1);
          tmem_ld_wait();
          if (tok >= 0) {
            uint4* dst = reinterpret_cast<uint4*>(yrow + cc);
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              uint32_t q4[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = 4 * v + u, q = 2 * (j & 15);
                const uint32_t y2 = pack_bf16x2(__uint_as_float(j < 16 ? a0[q] : a1[q]),
                                                __uint_as_float(j < 16 ? a0[q + 1] : a1[q + 1]));
                q4[u] = pack_bf16x2(w * bf16_lo(y2), w * bf16_hi(y2));
              }
              dst[v] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
            }
          }
        }
      } else {
#pragma unroll 1
        for (int cc = c_lo; cc < c_lo + SPAN; cc += OUT_BOX_COLS) {
          uint32_t a0[32], a1[32];
          tmem_ld_32x32b_x32(taddr + cc, a0);
          tmem_ld_32x32b_x32(taddr + cc + 32, a1);
          tmem_ld_wait();
          uint32_t packed[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int q = 2 * (j & 15);
            float v0 = __uint_as_float(j < 16 ? a0[q] : a1[q]), v1 = __uint_as_float(j < 16 ? a0[q + 1] : a1[q + 1]);
            if (EPI == EPI_RELU) {
              v0 = fmaxf(v0, 0.0f);
              v1 = fmaxf(v1, 0.0f);
            }
            packed[j] = pack_bf16x2(v0, v1);
          }
          store_box(p, &tmap_out, my_stage, orow + cc, packed, lane, col0 + cc, orow0);
        }
      }
      tc_fence_before();
      if (lane == 0) {
        if (CG == 1)
          mbar_arrive_relaxed(&tempty_bar[buf]);
        else
          mbar_arrive_leader_relaxed(&tempty_bar[buf]);
      }
      if (EPI == EPI_STORE && combine_partner >= 0) {
        // second of the token's rows to arrive: both bf16 rows are in Y_perm
        int32_t* arrive = p.scatter_arrive + ((int64_t)combine_tok * p.n_blocks + c.nb) * 2 + ew / 4;
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(arrive) : "memory");
        if (old != 0) {
          *arrive = 0;  // nobody else touches it this forward; the kernel boundary orders the next use
          const __nv_bfloat16* r0 = p.out + (int64_t)(combine_slot == 0 ? row : combine_partner) * p.ldo + col0;
          const __nv_bfloat16* r1 = p.out + (int64_t)(combine_slot == 0 ? combine_partner : row) * p.ldo + col0;
          __nv_bfloat16* yrow = p.scatter_out + (int64_t)combine_tok * p.ldo + col0;
#pragma unroll 1
          for (int cc = c_lo; cc < c_lo + SPAN; cc += 8) {
            const uint4 u0 = __ldcg(reinterpret_cast<const uint4*>(r0 + cc));
            const uint4 u1 = __ldcg(reinterpret_cast<const uint4*>(r1 + cc));
            const uint32_t y0[4] = {u0.x, u0.y, u0.z, u0.w}, y1[4] = {u1.x, u1.y, u1.z, u1.w};
            uint32_t q4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float lo = fmaf(combine_w1, bf16_lo(y1[u]), fmaf(combine_w0, bf16_lo(y0[u]), 0.0f));
              const float hi = fmaf(combine_w1, bf16_hi(y1[u]), fmaf(combine_w0, bf16_hi(y0[u]), 0.0f));
              q4[u] = pack_bf16x2(lo, hi);
            }
            *reinterpret_cast<uint4*>(yrow + cc) = make_uint4(q4[0], q4[1], q4[2], q4[3]);
          }
        }
      }
    }
    if (EPI != EPI_F32 && p.tma_store && lane == 0) bulk_wait_all();
    if (EPI == EPI_STORE && p.seg_out_rank != nullptr) __threadfence_system();  // pushes visible to the peers
  }

  if (CLUSTER)
    cluster_sync_all();  // the cluster's commits to our barriers and TMEM are done
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 1)
      tmem_dealloc(tmem_base, TMEM_COLS);
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
  }
}

}  // namespace gemm

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    EMOE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled not available");
    fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

// 2-D bf16 tensor [rows][cols] (row-major), box = box_rows x 64 columns, 128-B swizzle
CUtensorMap make_tmap_bf16_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// 2-D bf16 output [rows][cols] as the epilogue's TMA store target: 32 rows x 64 columns, 128-B swizzle
CUtensorMap make_tmap_bf16_store(const void* base, uint64_t rows, uint64_t cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {gemm::OUT_BOX_COLS, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (store) failed: " + std::to_string((int)r));
  return m;
}

static bool tma_store_enabled() {
  static const bool on = [] {
    const char* v = getenv("EMOE_GEMM_TMA_STORE");
    return !(v && v[0] == '0');
  }();
  return on;
}

int gemm_tile_m(int cta_group, int mc) { return 128 * cta_group * mc; }
int gemm_b_box_rows(int epi, int cta_group, int mc) { return epi == EPI_SWIGLU ? 128 : 256 / (cta_group * mc); }

// raster group: keep the A panel (group x tile_m rows x K) near `panel` MB of
// L2: 24 MB for long reductions (Mixtral shape, K >= 2048: best of
// 2/8/24/48/96 MB), 4 MB for short ones (Switch GEMM1, K = 768: 4-8 MB beat
// 24 MB by 4 %, profiles/r01_raster_sweep.jsonl).  EMOE_GEMM_PANEL_MB
// overrides for tuning.
// L2 policies for the operand loads (EMOE_GEMM_L2_HINTS): 0 = evict-normal
// for both; 1 = A panel evict-last, weight tiles evict-first (measured 3x the
// DRAM traffic: a weight tile is shared by the group's row blocks, which do
// not run in lockstep); 2 = A panel evict-last, weights normal
static void l2_hints(uint64_t& a, uint64_t& b) {
  static const int mode = [] {
    const char* v = getenv("EMOE_GEMM_L2_HINTS");
    return v ? atoi(v) : 0;
  }();
  a = mode == 1 || mode == 2 ? kCacheEvictLast : kCacheEvictNormal;
  b = mode == 1 ? kCacheEvictFirst : kCacheEvictNormal;
}

// Column-panel raster: the weight panel (npanel n-blocks) stays L2-resident
// (evict-last) while every row block streams past it once per panel
// (evict-first; a row block's npanel tiles run concurrently), group_m = 1.
// Default: GEMM2 with K >= 8192 (Mixtral shape: K = 14336, each 128 x 256
// tile touches 11 MB of operands, so the row-panel raster's concurrent tiles
// outgrow L2 and W2 is re-streamed per row group) uses 8-block panels:
// DRAM reads 13.2 -> 9.4 GB, +37 MHz at the power cap, +1.8 % tokens/s
// (profiles/r01_gemm_npanel_ab.jsonl); GEMM1 panels raise its traffic.
// EMOE_GEMM1_NPANEL / EMOE_GEMM2_NPANEL override (0 = off).
static int npanel_for(int epi, int K) {
  static const int g1 = [] {
    const char* v = getenv("EMOE_GEMM1_NPANEL");
    return v ? atoi(v) : -1;
  }();
  static const int g2 = [] {
    const char* v = getenv("EMOE_GEMM2_NPANEL");
    return v ? atoi(v) : -1;
  }();
  if (epi == EPI_STORE) return g2 >= 0 ? g2 : (K >= 8192 ? 8 : 0);
  if (epi == EPI_SWIGLU || epi == EPI_RELU) return g1 >= 0 ? g1 : 0;
  return 0;
}

static int group_rows(int K, int tile_m) {
  static int panel_env = [] {
    const char* v = getenv("EMOE_GEMM_PANEL_MB");
    return v ? atoi(v) : 0;
  }();
  const int panel_mb = panel_env > 0 ? panel_env : (K >= 2048 ? 24 : 4);
  static int forced = [] {  // EMOE_GEMM_GROUP_M: exact raster group (row blocks), for A/B runs
    const char* v = getenv("EMOE_GEMM_GROUP_M");
    return v ? atoi(v) : 0;
  }();
  if (forced > 0) return forced;
  const int64_t panel_row_bytes = (int64_t)tile_m * K * 2;
  int g = (int)(((int64_t)panel_mb << 20) / panel_row_bytes);
  return g < 2 ? 2 : (g > 64 ? 64 : g);
}

static void launch_params(int epi, int cta_group, int mc, const CUtensorMap& ta, const CUtensorMap& tb,
                          const CUtensorMap& tb2, const CUtensorMap& to, const gemm::Params& p, int num_sms,
                          cudaStream_t stream);

void launch_grouped_gemm(int epi, int cta_group, int mc, const CUtensorMap& ta, const CUtensorMap& tb,
                         const CUtensorMap& tb2, const int64_t* seg_offsets, const int32_t* slot_of_expert,
                         int num_experts, int K, int N_out, int b_rows_per_slot, __nv_bfloat16* out, int64_t ldo,
                         int num_sms, cudaStream_t stream, const int32_t* seg_expert, const CUtensorMap* tmap_out,
                         const ScatterCombine* scatter, const PeerOut* peer_out, const int64_t* seg_a_shift,
                         const int64_t* seg_o_shift) {
  EMOE_REQUIRE(num_experts <= gemm::MAX_EXPERTS, "grouped_gemm: too many segments");
  EMOE_REQUIRE(!scatter || epi == EPI_STORE, "grouped_gemm: the fused combine needs the GEMM2 epilogue");
  EMOE_REQUIRE(K % gemm::BK == 0, "grouped_gemm: K must be a multiple of 64");
  EMOE_REQUIRE(cta_group == 1 || cta_group == 2, "grouped_gemm: cta_group must be 1 or 2");
  EMOE_REQUIRE(mc == 1 || (mc == 2 && cta_group == 1 && epi != EPI_F32),
               "grouped_gemm: weight multicast pairs (mc = 2) run with cta_group 1");
  gemm::Params p;
  p.seg_offsets = seg_offsets;
  p.slot_of_expert = slot_of_expert;
  p.seg_expert = seg_expert;
  p.num_experts = num_experts;
  p.K = K;
  p.out_block_cols = epi == EPI_SWIGLU ? gemm::BN / 2 : gemm::BN;
  EMOE_REQUIRE(N_out % p.out_block_cols == 0, "grouped_gemm: N must be a multiple of the column block");
  p.n_blocks = N_out / p.out_block_cols;
  p.b_rows_per_slot = b_rows_per_slot;
  p.group_m = group_rows(K, 128 * cta_group * mc);
  l2_hints(p.hint_a, p.hint_b);
  p.group_n = p.n_blocks;
  {  // EMOE_GEMM_STORE_HINT: 0 none (default), 1 evict-first, 2 evict-last (A/B runs)
    static const int sh = [] {
      const char* v = getenv("EMOE_GEMM_STORE_HINT");
      return v ? atoi(v) : 0;
    }();
    p.hint_out = sh == 1 ? kCacheEvictFirst : (sh == 2 ? kCacheEvictLast : 0);
  }
  if (const int np = npanel_for(epi, K); np > 0 && np < p.n_blocks) {
    static const bool a_first = [] {  // EMOE_GEMM_PANEL_A_NORMAL=1: row blocks evict-normal (A/B runs)
      const char* v = getenv("EMOE_GEMM_PANEL_A_NORMAL");
      return !(v && v[0] == '1');
    }();
    p.group_n = np;
    p.group_m = 1;
    p.hint_a = a_first ? kCacheEvictFirst : kCacheEvictNormal;
    p.hint_b = kCacheEvictLast;
  }
  p.out = out;
  p.ldo = ldo;
  p.out_f32 = nullptr;
  p.row_limit = 0;
  p.col_limit = 0;
  p.single_rows = 0;
  EMOE_REQUIRE(!peer_out || epi == EPI_STORE, "grouped_gemm: peer output needs the GEMM2 epilogue");
  p.tma_store = tmap_out != nullptr && tma_store_enabled() && !scatter && !peer_out;
  p.seg_out_rank = peer_out ? peer_out->seg_rank : nullptr;
  p.seg_out_shift = peer_out ? peer_out->seg_shift : nullptr;
  p.seg_a_shift = seg_a_shift;
  p.seg_o_shift = seg_o_shift;
  for (int q = 0; q < kMaxPeers; ++q) p.out_peer[q] = peer_out ? peer_out->base[q] : nullptr;
  p.scatter_tok = scatter ? scatter->row_token : nullptr;
  p.scatter_w = scatter ? scatter->weight : nullptr;
  p.scatter_out = scatter ? scatter->y : nullptr;
  p.scatter_k = scatter ? scatter->k : 1;
  p.scatter_pos = scatter ? scatter->pos : nullptr;
  p.scatter_arrive = scatter ? scatter->arrive : nullptr;
  EMOE_REQUIRE(!scatter || scatter->k == 1 || (scatter->k == 2 && scatter->pos && scatter->arrive),
               "grouped_gemm: the fused top-2 combine needs positions and arrival counters");
  launch_params(epi, cta_group, mc, ta, tb, tb2, p.tma_store ? *tmap_out : ta, p, num_sms, stream);
}

__device__ int32_t g_slot_zero = 0;

void launch_dense_gemm_f32(const CUtensorMap& ta, const CUtensorMap& tb, int64_t M, int K, int N_out, float* out,
                           int64_t ldo, int col_limit, int num_sms, cudaStream_t stream, int cta_group) {
  EMOE_REQUIRE(K % gemm::BK == 0, "dense_gemm: K must be a multiple of 64");
  EMOE_REQUIRE(N_out % gemm::BN == 0, "dense_gemm: N must be a multiple of 256");
  gemm::Params p;
  void* zero = nullptr;
  EMOE_CUDA(cudaGetSymbolAddress(&zero, g_slot_zero));
  p.seg_offsets = nullptr;
  p.slot_of_expert = static_cast<const int32_t*>(zero);
  p.seg_expert = nullptr;
  p.num_experts = 1;
  p.K = K;
  p.out_block_cols = gemm::BN;
  p.n_blocks = N_out / gemm::BN;
  p.b_rows_per_slot = 0;
  p.group_m = group_rows(K, 128 * cta_group);
  p.group_n = p.n_blocks;
  p.hint_out = 0;
  p.hint_a = kCacheEvictNormal;
  p.hint_b = kCacheEvictNormal;
  p.out = nullptr;
  p.ldo = ldo;
  p.out_f32 = out;
  p.row_limit = M;
  p.col_limit = col_limit;
  p.single_rows = ceil_div(M, 128 * cta_group) * (128 * cta_group);
  p.tma_store = 0;
  p.scatter_tok = nullptr;
  p.scatter_w = nullptr;
  p.scatter_out = nullptr;
  p.scatter_k = 1;
  p.scatter_pos = nullptr;
  p.scatter_arrive = nullptr;
  p.seg_out_rank = nullptr;
  p.seg_out_shift = nullptr;
  p.seg_a_shift = nullptr;
  p.seg_o_shift = nullptr;
  launch_params(EPI_F32, cta_group, 1, ta, tb, tb, ta, p, num_sms, stream);
}

template <int EPI, int CG, int EW, int MC>
static void launch_one(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2, const CUtensorMap& to,
                       const gemm::Params& p, int num_sms, cudaStream_t stream) {
  using C = gemm::Cfg<CG, EW, MC>;
  auto kernel = gemm::grouped_gemm_kernel<EPI, CG, EW, MC>;
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(kernel), C::SMEM_BYTES);
  constexpr int CS = CG * MC;  // CTAs per cluster
  const int grid = (num_sms / CS) * CS;
  EMOE_CUDA(launch_pdl(kernel, dim3(grid), dim3(C::NUM_THREADS), (size_t)C::SMEM_BYTES, stream, CS, ta, tb, tb2, to, p));

  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

template <int EPI, int CG>
static void launch_ew(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2, const CUtensorMap& to,
                      const gemm::Params& p, int num_sms, cudaStream_t stream) {
  // 4 epilogue warps (one per TMEM lane quarter); 8 (two per quarter, each
  // draining half the columns) measured 1-2 % slower for the short-K Switch
  // GEMM1 and was dropped (profiles/r01_epilogue_warps_ab.jsonl)
  launch_one<EPI, CG, 4, 1>(ta, tb, tb2, to, p, num_sms, stream);
}

static void launch_params(int epi, int cta_group, int mc, const CUtensorMap& ta, const CUtensorMap& tb,
                          const CUtensorMap& tb2, const CUtensorMap& to, const gemm::Params& p, int num_sms,
                          cudaStream_t stream) {
  if (mc == 2) {  // 1-CTA MMAs, weight tile multicast over a cluster of 2 (4 epilogue warps)
    if (epi == EPI_SWIGLU)
      launch_one<EPI_SWIGLU, 1, 4, 2>(ta, tb, tb2, to, p, num_sms, stream);
    else if (epi == EPI_RELU)
      launch_one<EPI_RELU, 1, 4, 2>(ta, tb, tb2, to, p, num_sms, stream);
    else
      launch_one<EPI_STORE, 1, 4, 2>(ta, tb, tb2, to, p, num_sms, stream);
  } else if (cta_group == 1) {
    if (epi == EPI_SWIGLU)
      launch_ew<EPI_SWIGLU, 1>(ta, tb, tb2, to, p, num_sms, stream);
    else if (epi == EPI_RELU)
      launch_ew<EPI_RELU, 1>(ta, tb, tb2, to, p, num_sms, stream);
    else if (epi == EPI_F32)
      launch_ew<EPI_F32, 1>(ta, tb, tb2, to, p, num_sms, stream);
    else
      launch_ew<EPI_STORE, 1>(ta, tb, tb2, to, p, num_sms, stream);
  } else {
    if (epi == EPI_SWIGLU)
      launch_ew<EPI_SWIGLU, 2>(ta, tb, tb2, to, p, num_sms, stream);
    else if (epi == EPI_RELU)
      launch_ew<EPI_RELU, 2>(ta, tb, tb2, to, p, num_sms, stream);
    else if (epi == EPI_F32)
      launch_ew<EPI_F32, 2>(ta, tb, tb2, to, p, num_sms, stream);
    else
      launch_ew<EPI_STORE, 2>(ta, tb, tb2, to, p, num_sms, stream);
  }
}

}  // namespace emoe
