// K4, fp32 configuration (BASELINE config 1: fp32 weights and activations,
// outputs within 1e-5 of the fp32 reference) on the 5th-generation tensor
// cores: 3xTF32.
//
// Each fp32 operand is split into hi = tf32(x) (round to nearest, 11
// significant bits) and lo = x - hi (exact in fp32), and
//     a . b  ~=  a_hi b_hi + a_hi b_lo + a_lo b_hi
// accumulated in fp32 TMEM by tcgen05.mma.kind::tf32.  The dropped a_lo b_lo
// term and the tensor core's TF32 view of the lo parts each cost <= 2^-21 of
// |a b|, so a 1024-3584-long dot product stays ~1e-6 relative: fp32 accuracy
// at tensor-core rate (the SIMT FFMA kernel, grouped_gemm_f32.cu, ran at 36 %
// of the fp32 pipe).
//
// Operands are pre-split in HBM: the expert slot pools hold hi in place and lo
// in a twin pool (split once per H2D load), the permuted activations are split
// after the permute, and GEMM1's epilogue writes H as hi/lo for GEMM2.
//
// Tile 128 x 128, one CTA per SM (persistent), warp-specialised like the bf16
// kernel (grouped_gemm.cu): warp 0 TMA producer, warp 1 single-thread MMA
// issuer, warps 2-5 epilogue; 3-stage ring of {A_hi, A_lo, B_hi, B_lo} (64 KB
// per stage: 32 fp32 = one 128-B swizzle row of K per k-block).  The tensor
// core's accumulator rounding is biased (toward zero), which over K = 3584
// costs ~5e-5 relative; so each tile accumulates K in chunks of 128 into four
// rotating 128-column TMEM slots and the epilogue warps sum the chunks in
// fp32 registers (round to nearest), ~2e-6 relative.  SwiGLU: the B tile is 64
// rows of W1 and the same 64 rows of W3, so a tile yields 64 columns of H.
// Schedule: whole tiles round-robin, or stream-K (the tiles' k-blocks split
// evenly over the co-resident CTAs; a tile split between CTAs is finished by
// the CTA holding its first k-blocks, which adds the others' raw partials in
// k order) where the tile count leaves a wave mostly empty (config 1's GEMM2).
// Variants measured and dropped (CTA-pair 256 x 256 tiles, the split done in
// shared memory from raw fp32 operands): profiles/r02_tf32_variants_ab.txt.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace emoe {
namespace tf32x3 {

constexpr int BM = 128, BN = 128;  // per CTA: 128 rows (TMEM lanes) x 128 accumulator columns
constexpr int BK = 32;  // fp32 elements per 128-B swizzle row
constexpr int TILE_BYTES = 128 * 128;  // 128 rows x 128 B
constexpr int NUM_THREADS = 192;
constexpr int SLOTS = 4;     // rotating TMEM accumulator slots (4 x 128 columns)
constexpr int CHUNK_KB = 4;  // k-blocks (128 of K) per accumulator chunk
constexpr int TMEM_COLS = SLOTS * BN;
constexpr int MAX_SEGS = 256;
// CG = 1: one CTA per 128 x 128 tile, stage {A_hi, A_lo, B_hi, B_lo} = 64 KB, 3 stages.
// CG = 2: a CTA pair per 256 x 128 tile (tcgen05 cta_group::2, M = 256): each
// CTA holds its 128 A rows and half of the 128 B rows, stage = 48 KB, 4 stages
// -- a quarter fewer bytes per MAC and a deeper ring in the same shared memory.
template <int CG>
struct TCfg {
  static constexpr int B_ROWS = BN / CG;  // B rows this CTA loads per stage
  static constexpr int B_BYTES = B_ROWS * 128;
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = CG == 1 ? 3 : 4;
  static constexpr int TILE_M = BM * CG;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 4096;
  static_assert(2 * STAGES * 8 + 2 * SLOTS * 8 + 16 + 4 * (2 * MAX_SEGS + 1) <= 4096, "barrier / table area");
};

struct Params {
  const int64_t* seg_offsets;     // [n_seg + 1], multiples of 128
  const int32_t* slot_of_expert;  // [E]
  const int32_t* seg_expert;      // [n_seg] or null (segment i = expert i)
  int n_seg;
  int K;
  int n_blocks;
  int out_block_cols;  // 64 (SwiGLU) or 128
  int b_rows_per_slot;
  int group_m;
  float* out_hi;  // GEMM1: tf32(H); GEMM2: Y
  float* out_lo;  // GEMM1: H - tf32(H); GEMM2: null
  int64_t ldo;
  // stream-K: the tiles' k-blocks are divided evenly over the co-resident
  // CTAs; a tile split between CTAs is finished by the one that computed its
  // first k-blocks (see the epilogue)
  float* partial;   // [CTAs][32 float4 columns][128 rows] float4: one raw partial tile per CTA
  int32_t* arrive;  // [tiles] helper arrivals, zero between launches (the owner re-zeroes)
  int dp;           // 1: whole tiles round-robin (data-parallel), no split tiles
  int chunk_kb;     // k-blocks per TMEM accumulator chunk (CHUNK_KB; EMOE_TF32_CHUNK for A/B runs)
};

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, 1 CTA or a CTA pair
template <int CG>
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// A/B = TF32 (format 2), D = f32, both K-major
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// x rounded to 10 explicit mantissa bits (nearest, ties to even) with the low
// 13 bits exactly zero, so x - round_tf32(x) is the exact remainder (cvt.rna.tf32
// leaves the low bits unspecified).  Finite inputs only (weights/activations).
using emoe::round_tf32;

__device__ __forceinline__ void decode(int t, int total_mb, int n_blocks, int group_m, const int32_t* offs, int n_seg,
                                       int tile_m, int& mb, int& nb, int& seg) {
  const int per_group = group_m * n_blocks;
  const int g = t / per_group;
  const int local = t - g * per_group;
  const int rows_in_group = min(group_m, total_mb - g * group_m);
  nb = local / rows_in_group;
  mb = g * group_m + (local - nb * rows_in_group);
  const int row = mb * tile_m;
  // last segment starting at or before `row` (binary search: E = 128 made the
  // linear scan a ~2K-cycle per-tile stall of the producer warp)
  int e = 0, hi = n_seg - 1;
  while (e < hi) {
    const int mid = (e + hi + 1) >> 1;
    if (offs[mid] <= row)
      e = mid;
    else
      hi = mid - 1;
  }
  seg = e;
}

// stream-K work division: worker q of P takes units [q U / P, (q + 1) U / P)
__device__ __forceinline__ int64_t range_start(int q, int P, int64_t U) { return (int64_t)q * U / P; }

// the worker whose range holds unit u
__device__ __forceinline__ int worker_of(int64_t u, int P, int64_t U) {
  int q = (int)(u * P / U);
  while (q + 1 < P && range_start(q + 1, P, U) <= u) ++q;
  while (q > 0 && range_start(q, P, U) > u) --q;
  return q;
}

// one segment of a worker's range: k-blocks [kb0, kb1) of tile t
struct Segment {
  int t, kb0, kb1;
};
__device__ __forceinline__ Segment next_segment(int64_t& u, int64_t u_end, int KB) {
  Segment g;
  g.t = (int)(u / KB);
  g.kb0 = (int)(u - (int64_t)g.t * KB);
  g.kb1 = (u_end - u) < (int64_t)(KB - g.kb0) ? g.kb0 + (int)(u_end - u) : KB;
  u += g.kb1 - g.kb0;
  return g;
}

// the segments one worker processes: its stream-K range, or (dp) whole tiles
// me, me + P, ... (data-parallel)
struct Work {
  int64_t u, u_end;
  int KB, t, step, tiles, dp;
  __device__ bool next(Segment& g) {
    if (dp) {
      if (t >= tiles) return false;
      g.t = t;
      g.kb0 = 0;
      g.kb1 = KB;
      t += step;
      return true;
    }
    if (u >= u_end) return false;
    g = next_segment(u, u_end, KB);
    return true;
  }
};

// Owner side of a split tile: wait (one lane per warp, bounded) until
// `helpers` helpers have counted in on *cnt.
__device__ __forceinline__ void wait_helpers(const int32_t* cnt, int helpers, int lane) {
  if (lane == 0) {
    uint32_t spins = 0;
    int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
      if (v >= helpers) break;
      __nanosleep(64);
      if (++spins == (1u << 28)) __trap();  // a lost helper: fail loudly, never hang
    }
  }
  __syncwarp();
}

template <int EPI, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                       const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                       const __grid_constant__ CUtensorMap tb2_hi, const __grid_constant__ CUtensorMap tb2_lo,
                       Params p) {
  using C = TCfg<CG>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [SLOTS]
  uint64_t* tempty_bar = tfull_bar + SLOTS;  // [SLOTS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + SLOTS);
  int32_t* s_offs = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_slot = s_offs + MAX_SEGS + 1;  // weight slot per segment: no dependent global loads per tile

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int S = p.n_seg;
  // CTA pair: rank 0 (the leader) issues the M = 256 MMAs for both CTAs; the
  // pair walks one work list (worker = pair) and each CTA owns its 128 rows
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&ta_hi);
    tma_prefetch_desc(&ta_lo);
    tma_prefetch_desc(&tb_hi);
    tma_prefetch_desc(&tb_lo);
    if (EPI == EPI_SWIGLU) {
      tma_prefetch_desc(&tb2_hi);
      tma_prefetch_desc(&tb2_lo);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < SLOTS; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4 * CG);  // every epilogue warp of every CTA (the leader's copy counts)
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
  pdl_wait();  // set-up done: the segment table and rows come from preceding kernels
  pdl_trigger();
  for (int i = threadIdx.x; i <= S; i += NUM_THREADS) s_offs[i] = (int32_t)p.seg_offsets[i];
  for (int i = threadIdx.x; i < S; i += NUM_THREADS) s_slot[i] = p.slot_of_expert[p.seg_expert ? p.seg_expert[i] : i];
  tc_fence_before();
  if (CG == 2)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_mb = s_offs[S] / C::TILE_M;
  const int total_tiles = total_mb * p.n_blocks;
  const int KB = p.K / BK;
  const int64_t U = (int64_t)total_tiles * KB;
  const int workers = (int)gridDim.x / CG;
  // at most one worker per k-block, so every working worker's range is non-empty
  // (an owner's helpers are then exactly the workers after it up to the tile's end)
  const int P = (int)(U < (int64_t)workers ? U : (int64_t)workers);
  const int me = (int)blockIdx.x / CG;
  const int64_t u_begin = me < P ? range_start(me, P, U) : U;
  const int64_t u_end = me < P ? range_start(me + 1, P, U) : U;
  const Work work0{u_begin, u_end, KB, me, workers, total_tiles, p.dp};

  if (warp == 0) {
    {  // ===== TMA producer (every CTA: its A rows and its half of the B rows; warp-uniform, one lane issues)
      int stage = 0;
      uint32_t phase = 0;
      Work w = work0;
      Segment g;
      while (w.next(g)) {
        int mb, nb, seg;
        decode(g.t, total_mb, p.n_blocks, p.group_m, s_offs, S, C::TILE_M, mb, nb, seg);
        const int slot = s_slot[seg];
        const int a_row = mb * C::TILE_M + (int)rank * BM;
        // SwiGLU: B rows 0-63 = W1, 64-127 = W3 of the same 64 output columns
        // (pair: CTA 0 the W1 half, CTA 1 the W3 half); else 128 rows (pair: 64 each)
        const int b_row = EPI == EPI_SWIGLU ? slot * p.b_rows_per_slot + nb * (BN / 2)
                                            : slot * p.b_rows_per_slot + nb * BN + (int)rank * C::B_ROWS;
        for (int kb = g.kb0; kb < g.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::STAGE_BYTES;
          uint8_t* bh = st + 2 * TILE_BYTES;
          uint8_t* bl = bh + C::B_BYTES;
          const int kc = kb * BK;
          if (elect_one()) {
            if (CG == 1) {
              mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
              tma_load_2d(&ta_hi, &full_bar[stage], st, kc, a_row, kCacheEvictNormal);
              tma_load_2d(&ta_lo, &full_bar[stage], st + TILE_BYTES, kc, a_row, kCacheEvictNormal);
              if (EPI == EPI_SWIGLU) {
                tma_load_2d(&tb_hi, &full_bar[stage], bh, kc, b_row, kCacheEvictNormal);
                tma_load_2d(&tb2_hi, &full_bar[stage], bh + C::B_BYTES / 2, kc, b_row, kCacheEvictNormal);
                tma_load_2d(&tb_lo, &full_bar[stage], bl, kc, b_row, kCacheEvictNormal);
                tma_load_2d(&tb2_lo, &full_bar[stage], bl + C::B_BYTES / 2, kc, b_row, kCacheEvictNormal);
              } else {
                tma_load_2d(&tb_hi, &full_bar[stage], bh, kc, b_row, kCacheEvictNormal);
                tma_load_2d(&tb_lo, &full_bar[stage], bl, kc, b_row, kCacheEvictNormal);
              }
            } else {  // completion bytes of both CTAs go to the leader's barrier
              if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * C::STAGE_BYTES);
              const CUtensorMap* bhi = EPI == EPI_SWIGLU && rank == 1 ? &tb2_hi : &tb_hi;
              const CUtensorMap* blo = EPI == EPI_SWIGLU && rank == 1 ? &tb2_lo : &tb_lo;
              tma_load_2d_pair(&ta_hi, &full_bar[stage], st, kc, a_row, kCacheEvictNormal);
              tma_load_2d_pair(&ta_lo, &full_bar[stage], st + TILE_BYTES, kc, a_row, kCacheEvictNormal);
              tma_load_2d_pair(bhi, &full_bar[stage], bh, kc, b_row, kCacheEvictNormal);
              tma_load_2d_pair(blo, &full_bar[stage], bl, kc, b_row, kCacheEvictNormal);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (CG == 2) {
        // producer tail: every stage released, i.e. the leader's last
        // multicast commits to this CTA's barriers have landed before exit
        for (int i = 0; i < STAGES; ++i) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // ===== MMA issuer
      // The whole warp walks the schedule (barrier waits, descriptors: warp-
      // uniform values the compiler keeps in uniform registers) and one
      // elected lane issues the MMAs and their commits.  Issued from a
      // single-lane branch instead, every tcgen05.mma needed a waterfall loop
      // moving its operands to uniform registers (~200 instructions per
      // k-block for its 12 MMAs: the issue rate, not the tensor core, bounded
      // the k-loop -- profiles/r02_tf32_variants_ab.txt).
      // The tensor core adds each MMA into its fp32 accumulator with a
      // truncating (biased) rounding, so a tile's K range is accumulated in
      // chunks of CHUNK_KB k-blocks (on absolute k boundaries) into rotating
      // TMEM slots and the epilogue sums the chunks in registers (fp32, round
      // to nearest): the bias stays at ~CHUNK_KB * 12 roundings per chunk
      // instead of K * 3 / 8 per output.
      constexpr uint32_t idesc = umma_idesc_tf32(C::TILE_M, BN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk = 0;  // chunks issued by this worker (slot = chunk % SLOTS)
      Work w = work0;
      Segment g;
      while (w.next(g)) {
        for (int c0 = g.kb0; c0 < g.kb1; ++chunk) {
          const int c1 = min(g.kb1, (c0 / p.chunk_kb + 1) * p.chunk_kb);
          const int slot = chunk % SLOTS;
          mbar_wait(&tempty_bar[slot], ((chunk / SLOTS) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + slot * BN;
          for (int kb = c0; kb < c1; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            uint8_t* st = smem + stage * C::STAGE_BYTES;
            const uint64_t a_hi = umma_desc_sw128(st), a_lo = umma_desc_sw128(st + TILE_BYTES);
            const uint64_t b_hi = umma_desc_sw128(st + 2 * TILE_BYTES);
            const uint64_t b_lo = umma_desc_sw128(st + 2 * TILE_BYTES + C::B_BYTES);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk) {  // K = 8 tf32 = 32 B per MMA
                const uint64_t o = (uint64_t)(kk * 2);
                umma_tf32<CG>(tmem_d, a_lo + o, b_hi + o, idesc, (kb != c0 || kk != 0) ? 1u : 0u);
                umma_tf32<CG>(tmem_d, a_hi + o, b_lo + o, idesc, 1u);
                umma_tf32<CG>(tmem_d, a_hi + o, b_hi + o, idesc, 1u);
              }
              if (CG == 1)
                umma_commit(&empty_bar[stage]);
              else
                umma_commit_pair(&empty_bar[stage]);
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (elect_one()) {
            if (CG == 1)
              umma_commit(&tfull_bar[slot]);
            else
              umma_commit_pair(&tfull_bar[slot]);
          }
          __syncwarp();
          c0 = c1;
        }
      }
    }
  } else {  // ===== epilogue: warps 2..5, TMEM lane quarter = warp % 4
    const int quarter = warp & 3;
    const int r_local = quarter * 32 + lane;
    const int cta = (int)blockIdx.x;  // partial-tile slot of this CTA
    uint32_t chunk = 0;
    Work w = work0;
    Segment g;
    while (w.next(g)) {
      float acc[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
      for (int c0 = g.kb0; c0 < g.kb1; ++chunk) {
        const int c1 = min(g.kb1, (c0 / p.chunk_kb + 1) * p.chunk_kb);
        const int slot = chunk % SLOTS;
        mbar_wait(&tfull_bar[slot], (chunk / SLOTS) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + slot * BN;
#pragma unroll
        for (int cc = 0; cc < BN; cc += 32) {
          uint32_t a[32];
          tmem_ld_32x32b_x32(taddr + cc, a);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[cc + j] += __uint_as_float(a[j]);
        }
        tc_fence_before();
        if (lane == 0) {
          if (CG == 1)
            mbar_arrive(&tempty_bar[slot]);
          else
            mbar_arrive_leader_relaxed(&tempty_bar[slot]);
        }
        c0 = c1;
      }
      // stream-K: a segment not starting at k = 0 is a helper's share of the
      // tile (only a worker's first segment can be): raw partial out, then
      // count in.  The segment starting at k = 0 is the owner's (the last of
      // its range when the tile continues): it adds the helpers' partials in
      // k order -- deterministic for a given tile count -- then the epilogue.
      // Pairs: each CTA exchanges its own 128 rows (counter per tile and rank).
      if (g.kb0 > 0) {
        float4* mine = reinterpret_cast<float4*>(p.partial + (int64_t)cta * (BM * BN));
#pragma unroll
        for (int j = 0; j < BN; j += 4)
          __stcg(mine + (j / 4) * BM + r_local, make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
        if (warp == 2 && lane == 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.arrive + (int64_t)g.t * CG + rank)
                       : "memory");
        continue;
      }
      if (g.kb1 < KB) {
        const int last = worker_of((int64_t)g.t * KB + KB - 1, P, U);
        int32_t* cnt = p.arrive + (int64_t)g.t * CG + rank;
        wait_helpers(cnt, last - me, lane);
        for (int q = me + 1; q <= last; ++q) {
          const float4* hp = reinterpret_cast<const float4*>(p.partial + ((int64_t)q * CG + rank) * (BM * BN));
#pragma unroll
          for (int j = 0; j < BN; j += 4) {
            const float4 v = __ldcg(hp + (j / 4) * BM + r_local);
            acc[j] += v.x;
            acc[j + 1] += v.y;
            acc[j + 2] += v.z;
            acc[j + 3] += v.w;
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) *cnt = 0;  // the next launch (stream-ordered) starts from zero
      }
      int mb, nb, seg;
      decode(g.t, total_mb, p.n_blocks, p.group_m, s_offs, S, C::TILE_M, mb, nb, seg);
      const int64_t row = (int64_t)mb * C::TILE_M + (int)rank * BM + r_local;
      const int col0 = nb * p.out_block_cols;
      float* ohi = p.out_hi + row * p.ldo + col0;
      float* olo = p.out_lo ? p.out_lo + row * p.ldo + col0 : nullptr;
      constexpr int OUT = EPI == EPI_SWIGLU ? BN / 2 : BN;
#pragma unroll
      for (int cc = 0; cc < OUT; cc += 4) {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float gv = acc[cc + i];
          if (EPI == EPI_SWIGLU)
            v[i] = gv / (1.0f + expf(-gv)) * acc[BN / 2 + cc + i];
          else if (EPI == EPI_RELU)
            v[i] = fmaxf(gv, 0.0f);
          else
            v[i] = gv;
        }
        if (EPI == EPI_STORE) {
          *reinterpret_cast<float4*>(ohi + cc) = make_float4(v[0], v[1], v[2], v[3]);
        } else {  // H for GEMM2, already split into its tf32 hi / lo parts
          float h[4], l[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            h[i] = round_tf32(v[i]);
            l[i] = v[i] - h[i];
          }
          *reinterpret_cast<float4*>(ohi + cc) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(olo + cc) = make_float4(l[0], l[1], l[2], l[3]);
        }
      }
    }
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync_all();  // the peer's MMAs and TMEM reads are done before the pair frees TMEM
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

// x -> (tf32(x), x - tf32(x)) into hi (may alias x) / lo, n multiple of 4
// rows_dev (nullable): the device's row count (seg_offsets[E]); rows past it
// are never read by the GEMMs, so they are not split
__global__ void split_tf32_kernel(const float4* x, float4* hi, float4* __restrict__ lo, int64_t n4,
                                  const int64_t* rows_dev, int64_t row4) {
  if (rows_dev) n4 = min(n4, *rows_dev * row4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    float4 h, l;
    h.x = round_tf32(v.x);
    h.y = round_tf32(v.y);
    h.z = round_tf32(v.z);
    h.w = round_tf32(v.w);
    l.x = v.x - h.x;
    l.y = v.y - h.y;
    l.z = v.z - h.z;
    l.w = v.w - h.w;
    hi[i] = h;
    lo[i] = l;
  }
}

}  // namespace tf32x3


typedef CUresult (*PFN_encodeTiled32)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_tmap_f32_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  static PFN_encodeTiled32 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    EMOE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled not available");
    return reinterpret_cast<PFN_encodeTiled32>(ptr);
  }();
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)tf32x3::BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (f32) failed: " + std::to_string((int)r));
  return m;
}

void launch_split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s, const int64_t* rows_dev,
                       int row_elems) {
  EMOE_REQUIRE(n % 4 == 0, "split_tf32: element count must be a multiple of 4");
  EMOE_REQUIRE(!rows_dev || row_elems % 4 == 0, "split_tf32: row length must be a multiple of 4");
  if (n == 0) return;
  const int64_t n4 = n / 4;
  const int blocks = (int)std::min<int64_t>(ceil_div(n4, 256), 148 * 8);
  tf32x3::split_tf32_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(hi),
                                                   reinterpret_cast<float4*>(lo), n4, rows_dev, row_elems / 4);
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

bool gemm_tf32x3_supported(int epi, int K, int N_out) {
  return K % tf32x3::BK == 0 && N_out % (epi == EPI_SWIGLU ? tf32x3::BN / 2 : tf32x3::BN) == 0;
}

// CTA pair (M = 256 tiles) or single CTA (M = 128); EMOE_TF32_CG=1|2 (A/B runs)
int gemm_tf32x3_cta_group() {
  static const int cg = [] {
    const char* v = getenv("EMOE_TF32_CG");
    return v && v[0] == '1' ? 1 : v && v[0] == '2' ? 2 : 1;
  }();
  return cg;
}

int gemm_tf32x3_tile_m() { return tf32x3::BM * gemm_tf32x3_cta_group(); }

int gemm_tf32x3_b_box_rows(int epi) {
  if (gemm_tf32x3_cta_group() == 2) return tf32x3::BN / 2;  // each CTA of the pair loads half the B rows
  return epi == EPI_SWIGLU ? tf32x3::BN / 2 : tf32x3::BN;
}

// co-resident CTAs of the persistent stream-K kernel (owners wait on
// helpers, so every CTA of the grid must be resident at once), per device
static int coresident_ctas(const void* kernel, int threads, int smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  EMOE_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, kernel});
  if (it != cache.end()) return it->second;
  ensure_max_dynamic_smem(kernel, smem);
  int sms = 0, per_sm = 0;
  EMOE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  EMOE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  const int n = std::min(per_sm, 1) * sms;  // persistent: one CTA per SM
  if (n < 1) throw CudaError("gemm_tf32x3: the kernel does not fit on this device");
  cache[{dev, kernel}] = n;
  return n;
}

size_t gemm_tf32x3_partial_floats(int num_sms) { return (size_t)num_sms * tf32x3::BM * tf32x3::BN; }

int64_t gemm_tf32x3_arrivals(int epi, int N_out, int64_t rows) {
  return ceil_div(rows, tf32x3::BM) * (N_out / (epi == EPI_SWIGLU ? tf32x3::BN / 2 : tf32x3::BN));
}

template <int EPI, int CG>
static void launch_tf32(const Tf32Operands& ops, const tf32x3::Params& p, int ctas, cudaStream_t stream) {
  using namespace tf32x3;
  EMOE_CUDA(launch_pdl(gemm_tf32x3_kernel<EPI, CG>, dim3(ctas), dim3(NUM_THREADS), (size_t)TCfg<CG>::SMEM_BYTES, stream,
                       CG, ops.a_hi, ops.a_lo, ops.b_hi, ops.b_lo, ops.b2_hi, ops.b2_lo, p));
}

template <int CG>
static void launch_cg(int epi, const Tf32Operands& ops, const tf32x3::Params& p, const StreamK& sk,
                      cudaStream_t stream) {
  using namespace tf32x3;
  const void* kern = epi == EPI_SWIGLU ? reinterpret_cast<const void*>(gemm_tf32x3_kernel<EPI_SWIGLU, CG>)
                     : epi == EPI_RELU ? reinterpret_cast<const void*>(gemm_tf32x3_kernel<EPI_RELU, CG>)
                                       : reinterpret_cast<const void*>(gemm_tf32x3_kernel<EPI_STORE, CG>);
  int ctas = coresident_ctas(kern, NUM_THREADS, TCfg<CG>::SMEM_BYTES);
  ctas = (int)std::min<size_t>(ctas, sk.partial_floats / (BM * BN));
  ctas = ctas / CG * CG;
  EMOE_REQUIRE(ctas >= CG, "gemm_tf32x3: stream-K partial buffer too small");
  if (epi == EPI_SWIGLU)
    launch_tf32<EPI_SWIGLU, CG>(ops, p, ctas, stream);
  else if (epi == EPI_RELU)
    launch_tf32<EPI_RELU, CG>(ops, p, ctas, stream);
  else
    launch_tf32<EPI_STORE, CG>(ops, p, ctas, stream);
}

void launch_grouped_gemm_tf32x3(int epi, const Tf32Operands& ops, const int64_t* seg_offsets,
                                const int32_t* slot_of_expert, const int32_t* seg_expert, int n_seg, int K, int N_out,
                                int b_rows_per_slot, float* out_hi, float* out_lo, int64_t ldo, int64_t max_rows,
                                const StreamK& sk, cudaStream_t stream) {
  using namespace tf32x3;
  EMOE_REQUIRE(n_seg >= 1 && n_seg <= MAX_SEGS, "gemm_tf32x3: segment count out of range");
  EMOE_REQUIRE(gemm_tf32x3_supported(epi, K, N_out), "gemm_tf32x3: K % 32 and N % tile must be 0");
  EMOE_REQUIRE(epi == EPI_STORE || out_lo, "gemm_tf32x3: GEMM1 needs the lo output");
  Params p;
  p.seg_offsets = seg_offsets;
  p.slot_of_expert = slot_of_expert;
  p.seg_expert = seg_expert;
  p.n_seg = n_seg;
  p.K = K;
  p.out_block_cols = epi == EPI_SWIGLU ? BN / 2 : BN;
  p.n_blocks = N_out / p.out_block_cols;
  p.b_rows_per_slot = b_rows_per_slot;
  // raster: A panel of ~8 MB (the fp32 hi + lo rows of the group) stays in L2
  p.group_m = std::max(2, std::min(64, (int)((8ll << 20) / ((int64_t)gemm_tf32x3_tile_m() * K * 8))));
  p.out_hi = out_hi;
  p.out_lo = out_lo;
  p.ldo = ldo;
  p.partial = sk.partial;
  p.arrive = sk.arrive;
  // Schedule (profiles/r02_tf32_variants_ab.txt): GEMM2 stream-K (config 1:
  // 64 tiles of 112 k-blocks for 148 SMs, 56.3 -> 50.3 us over split-K),
  // GEMM1 whole tiles round-robin (448 tiles = 3.03 waves: stream-K's fixups
  // cost more than the 4th round's 4 tiles).  EMOE_TF32_SK = bitmask of the
  // GEMMs on stream-K (1 = GEMM1, 2 = GEMM2), A/B runs.
  static const int sk_mask = [] {
    const char* v = getenv("EMOE_TF32_SK");
    return v ? atoi(v) : 2;
  }();
  p.dp = (sk_mask & (epi == EPI_STORE ? 2 : 1)) ? 0 : 1;
  static const int chunk_kb = [] {
    const char* v = getenv("EMOE_TF32_CHUNK");
    return v ? std::max(1, atoi(v)) : CHUNK_KB;
  }();
  p.chunk_kb = chunk_kb;
  EMOE_REQUIRE(gemm_tf32x3_arrivals(epi, N_out, max_rows) <= sk.arrivals,
               "gemm_tf32x3: stream-K arrival table smaller than the tile count");
  if (gemm_tf32x3_cta_group() == 2)
    launch_cg<2>(epi, ops, p, sk, stream);
  else
    launch_cg<1>(epi, ops, p, sk, stream);
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace emoe
