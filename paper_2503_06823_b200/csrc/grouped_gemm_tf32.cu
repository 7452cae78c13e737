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
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace emoe {
namespace tf32x3 {

constexpr int BM = 128, BN = 128;
constexpr int BK = 32;  // fp32 elements per 128-B swizzle row
constexpr int STAGES = 3;
constexpr int TILE_BYTES = 128 * 128;  // 128 rows x 128 B
constexpr int STAGE_BYTES = 4 * TILE_BYTES;
constexpr int NUM_THREADS = 192;
constexpr int SLOTS = 4;     // rotating TMEM accumulator slots (4 x 128 columns)
constexpr int CHUNK_KB = 4;  // k-blocks (128 of K) per accumulator chunk
constexpr int TMEM_COLS = SLOTS * BN;
constexpr int MAX_SEGS = 256;
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 4096;
static_assert(2 * STAGES * 8 + 2 * SLOTS * 8 + 16 + 4 * (2 * MAX_SEGS + 1) <= 4096, "barrier / table area");

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
  // split-K (few output tiles): work item = (tile, split); split s reduces
  // k-blocks [s KB / k_splits, (s + 1) KB / k_splits) and stores its raw
  // fp32 accumulators to partial[s][row][nb * BN + col]; splitk_reduce_kernel
  // sums the splits in order and applies the epilogue
  int k_splits;
  float* partial;
  int64_t partial_rows;
};

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, 1 CTA
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
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
                                       int& mb, int& nb, int& seg) {
  const int per_group = group_m * n_blocks;
  const int g = t / per_group;
  const int local = t - g * per_group;
  const int rows_in_group = min(group_m, total_mb - g * group_m);
  nb = local / rows_in_group;
  mb = g * group_m + (local - nb * rows_in_group);
  const int row = mb * BM;
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

template <int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                       const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                       const __grid_constant__ CUtensorMap tb2_hi, const __grid_constant__ CUtensorMap tb2_lo,
                       Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [SLOTS]
  uint64_t* tempty_bar = tfull_bar + SLOTS;  // [SLOTS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + SLOTS);
  int32_t* s_offs = reinterpret_cast<int32_t*>(tmem_slot + 4);
  int32_t* s_slot = s_offs + MAX_SEGS + 1;  // weight slot per segment: no dependent global loads per tile

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int S = p.n_seg;
  for (int i = threadIdx.x; i <= S; i += NUM_THREADS) s_offs[i] = (int32_t)p.seg_offsets[i];
  for (int i = threadIdx.x; i < S; i += NUM_THREADS) s_slot[i] = p.slot_of_expert[p.seg_expert ? p.seg_expert[i] : i];
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
      mbar_init(&tempty_bar[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_mb = s_offs[S] / BM;
  const int total_tiles = total_mb * p.n_blocks;
  const int total_items = total_tiles * p.k_splits;
  const int k_blocks = p.K / BK;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < total_items; w += gridDim.x) {
        const int t = w / p.k_splits, split = w - t * p.k_splits;
        int mb, nb, seg;
        decode(t, total_mb, p.n_blocks, p.group_m, s_offs, S, mb, nb, seg);
        const int slot = s_slot[seg];
        const int a_row = mb * BM;
        const int b_row = slot * p.b_rows_per_slot + nb * (EPI == EPI_SWIGLU ? BN / 2 : BN);
        const int kbeg = split * k_blocks / p.k_splits, kend = (split + 1) * k_blocks / p.k_splits;
        for (int kb = kbeg; kb < kend; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          uint8_t* st = smem + stage * STAGE_BYTES;
          const int kc = kb * BK;
          tma_load_2d(&ta_hi, &full_bar[stage], st, kc, a_row, kCacheEvictNormal);
          tma_load_2d(&ta_lo, &full_bar[stage], st + TILE_BYTES, kc, a_row, kCacheEvictNormal);
          if (EPI == EPI_SWIGLU) {  // B tile rows 0-63: W1, 64-127: W3 (same output columns)
            tma_load_2d(&tb_hi, &full_bar[stage], st + 2 * TILE_BYTES, kc, b_row, kCacheEvictNormal);
            tma_load_2d(&tb2_hi, &full_bar[stage], st + 2 * TILE_BYTES + TILE_BYTES / 2, kc, b_row,
                        kCacheEvictNormal);
            tma_load_2d(&tb_lo, &full_bar[stage], st + 3 * TILE_BYTES, kc, b_row, kCacheEvictNormal);
            tma_load_2d(&tb2_lo, &full_bar[stage], st + 3 * TILE_BYTES + TILE_BYTES / 2, kc, b_row,
                        kCacheEvictNormal);
          } else {
            tma_load_2d(&tb_hi, &full_bar[stage], st + 2 * TILE_BYTES, kc, b_row, kCacheEvictNormal);
            tma_load_2d(&tb_lo, &full_bar[stage], st + 3 * TILE_BYTES, kc, b_row, kCacheEvictNormal);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      // The tensor core adds each MMA into its fp32 accumulator with a
      // truncating (biased) rounding, so a tile's K range is accumulated in
      // chunks of CHUNK_KB k-blocks into rotating TMEM slots and the epilogue
      // sums the chunks in registers (fp32, round to nearest): the bias stays
      // at ~CHUNK_KB * 12 roundings per chunk instead of K * 3 / 8 per output.
      constexpr uint32_t idesc = umma_idesc_tf32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk = 0;  // chunks issued by this CTA (slot = chunk % SLOTS)
      for (int w = blockIdx.x; w < total_items; w += gridDim.x) {
        const int split = w % p.k_splits;
        const int kbeg = split * k_blocks / p.k_splits, kend = (split + 1) * k_blocks / p.k_splits;
        for (int kb0 = kbeg; kb0 < kend; kb0 += CHUNK_KB, ++chunk) {
          const int slot = chunk % SLOTS;
          mbar_wait(&tempty_bar[slot], ((chunk / SLOTS) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + slot * BN;
          const int kb1 = min(kend, kb0 + CHUNK_KB);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            uint8_t* st = smem + stage * STAGE_BYTES;
            const uint64_t a_hi = umma_desc_sw128(st), a_lo = umma_desc_sw128(st + TILE_BYTES);
            const uint64_t b_hi = umma_desc_sw128(st + 2 * TILE_BYTES), b_lo = umma_desc_sw128(st + 3 * TILE_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {  // K = 8 tf32 = 32 B per MMA
              const uint64_t o = (uint64_t)(kk * 2);
              umma_tf32(tmem_d, a_lo + o, b_hi + o, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
              umma_tf32(tmem_d, a_hi + o, b_lo + o, idesc, 1u);
              umma_tf32(tmem_d, a_hi + o, b_hi + o, idesc, 1u);
            }
            umma_commit(&empty_bar[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&tfull_bar[slot]);
        }
      }
    }
  } else {  // ===== epilogue: warps 2..5, TMEM lane quarter = warp % 4
    const int quarter = warp & 3;
    uint32_t chunk = 0;
    for (int w = blockIdx.x; w < total_items; w += gridDim.x) {
      const int t = w / p.k_splits, split = w - t * p.k_splits;
      const int kbeg = split * k_blocks / p.k_splits, kend = (split + 1) * k_blocks / p.k_splits;
      int mb, nb, seg;
      decode(t, total_mb, p.n_blocks, p.group_m, s_offs, S, mb, nb, seg);
      float acc[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
      for (int kb0 = kbeg; kb0 < kend; kb0 += CHUNK_KB, ++chunk) {
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
        if (lane == 0) mbar_arrive(&tempty_bar[slot]);
      }
      const int64_t row = (int64_t)mb * BM + quarter * 32 + lane;
      if (p.k_splits > 1) {  // raw partial sums; the reduce kernel finishes the tile
        float* dst = p.partial + ((int64_t)split * p.partial_rows + row) * ((int64_t)p.n_blocks * BN) + nb * BN;
#pragma unroll
        for (int j = 0; j < BN; j += 4)
          *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        continue;
      }
      const int col0 = nb * p.out_block_cols;
      float* ohi = p.out_hi + row * p.ldo + col0;
      float* olo = p.out_lo ? p.out_lo + row * p.ldo + col0 : nullptr;
      constexpr int OUT = EPI == EPI_SWIGLU ? BN / 2 : BN;
#pragma unroll
      for (int cc = 0; cc < OUT; cc += 4) {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float g = acc[cc + i];
          if (EPI == EPI_SWIGLU)
            v[i] = g / (1.0f + expf(-g)) * acc[BN / 2 + cc + i];
          else if (EPI == EPI_RELU)
            v[i] = fmaxf(g, 0.0f);
          else
            v[i] = g;
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
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
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

// split-K: out = epilogue(sum over splits of partial, in split order); one
// thread per output element (SwiGLU: gate column c and up column 64 + c of
// the tile's accumulators)
template <int EPI>
__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int k_splits, int64_t rows, int n_blocks,
                                     int out_block_cols, float* __restrict__ out_hi, float* __restrict__ out_lo,
                                     int64_t ldo, const int64_t* __restrict__ rows_dev) {
  // rows = the partial buffer's row stride; only the rows the GEMM wrote
  // (seg_offsets[E] on the device) are reduced
  const int64_t n_out = min(rows, *rows_dev) * (int64_t)n_blocks * out_block_cols;
  const int64_t acc_cols = (int64_t)n_blocks * BN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / ((int64_t)n_blocks * out_block_cols);
    const int oc = (int)(i - row * (int64_t)n_blocks * out_block_cols);
    const int nb = oc / out_block_cols, c = oc - nb * out_block_cols;
    const float* src = partial + row * acc_cols + nb * BN + c;
    float g = 0.0f, u = 0.0f;
    for (int sp = 0; sp < k_splits; ++sp) {
      g += src[(int64_t)sp * rows * acc_cols];
      if (EPI == EPI_SWIGLU) u += src[(int64_t)sp * rows * acc_cols + BN / 2];
    }
    float v;
    if (EPI == EPI_SWIGLU)
      v = g / (1.0f + expf(-g)) * u;
    else if (EPI == EPI_RELU)
      v = fmaxf(g, 0.0f);
    else
      v = g;
    const int64_t o = row * ldo + oc;
    if (EPI == EPI_STORE) {
      out_hi[o] = v;
    } else {
      const float h = round_tf32(v);
      out_hi[o] = h;
      out_lo[o] = v - h;
    }
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

int gemm_tf32x3_b_box_rows(int epi) { return epi == EPI_SWIGLU ? tf32x3::BN / 2 : tf32x3::BN; }

// one function per kernel instantiation
template <int EPI>
static void launch_kernel(const Tf32Operands& ops, const tf32x3::Params& p, int num_sms, cudaStream_t stream) {
  using namespace tf32x3;
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(gemm_tf32x3_kernel<EPI>), SMEM_BYTES);
  gemm_tf32x3_kernel<EPI><<<num_sms, NUM_THREADS, SMEM_BYTES, stream>>>(ops.a_hi, ops.a_lo, ops.b_hi, ops.b_lo,
                                                                       ops.b2_hi, ops.b2_lo, p);
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

void launch_grouped_gemm_tf32x3(int epi, const Tf32Operands& ops, const int64_t* seg_offsets,
                                const int32_t* slot_of_expert, const int32_t* seg_expert, int n_seg, int K, int N_out,
                                int b_rows_per_slot, float* out_hi, float* out_lo, int64_t ldo, int num_sms,
                                cudaStream_t stream, const SplitK* split) {
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
  p.group_m = std::max(2, std::min(64, (int)((8ll << 20) / ((int64_t)BM * K * 8))));
  p.out_hi = out_hi;
  p.out_lo = out_lo;
  p.ldo = ldo;
  p.k_splits = 1;
  p.partial = nullptr;
  p.partial_rows = 0;
  // split-K when even the row capacity gives fewer than two waves of tiles
  // (small token batches: config 1's GEMM2 has <= 128 tiles for 148 SMs)
  if (split && split->partial) {
    const int64_t max_tiles = split->rows / BM * p.n_blocks;
    int ks = 1;
    // at most 2 splits: config 1's GEMM2 runs 64.0 us with 4 splits, 59.7 us with 2 (the
    // reduce reads half the partials; profiles/r01_tf32_splitk_ab.jsonl)
    while (ks < 2 && max_tiles * ks < 2 * num_sms && (K / BK) / (2 * ks) >= 2 * CHUNK_KB) ks *= 2;
    static const int forced = [] {  // EMOE_TF32_SPLITK=n: force n splits where the scratch allows (A/B runs)
      const char* v = getenv("EMOE_TF32_SPLITK");
      return v ? atoi(v) : 0;
    }();
    if (forced > 0) ks = forced;
    if (ks > 1 && (size_t)ks * split->rows * p.n_blocks * BN <= split->capacity) {
      p.k_splits = ks;
      p.partial = split->partial;
      p.partial_rows = split->rows;
    }
  }
  if (epi == EPI_SWIGLU)
    launch_kernel<EPI_SWIGLU>(ops, p, num_sms, stream);
  else if (epi == EPI_RELU)
    launch_kernel<EPI_RELU>(ops, p, num_sms, stream);
  else
    launch_kernel<EPI_STORE>(ops, p, num_sms, stream);
  if (p.k_splits > 1) {
    const int64_t n_out = split->rows * p.n_blocks * p.out_block_cols;
    const int blocks = (int)std::min<int64_t>(ceil_div(n_out, 256), (int64_t)num_sms * 8);
    if (epi == EPI_SWIGLU)
      splitk_reduce_kernel<EPI_SWIGLU><<<blocks, 256, 0, stream>>>(p.partial, p.k_splits, split->rows, p.n_blocks,
                                                                    p.out_block_cols, out_hi, out_lo, ldo,
                                                                   seg_offsets + n_seg);
    else if (epi == EPI_RELU)
      splitk_reduce_kernel<EPI_RELU><<<blocks, 256, 0, stream>>>(p.partial, p.k_splits, split->rows, p.n_blocks,
                                                                  p.out_block_cols, out_hi, out_lo, ldo,
                                                                   seg_offsets + n_seg);
    else
      splitk_reduce_kernel<EPI_STORE><<<blocks, 256, 0, stream>>>(p.partial, p.k_splits, split->rows, p.n_blocks,
                                                                   p.out_block_cols, out_hi, out_lo, ldo,
                                                                   seg_offsets + n_seg);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
  }
}

}  // namespace emoe
