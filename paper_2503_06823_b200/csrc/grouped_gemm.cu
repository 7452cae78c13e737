// K4: grouped expert FFN GEMM on 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel computes, for every resident expert
// e with rows X[off_e : off_e + n_e) of the permuted activations,
//     out[rows, n-block] = epilogue( X_rows . W_e[n-block rows]^T )
// with three epilogues:
//   EPI_SWIGLU  B tile = 128 rows of W1 + the same 128 rows of W3,
//               H = silu(X W1^T) * (X W3^T) -> bf16  (GEMM1, Mixtral / synthetic)
//   EPI_RELU    B tile = 256 rows of W1, H = relu(X W1^T) -> bf16  (GEMM1, Switch)
//   EPI_STORE   B tile = 256 rows of W2, Y = H W2^T -> bf16          (GEMM2)
//
// Hardware mapping (B200, one CTA per SM, 6 warps):
//   warp 0      TMA producer: A (128 x 64) and B (256 x 64) bf16 tiles, 128-B
//               swizzle, into a 4-stage shared-memory ring (48 KB / stage)
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.cta_group::1
//               kind::f16 M=128 N=256 K=16 (4 per 64-wide k-block); accumulators
//               live in TMEM, double-buffered (2 x 256 of 512 columns) so the
//               epilogue of tile i overlaps the mainloop of tile i+1
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> activation -> bf16
//               -> global (each warp owns its 32-lane TMEM quarter)
// Segments are padded to 128 rows by the permute kernel, so every 128-row
// block belongs to exactly one expert and all loads/stores stay in bounds.
// Tiles are walked in a grouped raster (8 row blocks x all n blocks) so the
// 148 concurrently running tiles share A and B tiles through L2.
#include "common.cuh"
#include "kernels.h"

namespace emoe {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 256;  // UMMA N / accumulator columns per tile
constexpr int BK = 64;   // one 128-byte swizzle row of bf16
constexpr int STAGES = 4;
constexpr int GROUP_M = 8;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int MAX_EXPERTS = 256;
constexpr int NUM_THREADS = 192;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 4096 /*barriers + offsets*/;

struct Params {
  const int64_t* seg_offsets;   // [E+1], multiples of BM
  const int32_t* slot_of_expert;  // [E]
  int num_experts;
  int K;                // reduction length (multiple of BK)
  int n_blocks;         // output column blocks
  int out_block_cols;   // 128 (SwiGLU) or 256
  int b_rows_per_slot;  // rows of one expert in the B pool
  __nv_bfloat16* out;
  int64_t ldo;
};

struct TileCoord {
  int rb, nb, expert;
};

__device__ __forceinline__ TileCoord decode_tile(int t, int total_rb, int n_blocks, const int64_t* offs,
                                                 int num_experts) {
  const int per_group = GROUP_M * n_blocks;
  const int g = t / per_group;
  const int local = t - g * per_group;
  const int rows_in_group = min(GROUP_M, total_rb - g * GROUP_M);
  TileCoord c;
  c.nb = local / rows_in_group;
  c.rb = g * GROUP_M + (local - c.nb * rows_in_group);
  const int64_t row = (int64_t)c.rb * BM;
  int e = 0;
  while (e + 1 < num_experts && offs[e + 1] <= row) ++e;
  c.expert = e;
  return c;
}

template <int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const __grid_constant__ CUtensorMap tmap_b2, Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int64_t* s_offs = reinterpret_cast<int64_t*>(tmem_slot + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int E = p.num_experts;

  for (int i = threadIdx.x; i <= E; i += NUM_THREADS) s_offs[i] = p.seg_offsets[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    if (EPI == EPI_SWIGLU) tma_prefetch_desc(&tmap_b2);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 128);
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

  const int total_rb = (int)(s_offs[E] / BM);
  const int total_tiles = total_rb * p.n_blocks;
  const int k_blocks = p.K / BK;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const TileCoord c = decode_tile(t, total_rb, p.n_blocks, s_offs, E);
        const int slot = p.slot_of_expert[c.expert];
        const int a_row = c.rb * BM;
        const int b_row = slot * p.b_rows_per_slot + c.nb * (EPI == EPI_SWIGLU ? BN / 2 : BN);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          const int kc = kb * BK;
          tma_load_2d(&tmap_a, &full_bar[stage], smem_a + stage * A_STAGE_BYTES, kc, a_row, kCacheEvictNormal);
          uint8_t* bdst = smem_b + stage * B_STAGE_BYTES;
          if (EPI == EPI_SWIGLU) {
            tma_load_2d(&tmap_b, &full_bar[stage], bdst, kc, b_row, kCacheEvictNormal);
            tma_load_2d(&tmap_b2, &full_bar[stage], bdst + B_STAGE_BYTES / 2, kc, b_row, kCacheEvictNormal);
          } else {
            tma_load_2d(&tmap_b, &full_bar[stage], bdst, kc, b_row, kCacheEvictNormal);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++local) {
        const int buf = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[buf], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = umma_desc_sw128(smem_a + stage * A_STAGE_BYTES);
          const uint64_t b_desc = umma_desc_sw128(smem_b + stage * B_STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // advance 16 bf16 = 32 B inside the 128-B swizzle row
            umma_bf16(tmem_d, a_desc + (uint64_t)(kk * 2), b_desc + (uint64_t)(kk * 2), idesc,
                      (kb | kk) != 0 ? 1u : 0u);
          }
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
    // ===================== epilogue (warps 2..5) =====================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    int local = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++local) {
      const TileCoord c = decode_tile(t, total_rb, p.n_blocks, s_offs, E);
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      const int64_t row = (int64_t)c.rb * BM + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * BN;
      __nv_bfloat16* orow = p.out + row * p.ldo + (int64_t)c.nb * p.out_block_cols;
      if (EPI == EPI_SWIGLU) {
#pragma unroll 1
        for (int cc = 0; cc < BN / 2; cc += 32) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(taddr + cc, g);
          tmem_ld_32x32b_x32(taddr + BN / 2 + cc, u);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float g0 = __uint_as_float(g[2 * j]), g1 = __uint_as_float(g[2 * j + 1]);
            float u0 = __uint_as_float(u[2 * j]), u1 = __uint_as_float(u[2 * j + 1]);
            float h0 = g0 / (1.0f + __expf(-g0)) * u0;
            float h1 = g1 / (1.0f + __expf(-g1)) * u1;
            packed[j] = pack_bf16x2(h0, h1);
          }
          uint4* dst = reinterpret_cast<uint4*>(orow + cc);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
        }
      } else {
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 32) {
          uint32_t a[32];
          tmem_ld_32x32b_x32(taddr + cc, a);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float v0 = __uint_as_float(a[2 * j]), v1 = __uint_as_float(a[2 * j + 1]);
            if (EPI == EPI_RELU) {
              v0 = fmaxf(v0, 0.0f);
              v1 = fmaxf(v1, 0.0f);
            }
            packed[j] = pack_bf16x2(v0, v1);
          }
          uint4* dst = reinterpret_cast<uint4*>(orow + cc);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[buf]);
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
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

int gemm_smem_bytes() { return gemm::SMEM_BYTES; }

void launch_grouped_gemm(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2,
                         const int64_t* seg_offsets, const int32_t* slot_of_expert, int num_experts, int K,
                         int N_out, int b_rows_per_slot, __nv_bfloat16* out, int64_t ldo, int num_sms,
                         cudaStream_t stream) {
  EMOE_REQUIRE(num_experts <= gemm::MAX_EXPERTS, "grouped_gemm: too many experts");
  EMOE_REQUIRE(K % gemm::BK == 0, "grouped_gemm: K must be a multiple of 64");
  gemm::Params p;
  p.seg_offsets = seg_offsets;
  p.slot_of_expert = slot_of_expert;
  p.num_experts = num_experts;
  p.K = K;
  p.out_block_cols = epi == EPI_SWIGLU ? gemm::BN / 2 : gemm::BN;
  EMOE_REQUIRE(N_out % p.out_block_cols == 0, "grouped_gemm: N must be a multiple of the column block");
  p.n_blocks = N_out / p.out_block_cols;
  p.b_rows_per_slot = b_rows_per_slot;
  p.out = out;
  p.ldo = ldo;
  auto run = [&](auto kernel) {
    static bool attr_set[3] = {false, false, false};
    if (!attr_set[epi]) {
      EMOE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm::SMEM_BYTES));
      attr_set[epi] = true;
    }
    kernel<<<num_sms, gemm::NUM_THREADS, gemm::SMEM_BYTES, stream>>>(ta, tb, tb2, p);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
  };
  if (epi == EPI_SWIGLU)
    run(gemm::grouped_gemm_kernel<EPI_SWIGLU>);
  else if (epi == EPI_RELU)
    run(gemm::grouped_gemm_kernel<EPI_RELU>);
  else
    run(gemm::grouped_gemm_kernel<EPI_STORE>);
}

}  // namespace emoe
