// Probe: TMA tile::gather4 semantics on sm_100a (box shape, swizzle placement).
// Loads 32 gathered rows (8 x gather4) of a bf16 [rows][64] tensor into a
// 128-B-swizzled 32 x 128 B smem tile and compares with the expected layout
// (16-B chunk c of tile row r at chunk c ^ (r & 7)).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap tm, const int* idx, uint16_t* out) {
  __shared__ __align__(1024) uint16_t tile[32 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32 * 128));
    for (int g = 0; g < 8; ++g) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(tile + g * 4 * 64);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(b), "r"(0), "r"(idx[4 * g]), "r"(idx[4 * g + 1]),
          "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3])
          : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) out[i] = tile[i];
}

int main() {
  const int R = 1000, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 64 + c);  // unique per element (mod 65536)
  uint16_t *d, *o;
  int* di;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 32 * 64 * 2);
  cudaMalloc(&di, 32 * 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  std::vector<int> idx(32);
  for (int i = 0; i < 32; ++i) idx[i] = (i * 37 + 11) % R;
  cudaMemcpy(di, idx.data(), 32 * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  int rc_all = 0;
  for (int boxr : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxr};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((PFN)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("box rows %d: encode failed %d\n", boxr, (int)r);
      continue;
    }
    cudaMemset(o, 0, 32 * 64 * 2);
    probe<<<1, 128>>>(tm, di, o);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("box rows %d: kernel error %s\n", boxr, cudaGetErrorString(e));
      return 1;
    }
    std::vector<uint16_t> got(32 * 64);
    cudaMemcpy(got.data(), o, got.size() * 2, cudaMemcpyDeviceToHost);
    int bad_sw = 0, bad_lin = 0;
    for (int rr = 0; rr < 32; ++rr)
      for (int c = 0; c < 64; ++c) {
        const uint16_t want = h[idx[rr] * C + c];
        const int chunk = c / 8, within = c % 8;
        const int sw = rr * 64 + ((chunk ^ (rr & 7)) * 8) + within;
        if (got[sw] != want) ++bad_sw;
        if (got[rr * 64 + c] != want) ++bad_lin;
      }
    printf("box rows %d: mismatches swizzled=%d linear=%d\n", boxr, bad_sw, bad_lin);
    rc_all |= bad_sw != 0;
  }
  return 0;
}
