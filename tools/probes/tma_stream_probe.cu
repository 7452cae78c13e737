// Probe: how fast can a persistent kernel stream x [T][d] bf16 (Switch
// shape: T = 65,536, d = 768, 100 MB) from HBM into shared memory?  Used to
// find the floor of the fused gate kernel (gate_tc.cu), which is ~35 us in
// every variant.  Modes:
//   tma  R   one CTA per SM, ring of S stages, each stage one TMA box of R
//            rows x 64 bf16 (SWIZZLE_128B, the gate kernel's x box), rows
//            walked tile by tile (128 rows x 12 k-blocks per tile)
//   tmar R   the same, but the k-blocks of a tile are walked row-panel by
//            row-panel (all 12 k-blocks of R rows before the next R rows)
//   ldg      every thread LDG.128 over the flat buffer (a read-only copy)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream_probe tma_stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap tm, int T, int d, int R,
                                                    int S, int rowmajor, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = R * 128;
  uint64_t* full = (uint64_t*)(smem + S * stage_bytes);
  uint64_t* empty = full + 16;
  const int kblocks = d / 64;
  const int ntiles = T / 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int sub = 128 / R;  // boxes per 128-row tile per k-block
  const int per_tile = kblocks * sub;
  if (threadIdx.x == 0) {  // producer
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int i = 0; i < per_tile; ++i) {
        const int kb = rowmajor ? i % kblocks : i / sub;
        const int rb = rowmajor ? i / kblocks : i % sub;
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
              : "=r"(ok)
              : "r"(su(&empty[stage])), "r"(phase ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[stage])),
                     "r"(stage_bytes));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su(smem + stage * stage_bytes)),
            "l"((uint64_t)&tm), "r"(su(&full[stage])), "r"(kb * 64), "r"(t * 128 + rb * R)
            : "memory");
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
  } else if (threadIdx.x == 32) {  // consumer: touch one word, release
    int stage = 0;
    uint32_t phase = 0;
    unsigned long long acc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int i = 0; i < per_tile; ++i) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
              : "=r"(ok)
              : "r"(su(&full[stage])), "r"(phase));
        acc += *(volatile uint32_t*)(smem + stage * stage_bytes);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[stage])));
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    if (acc == 0x123456789ull) *sink = acc;
  }
}

__global__ void ldg_stream(const uint4* x, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(x + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const int T = 65536, d = argc > 1 ? atoi(argv[1]) : 768;
  const size_t bytes = (size_t)T * d * 2;
  void* x;
  cudaMalloc(&x, bytes);
  cudaMemset(x, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* flush;
  const size_t fbytes = 256ull << 20;
  cudaMalloc(&flush, fbytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  PFN enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn) {
    float best = 1e9;
    for (int rep = 0; rep < 7; ++rep) {
      cudaMemset(flush, rep, fbytes);  // evict x from L2
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    return best * 1e3f;
  };
  for (int R : {128, 64, 32}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)R};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int rowmajor : {0, 1})
      for (int S : {4, 8, 12}) {
        const int smem = 1024 + S * R * 128 + 256;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const float us = timeit([&] { tma_stream<<<sms, 64, smem>>>(tm, T, d, R, S, rowmajor, sink); });
        printf("tma box %3dx64 %s stages %2d (%3d KB in flight/SM): %7.2f us  %6.0f GB/s\n", R,
               rowmajor ? "row-panel" : "k-outer  ", S, S * R * 128 / 1024, us, bytes / (us * 1e3));
      }
  }
  for (int blocks : {sms * 4, sms * 8, sms * 16}) {
    const float us = timeit([&] { ldg_stream<<<blocks, 256>>>((const uint4*)x, bytes / 16, sink); });
    printf("ldg.128 %5d blocks x 256: %7.2f us  %6.0f GB/s\n", blocks, us, bytes / (us * 1e3));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
