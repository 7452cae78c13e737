// Probe: issue rate of tcgen05.mma from shared-memory operands, no loads.
// One persistent CTA per SM; one thread issues R back-to-back MMAs into one
// TMEM accumulator (operands: zero-filled 128-B-swizzled tiles already in
// shared memory), commits, waits.  Reports the clocks per MMA and the MAC
// rate per SM, for the shapes the 3xTF32 config-1 kernels could use:
//   tf32 M128 N128 K8   (the 1-CTA 3xTF32 tile)
//   tf32 M128 N256 K8
//   tf32 M256 N256 K8   (CTA pair, cta_group::2)
//   bf16 M128 N256 K16  (the bf16 GEMM tile, reference point)
// With BG = 1 a second warp streams 16-KB bulk copies (cp.async.bulk, an
// L2-resident 2 MB source) into an 8-slot shared-memory ring for as long as
// the MMAs run: operand reads of the tensor core against TMA writes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2503_06823_b200/csrc -o umma_rate_probe umma_rate_probe.cu
#include <cstdio>

#include "common.cuh"

using namespace emoe;

constexpr int R = 4096;

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// kind: 0 tf32 1-CTA, 1 bf16 1-CTA, 2 tf32 pair
template <int KIND, int N, int BG>
__global__ void __launch_bounds__(128, 1) umma_rate(long long* cycles, const uint8_t* src, int* stop) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;                 // 128 rows x 128 B
  uint8_t* b = smem + 128 * 128;     // up to 256 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 128 * 128 + 256 * 128);
  uint8_t* ring = smem + 128 * 128 + 256 * 128 + 1024;  // 8 x 16 KB background ring
  uint64_t* rbar = bar + 8;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const bool pair = KIND == 2;
  const uint32_t rank = pair ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  __shared__ int done;
  if (threadIdx.x == 0) done = 0;
  fence_proxy_async();
  if (threadIdx.x < 32) {
    if (pair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(slot, 512);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (pair)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t ad = umma_desc_sw128(a), bd = umma_desc_sw128(b);
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const uint64_t o = (uint64_t)((i & 3) * 2);
      if (KIND == 0) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad + o), "l"(bd + o), "r"(idesc_tf32(128, N)), "r"(1)
            : "memory");
      } else if (KIND == 1) {
        umma_bf16(tmem, ad + o, bd + o, umma_idesc_bf16(128, N), 1u);
      } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad + o), "l"(bd + o), "r"(idesc_tf32(256, N)), "r"(1)
            : "memory");
      }
    }
    if (pair)
      umma_commit_pair(bar);
    else
      umma_commit(bar);
    mbar_wait(bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    atomicExch(&done, 1);
  }
  if (BG && threadIdx.x == 32) {  // background bulk copies until the MMAs finish
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int it = 0;
    while (atomicAdd(&done, 0) == 0 && it < (1 << 20)) {
      const int sl = it & 7;
      if (it >= 8) {
        mbar_wait(&rbar[sl], ph[sl]);
        ph[sl] ^= 1;
      }
      mbar_arrive_expect_tx(&rbar[sl], 16384);
      bulk_load_g2s(ring + sl * 16384, src + ((blockIdx.x * 8 + it) & 127) * 16384, 16384, &rbar[sl]);
      ++it;
    }
    for (int j = it - 8 > 0 ? it - 8 : 0; j < it; ++j) {  // drain
      const int sl = j & 7;
      mbar_wait(&rbar[sl], ph[sl]);
      ph[sl] ^= 1;
    }
  }
  if (pair && threadIdx.x == 0 && rank == 1) mbar_wait(bar, 0);
  tc_fence_before();
  if (pair)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) {
    if (pair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      tmem_dealloc(tmem, 512);
  }
}

template <int KIND, int N, int BG>
void run(const char* name, long long macs_per_mma) {
  const int smem = 1024 + (128 + 256) * 128 + 1024 + 8 * 16384;
  auto k = umma_rate<KIND, N, BG>;
  static uint8_t* src = nullptr;
  if (!src) {
    cudaMalloc(&src, 2 << 20);
    cudaMemset(src, 0, 2 << 20);
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d = nullptr;
  cudaMalloc(&d, sizeof(long long) * sms);
  cudaMemset(d, 0, sizeof(long long) * sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = KIND == 2 ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, d, (const uint8_t*)src, (int*)nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cpm = (double)mx / R;
  // MACs per SM per clock: a pair MMA covers two SMs
  const double mac_clk = (double)macs_per_mma / cpm / (KIND == 2 ? 2 : 1);
  printf("%-22s bg=%d %7.1f clk/MMA  %7.0f MAC/clk/SM  (%s)\n", name, BG, cpm, mac_clk, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 128, 0>("tf32 M128 N128 K8", 128LL * 128 * 8);
  run<0, 128, 1>("tf32 M128 N128 K8", 128LL * 128 * 8);
  run<0, 256, 0>("tf32 M128 N256 K8", 128LL * 256 * 8);
  run<0, 256, 1>("tf32 M128 N256 K8", 128LL * 256 * 8);
  run<2, 256, 0>("tf32 M256 N256 K8 pair", 256LL * 256 * 8);
  run<2, 256, 1>("tf32 M256 N256 K8 pair", 256LL * 256 * 8);
  run<1, 256, 0>("bf16 M128 N256 K16", 128LL * 256 * 16);
  run<1, 256, 1>("bf16 M128 N256 K16", 128LL * 256 * 16);
  run<1, 128, 1>("bf16 M128 N128 K16", 128LL * 128 * 16);
  return 0;
}
