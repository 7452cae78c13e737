// K4, fp32 configuration (BASELINE config 1: fp32 weights, 1e-5 tolerance).
//
// TF32 tensor cores cannot meet a 1e-5 relative tolerance, so the fp32 grouped
// FFN runs on the FFMA pipe: 64 x 64 output tiles, 16-deep k slices staged in
// shared memory, 4 x 4 register micro-tiles per thread (8 x 4 x 4 for SwiGLU's
// paired W1/W3 accumulators).  Same padded-segment grouping and epilogues as
// the tcgen05 kernel (grouped_gemm.cu).
#include "common.cuh"
#include "kernels.h"

namespace emoe {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <int EPI>
__global__ void __launch_bounds__(256) grouped_gemm_f32_kernel(const float* __restrict__ A, int64_t lda,
                                                               const float* __restrict__ B,
                                                               const float* __restrict__ B2,
                                                               const int64_t* __restrict__ seg,
                                                               const int32_t* __restrict__ slot_of_expert, int E,
                                                               int K, int b_rows_per_slot, float* __restrict__ out,
                                                               int64_t ldo, const int32_t* __restrict__ seg_expert) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  __shared__ float B2s[EPI == EPI_SWIGLU ? TK : 1][TN + 4];
  const int64_t row0 = (int64_t)blockIdx.y * TM;
  if (row0 >= seg[E]) return;
  int e = 0;
  while (e + 1 < E && seg[e + 1] <= row0) ++e;
  const int slot = slot_of_expert[seg_expert ? seg_expert[e] : e];
  const int n0 = blockIdx.x * TN;
  const float* Bp = B + ((int64_t)slot * b_rows_per_slot + n0) * K;
  const float* B2p = EPI == EPI_SWIGLU ? B2 + ((int64_t)slot * b_rows_per_slot + n0) * K : nullptr;
  const float* Ap = A + row0 * lda;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int lr = tid / 4, lk = (tid % 4) * 4;
  float acc[4][4] = {};
  float acc2[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    const float4 av = *reinterpret_cast<const float4*>(Ap + (int64_t)lr * lda + k0 + lk);
    As[lk + 0][lr] = av.x;
    As[lk + 1][lr] = av.y;
    As[lk + 2][lr] = av.z;
    As[lk + 3][lr] = av.w;
    const float4 bv = *reinterpret_cast<const float4*>(Bp + (int64_t)lr * K + k0 + lk);
    Bs[lk + 0][lr] = bv.x;
    Bs[lk + 1][lr] = bv.y;
    Bs[lk + 2][lr] = bv.z;
    Bs[lk + 3][lr] = bv.w;
    if (EPI == EPI_SWIGLU) {
      const float4 cv = *reinterpret_cast<const float4*>(B2p + (int64_t)lr * K + k0 + lk);
      B2s[lk + 0][lr] = cv.x;
      B2s[lk + 1][lr] = cv.y;
      B2s[lk + 2][lr] = cv.z;
      B2s[lk + 3][lr] = cv.w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      if (EPI == EPI_SWIGLU) {
        float c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = B2s[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc2[i][j] = fmaf(a[i], c[j], acc2[i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float g = acc[i][j];
      if (EPI == EPI_SWIGLU)
        v[j] = g / (1.0f + expf(-g)) * acc2[i][j];
      else if (EPI == EPI_RELU)
        v[j] = fmaxf(g, 0.0f);
      else
        v[j] = g;
    }
    *reinterpret_cast<float4*>(out + (row0 + ty * 4 + i) * ldo + n0 + tx * 4) = make_float4(v[0], v[1], v[2], v[3]);
  }
}

}  // namespace

void launch_grouped_gemm_f32(int epi, const float* A, int64_t lda, const float* B, const float* B2,
                             const int64_t* seg_offsets, const int32_t* slot_of_expert, int num_experts, int K,
                             int N_out, int b_rows_per_slot, int64_t rows_cap, float* out, int64_t ldo,
                             cudaStream_t stream, const int32_t* seg_expert) {
  EMOE_REQUIRE(K % TK == 0 && N_out % TN == 0, "grouped_gemm_f32: K % 16 and N % 64 must be 0");
  const int64_t rb = ceil_div(rows_cap, TM);
  if (rb == 0) return;
  dim3 grid(N_out / TN, (unsigned)rb);
  if (epi == EPI_SWIGLU)
    grouped_gemm_f32_kernel<EPI_SWIGLU><<<grid, 256, 0, stream>>>(
        A, lda, B, B2, seg_offsets, slot_of_expert, num_experts, K, b_rows_per_slot, out, ldo, seg_expert);
  else if (epi == EPI_RELU)
    grouped_gemm_f32_kernel<EPI_RELU><<<grid, 256, 0, stream>>>(
        A, lda, B, B2, seg_offsets, slot_of_expert, num_experts, K, b_rows_per_slot, out, ldo, seg_expert);
  else
    grouped_gemm_f32_kernel<EPI_STORE><<<grid, 256, 0, stream>>>(
        A, lda, B, B2, seg_offsets, slot_of_expert, num_experts, K, b_rows_per_slot, out, ldo, seg_expert);
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace emoe
