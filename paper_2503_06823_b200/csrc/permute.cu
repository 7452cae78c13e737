// K3 (scan + stable permute/gather) and K5 (gate-weighted combine).
//
// Permutation contract (builder-defined, restated in
// oracle_permute): expert e owns rows [off_e, off_e + pad_up(n_e)) of X_perm;
// the served pair (t, e) lands at off_e + #{t' < t : e in served(t')}, i.e. the
// segment is stable in token order.  No atomics decide positions, so the
// layout is bit-reproducible and identical to the CPU oracle.
//
// Data movement: x is read once (one warp per token, 16-byte vectors) and
// written to each of its <= k destinations; the combine reads each served row
// of Y once and writes y once, accumulating in fp32 in slot order.
#include "common.cuh"
#include "kernels.h"

namespace emoe {

namespace {

constexpr int RT = kRouteBlockTokens;

// One thread per expert walks the per-block counts in block order.
__global__ void scan_kernel(const int32_t* __restrict__ block_counts, int nblocks, int E, int pad,
                            int32_t* __restrict__ counts, int64_t* __restrict__ seg_offsets,
                            int64_t* __restrict__ block_base) {
  __shared__ int64_t totals[1024];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t run = 0;
    for (int b = 0; b < nblocks; ++b) {
      block_base[(int64_t)b * E + e] = run;
      run += block_counts[(int64_t)b * E + e];
    }
    totals[e] = run;
    counts[e] = (int32_t)run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int e = 0; e < E; ++e) {
      seg_offsets[e] = off;
      off += (totals[e] + pad - 1) / pad * pad;
    }
    seg_offsets[E] = off;
  }
}

// Block = 128 tokens (the route kernel's blocks), 4 warps x 32 tokens.
__global__ void __launch_bounds__(128) permute_kernel(const uint8_t* __restrict__ x, int row_bytes, int64_t T, int E,
                                                      int k, const int32_t* __restrict__ served_idx,
                                                      const int64_t* __restrict__ seg_offsets,
                                                      const int64_t* __restrict__ block_base,
                                                      uint8_t* __restrict__ x_perm, int32_t* __restrict__ pos,
                                                      int32_t* __restrict__ row_token) {
  extern __shared__ int32_t warp_counts[];  // [4][E]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * RT + threadIdx.x;
  const bool valid = t < T;
  int my[8];
  for (int j = 0; j < k; ++j) my[j] = valid ? served_idx[t * k + j] : -1;
  const uint32_t lt = (1u << lane) - 1u;
  int rank[8];
  for (int j = 0; j < k; ++j) rank[j] = 0;
  // per expert: lanes (tokens) that serve it; a token serves an expert at most once
  for (int e = 0; e < E; ++e) {
    bool has = false;
    for (int j = 0; j < k; ++j) has |= (my[j] == e);
    const uint32_t m = __ballot_sync(0xffffffffu, has);
    if (m == 0) {
      if (lane == 0) warp_counts[warp * E + e] = 0;
      continue;
    }
    if (lane == 0) warp_counts[warp * E + e] = __popc(m);
    if (has)
      for (int j = 0; j < k; ++j)
        if (my[j] == e) rank[j] = __popc(m & lt);
  }
  __syncthreads();
  int32_t dst[8];
  for (int j = 0; j < k; ++j) {
    const int e = my[j];
    if (e < 0) {
      dst[j] = -1;
      continue;
    }
    int64_t base = seg_offsets[e] + block_base[(int64_t)blockIdx.x * E + e];
    for (int w = 0; w < warp; ++w) base += warp_counts[w * E + e];
    dst[j] = (int32_t)(base + rank[j]);
  }
  if (valid)
    for (int j = 0; j < k; ++j) {
      if (pos) pos[t * k + j] = dst[j];
      if (row_token && dst[j] >= 0) row_token[dst[j]] = (int32_t)t;
    }
  // gather: the warp copies its 32 tokens' rows, 16 B per lane per step
  const int nvec = row_bytes / 16;
  for (int i = 0; i < 32; ++i) {
    const int64_t tt = (int64_t)blockIdx.x * RT + warp * 32 + i;
    if (tt >= T) break;
    int32_t d_i[8];
    int nd = 0;
    for (int j = 0; j < k; ++j) {
      const int32_t v = __shfl_sync(0xffffffffu, dst[j], i);
      if (v >= 0) d_i[nd++] = v;
    }
    if (nd == 0) continue;
    const uint4* src = reinterpret_cast<const uint4*>(x + tt * row_bytes);
    for (int v = lane; v < nvec; v += 32) {
      const uint4 val = __ldg(src + v);
      for (int q = 0; q < nd; ++q) reinterpret_cast<uint4*>(x_perm + (int64_t)d_i[q] * row_bytes)[v] = val;
    }
  }
}

// One warp per token; lanes own 16-byte column chunks.
__global__ void __launch_bounds__(256) combine_bf16_kernel(const __nv_bfloat16* __restrict__ Y, int64_t T, int d,
                                                           int k, const int32_t* __restrict__ pos,
                                                           const float* __restrict__ served_w,
                                                           __nv_bfloat16* __restrict__ y) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  if (t >= T) return;
  int32_t p[8];
  float w[8];
  for (int j = 0; j < k; ++j) {
    p[j] = pos[t * k + j];
    w[j] = served_w[t * k + j];
  }
  const int nvec = d / 8;
  for (int v = lane; v < nvec; v += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < k; ++j) {
      if (p[j] < 0) continue;
      const uint4 r = __ldg(reinterpret_cast<const uint4*>(Y + (int64_t)p[j] * d) + v);
      const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[2 * q] += w[j] * bf16_lo(u[q]);
        acc[2 * q + 1] += w[j] * bf16_hi(u[q]);
      }
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    reinterpret_cast<uint4*>(y + t * d)[v] = o;
  }
}

__global__ void __launch_bounds__(256) combine_f32_kernel(const float* __restrict__ Y, int64_t T, int d, int k,
                                                          const int32_t* __restrict__ pos,
                                                          const float* __restrict__ served_w, float* __restrict__ y) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  if (t >= T) return;
  int32_t p[8];
  float w[8];
  for (int j = 0; j < k; ++j) {
    p[j] = pos[t * k + j];
    w[j] = served_w[t * k + j];
  }
  const int nvec = d / 4;
  for (int v = lane; v < nvec; v += 32) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int j = 0; j < k; ++j) {
      if (p[j] < 0) continue;
      const float4 r = __ldg(reinterpret_cast<const float4*>(Y + (int64_t)p[j] * d) + v);
      acc.x += w[j] * r.x;
      acc.y += w[j] * r.y;
      acc.z += w[j] * r.z;
      acc.w += w[j] * r.w;
    }
    reinterpret_cast<float4*>(y + t * d)[v] = acc;
  }
}

}  // namespace

void launch_scan(const int32_t* block_counts, int nblocks, int E, int pad, int32_t* counts, int64_t* seg_offsets,
                 int64_t* block_base, cudaStream_t s) {
  EMOE_REQUIRE(E <= 1024, "scan: too many experts");
  scan_kernel<<<1, 256, 0, s>>>(block_counts, nblocks, E, pad, counts, seg_offsets, block_base);
  EMOE_CUDA(cudaGetLastError());
    count_launch();
}

void launch_permute(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                    const int64_t* seg_offsets, const int64_t* block_base, void* x_perm, int32_t* pos,
                    int32_t* row_token, cudaStream_t s) {
  const int row_bytes = d * elem_bytes;
  EMOE_REQUIRE(row_bytes % 16 == 0, "permute: row bytes must be a multiple of 16");
  const int nblocks = (int)ceil_div(T, RT);
  if (nblocks == 0) return;
  permute_kernel<<<nblocks, RT, 4 * E * sizeof(int32_t), s>>>(
      static_cast<const uint8_t*>(x), row_bytes, T, E, k, served_idx, seg_offsets, block_base,
      static_cast<uint8_t*>(x_perm), pos, row_token);
  EMOE_CUDA(cudaGetLastError());
    count_launch();
}

void launch_combine(const void* Y, int dtype, int64_t T, int d, int k, const int32_t* pos, const float* served_w,
                    void* y, cudaStream_t s) {
  const int nblocks = (int)ceil_div(T, 8);
  if (nblocks == 0) return;
  if (dtype == DT_F32) {
    EMOE_REQUIRE(d % 4 == 0, "combine: d must be a multiple of 4");
    combine_f32_kernel<<<nblocks, 256, 0, s>>>(static_cast<const float*>(Y), T, d, k, pos, served_w,
                                               static_cast<float*>(y));
  } else {
    EMOE_REQUIRE(d % 8 == 0, "combine: d must be a multiple of 8");
    combine_bf16_kernel<<<nblocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(Y), T, d, k, pos, served_w,
                                                static_cast<__nv_bfloat16*>(y));
  }
  EMOE_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace emoe
