// K1: gate logits + top-k + residency remap (route_token) + gate weights.
//
// bf16 activations: a block of 128 tokens x all E experts is one small GEMM
// (x[128 x d] . wg[E x d]^T) on mma.sync.m16n8k16 (bf16 in, fp32 out): the
// op is HBM-bound on reading x once (d*2 bytes per token), so the legacy
// tensor path is enough to keep the FFMA pipe out of the way; x and wg
// k-chunks are double-buffered in XOR-swizzled shared memory by cp.async.
// fp32 activations (config 1) use a warp-per-token FFMA dot product.
//
// The routing epilogue runs one thread per token on the logits row in shared
// memory and restates the reference exactly:
//   top-k        descending logit, ascending index on ties
//   route_token  first resident gate choice; else the resident expert with the
//                highest layer score, smallest index on ties; empty scores ->
//                smallest resident (expert_store.cpp:206-220)
//   forced miss  no resident expert -> {choice0, -1, miss} (engine.cpp:533-537)
// plus the builder-defined k-slot served set and weights.
// Per-block expert counts feed the deterministic permutation (permute.cu).
#include "common.cuh"
#include "kernels.h"
#include "route_tail.cuh"

namespace emoe {

namespace {

using routing::load_route_state;
using routing::route_one_token;
using routing::route_tail;
using routing::SharedRouteState;

constexpr int RT = kRouteBlockTokens;  // 128 tokens per block
constexpr int KC = 64;                 // k chunk (one 128-B row of bf16)
constexpr int MAX_E = routing::MAX_E;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// XOR-swizzled [rows][64] bf16 tile: 16-B chunk c of row r lives at chunk c ^ (r & 7)
__device__ __forceinline__ uint32_t swz(int r, int chunk) { return r * 128 + ((chunk ^ (r & 7)) << 4); }

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// logits-bias mode: tile[r][e] += bias[t0 + r][e] (coalesced over the tile)
__device__ void add_bias_tile(float* tile, int ld, int64_t t0, const RouteArgs& a) {
  __syncthreads();  // every thread's logits are in the tile
  const int64_t rows = min((int64_t)RT, a.T - t0);
  for (int64_t i = threadIdx.x; i < rows * a.E; i += blockDim.x) {
    const int r = (int)(i / a.E), e = (int)(i % a.E);
    tile[r * ld + e] += __ldg(a.bias + t0 * a.E + i);
  }
}

// block's logits tile [rows][ld] in shared memory -> global [T][E], coalesced
__device__ void store_logits_tile(const float* tile, int ld, int64_t t0, const RouteArgs& a, const RouteOut& o) {
  if (!o.logits) return;
  const int64_t rows = min((int64_t)RT, a.T - t0);
  for (int64_t i = threadIdx.x; i < rows * a.E; i += blockDim.x) {
    const int r = (int)(i / a.E), e = (int)(i % a.E);
    o.logits[t0 * a.E + i] = tile[r * ld + e];
  }
}

__device__ void flush_block_counts(const RouteArgs& a, const RouteOut& o, SharedRouteState& st) {
  __syncthreads();
  if (o.block_counts)
    for (int e = threadIdx.x; e < a.E; e += blockDim.x) o.block_counts[(int64_t)blockIdx.x * a.E + e] = st.counts[e];
}

// ---------------------------------------------------------------------------
// bf16: mma.sync gate.  NT = number of 8-expert column tiles (E <= 8*NT).
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(128) gate_route_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ wg, RouteArgs a,
                                                              RouteOut o) {
  pdl_wait();
  pdl_trigger();
  constexpr int EP = NT * 8;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* xs = smem;                      // [2][RT][64] bf16
  uint8_t* ws = smem + 2 * RT * 128;       // [2][EP][64] bf16
  float* logits = reinterpret_cast<float*>(smem);  // reused after the K loop: [RT][EP+1]
  __shared__ SharedRouteState st;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int64_t t0 = (int64_t)blockIdx.x * RT;
  const int d = a.d;
  const int nk = d / KC;

  auto issue = [&](int kc, int buf) {
    uint8_t* xb = xs + buf * RT * 128;
    uint8_t* wb = ws + buf * EP * 128;
    for (int i = tid; i < RT * 8; i += 128) {
      const int r = i >> 3, c = i & 7;
      const int64_t t = t0 + r;
      const bool ok = t < a.T;
      cp_async16(xb + swz(r, c), x + (ok ? t : 0) * d + kc * KC + c * 8, ok);
    }
    for (int i = tid; i < EP * 8; i += 128) {
      const int r = i >> 3, c = i & 7;
      const bool ok = r < a.E;
      cp_async16(wb + swz(r, c), wg + (int64_t)(ok ? r : 0) * d + kc * KC + c * 8, ok);
    }
    cp_async_commit();
  };

  float acc[2][NT][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.0f;

  issue(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      issue(kc + 1, (kc + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t xb = smem_u32(xs + (kc & 1) * RT * 128);
    const uint32_t wb = smem_u32(ws + (kc & 1) * EP * 128);
#pragma unroll
    for (int ks = 0; ks < KC / 16; ++ks) {
      uint32_t af[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r = warp * 32 + mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int ch = ks * 2 + (lane >> 4);
        ldmatrix_x4(xb + swz(r, ch), af[mt][0], af[mt][1], af[mt][2], af[mt][3]);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t b0, b1;
        const int r = nt * 8 + (lane & 7);
        const int ch = ks * 2 + ((lane >> 3) & 1);
        ldmatrix_x2(wb + swz(r, ch), b0, b1);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) mma_bf16_16816(acc[mt][nt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], b0, b1);
      }
    }
    __syncthreads();
  }

  // accumulators -> logits tile in shared memory (stage buffers are free now)
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int r = warp * 32 + mt * 16 + g;
      const int c = nt * 8 + q * 2;
      logits[r * (EP + 1) + c] = acc[mt][nt][0];
      logits[r * (EP + 1) + c + 1] = acc[mt][nt][1];
      logits[(r + 8) * (EP + 1) + c] = acc[mt][nt][2];
      logits[(r + 8) * (EP + 1) + c + 1] = acc[mt][nt][3];
    }
  if (a.bias) add_bias_tile(logits, EP + 1, t0, a);
  load_route_state(st, a);  // contains __syncthreads
  store_logits_tile(logits, EP + 1, t0, a, o);
  // thread per token: with the logits tile in shared memory even E = 128 costs
  // only a few microseconds here (the mma.sync gate above is the cost for large E)
  const int64_t t = t0 + tid;
  if (t < a.T) route_one_token(logits + tid * (EP + 1), t, a, o, st);
  flush_block_counts(a, o, st);
}

// ---------------------------------------------------------------------------
// fp32: warp-per-token FFMA gate, logits staged in shared memory
// ---------------------------------------------------------------------------
// fp32 gate (config 1): 16 warps per 128-token block, 8 tokens per warp; each
// lane keeps 8 experts' partial dot products over float4 slices of x and W_g
// (x row read once per 8 experts), then a warp reduction per expert.
constexpr int F32_GATE_THREADS = 512;
__global__ void __launch_bounds__(F32_GATE_THREADS) gate_route_f32_kernel(const float* __restrict__ x,
                                                                          const float* __restrict__ wg, RouteArgs a,
                                                                          RouteOut o) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t smem[];
  float* logits = reinterpret_cast<float*>(smem);  // [RT][E]
  __shared__ SharedRouteState st;
  constexpr int NW = F32_GATE_THREADS / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t0 = (int64_t)blockIdx.x * RT;
  const bool vec = (a.d & 3) == 0;
  for (int r = warp; r < RT; r += NW) {
    const int64_t t = t0 + r;
    if (t >= a.T) break;
    const float* xr = x + t * a.d;
    for (int e0 = 0; e0 < a.E; e0 += 8) {
      const int ne = min(8, a.E - e0);
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (vec) {
        for (int i = lane * 4; i < a.d; i += 128) {
          const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + i));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < ne) {
              const float4 wv = __ldg(reinterpret_cast<const float4*>(wg + (int64_t)(e0 + j) * a.d + i));
              acc[j] = fmaf(xv.x, wv.x, acc[j]);
              acc[j] = fmaf(xv.y, wv.y, acc[j]);
              acc[j] = fmaf(xv.z, wv.z, acc[j]);
              acc[j] = fmaf(xv.w, wv.w, acc[j]);
            }
          }
        }
      } else {
        for (int i = lane; i < a.d; i += 32) {
          const float xv = xr[i];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < ne) acc[j] = fmaf(xv, wg[(int64_t)(e0 + j) * a.d + i], acc[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v = acc[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0 && j < ne) logits[r * a.E + e0 + j] = v;
      }
    }
  }
  if (a.bias) add_bias_tile(logits, a.E, t0, a);
  load_route_state(st, a);
  store_logits_tile(logits, a.E, t0, a, o);
  const int64_t t = t0 + threadIdx.x;
  if (threadIdx.x < RT && t < a.T) route_one_token(logits + threadIdx.x * a.E, t, a, o, st);
  flush_block_counts(a, o, st);
}

// fp32 gate logits only, one warp per token (small T: the fused kernel above
// has one block per 128 tokens, too few blocks to cover the GPU), followed by
// route_from_logits_kernel.  Same dot-product order as the fused kernel.
// blockIdx.y selects a slice of the experts (each expert's sum is computed
// in the same order whatever the slicing), so small T still spans the GPU.
// one token's logits over the experts of this block's column slice (a warp)
__device__ void gate_logits_f32_token(const float* __restrict__ x, const float* __restrict__ wg, int64_t t, int d,
                                      int E, float* __restrict__ logits, const float* __restrict__ bias, int lane) {
  const float* xr = x + t * d;
  const bool vec = (d & 3) == 0;
  const int e_beg = E * blockIdx.y / gridDim.y, e_end = E * (blockIdx.y + 1) / gridDim.y;
  for (int e0 = e_beg; e0 < e_end; e0 += 8) {
    const int ne = min(8, e_end - e0);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (vec) {
      // four 128-element slices per round, every load issued before the FMAs
      // (a latency-bound loop at small T: ~1 round trip per 512 elements)
      int i = lane * 4;
      for (; i + 3 * 128 < d; i += 4 * 128) {
        float4 xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = __ldg(reinterpret_cast<const float4*>(xr + i + u * 128));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < ne) {
            float4 wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              wv[u] = __ldg(reinterpret_cast<const float4*>(wg + (int64_t)(e0 + j) * d + i + u * 128));
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              acc[j] = fmaf(xv[u].x, wv[u].x, acc[j]);
              acc[j] = fmaf(xv[u].y, wv[u].y, acc[j]);
              acc[j] = fmaf(xv[u].z, wv[u].z, acc[j]);
              acc[j] = fmaf(xv[u].w, wv[u].w, acc[j]);
            }
          }
        }
      }
      for (; i < d; i += 128) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + i));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < ne) {
            const float4 wv = __ldg(reinterpret_cast<const float4*>(wg + (int64_t)(e0 + j) * d + i));
            acc[j] = fmaf(xv.x, wv.x, acc[j]);
            acc[j] = fmaf(xv.y, wv.y, acc[j]);
            acc[j] = fmaf(xv.z, wv.z, acc[j]);
            acc[j] = fmaf(xv.w, wv.w, acc[j]);
          }
        }
      }
    } else {
      for (int i = lane; i < d; i += 32) {
        const float xv = xr[i];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < ne) acc[j] = fmaf(xv, wg[(int64_t)(e0 + j) * d + i], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = acc[j];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0 && j < ne) logits[t * E + e0 + j] = bias ? v + bias[t * E + e0 + j] : v;
    }
  }
}

// With a.sync set, the blocks covering one 128-token route block count in
// on a.sync[route block] and the last of them routes its tokens (the logits
// of the other blocks read through L2), so the small-T gate is one launch.
__global__ void __launch_bounds__(256) gate_logits_f32_kernel(const float* __restrict__ x,
                                                              const float* __restrict__ wg, int64_t T, int d, int E,
                                                              float* __restrict__ logits,
                                                              const float* __restrict__ bias, RouteArgs a,
                                                              RouteOut o) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * 8 + warp;
  if (t < T) gate_logits_f32_token(x, wg, t, d, E, logits, bias, lane);
  if (!a.sync) return;
  __shared__ SharedRouteState st;
  __shared__ int is_last;
  extern __shared__ float s_rows[];  // [RT][E + 1]: the route block's logits
  constexpr int XB = RT / 8;         // x blocks per route block
  const int rb = blockIdx.x / XB;
  const int members = min(XB, (int)gridDim.x - rb * XB) * (int)gridDim.y;
  __syncthreads();  // this block's logits are stored
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(a.sync + rb, 1) == members - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int64_t t0 = (int64_t)rb * RT;
  const int rows = (int)min((int64_t)RT, T - t0);
  for (int i = threadIdx.x; i < rows * E; i += blockDim.x) {
    const int r = i / E;
    s_rows[r * (E + 1) + (i - r * E)] = __ldcg(logits + t0 * E + i);
  }
  load_route_state(st, a);  // its barriers also publish s_rows
  if (threadIdx.x < rows) route_one_token(s_rows + threadIdx.x * (E + 1), t0 + threadIdx.x, a, o, st);
  __syncthreads();
  if (o.block_counts)
    for (int e = threadIdx.x; e < E; e += blockDim.x) o.block_counts[(int64_t)rb * E + e] = st.counts[e];
  if (threadIdx.x == 0) a.sync[rb] = 0;  // for the next launch (stream-ordered)
}


// ---------------------------------------------------------------------------
// routing-driven mode: logits supplied by the caller
// ---------------------------------------------------------------------------
// Routing from precomputed logits.  Many experts (E >= 32): the block's 128
// logits rows are staged in shared memory (row pitch E + 1 floats, so the
// per-thread row scans are bank-conflict free) and every thread routes its own
// token from its row — the same serial top-k / softmax order as the
// reference, ~4 instructions per logit.  The staging keeps 8 coalesced 16-B
// loads per thread in flight (a load -> st.shared loop: 31 -> 26 us at the
// Switch shape; 4-B cp.async per element and four threads per token with a
// quad-parallel argmax / expf were both slower).
__global__ void __launch_bounds__(RT) route_from_logits_kernel(const float* __restrict__ logits, RouteArgs a,
                                                               RouteOut o) {
  pdl_wait();
  pdl_trigger();
  __shared__ SharedRouteState st;
  extern __shared__ float s_rows[];  // [RT][E + 1] when E >= 32
  const int64_t t0 = (int64_t)blockIdx.x * RT;
  const int rows = (int)min((int64_t)RT, a.T - t0);
  const float* src = logits + t0 * a.E;
  if (o.logits && o.logits != logits)
    for (int64_t i = threadIdx.x; i < (int64_t)rows * a.E; i += blockDim.x) o.logits[t0 * a.E + i] = src[i];
  const float* lg = src + (int64_t)threadIdx.x * a.E;
  if (a.E >= 32 || a.bias) {
    const int ld = a.E + 1, n = rows * a.E;
    if ((a.E & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      constexpr int U = 8;  // 16-B loads in flight per thread before the shared stores
      const float4* src4 = reinterpret_cast<const float4*>(src);
      for (int i0 = threadIdx.x; i0 < n / 4; i0 += RT * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * RT < n / 4) v[u] = __ldg(src4 + i0 + u * RT);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * RT;
          if (i >= n / 4) break;
          const int r = (4 * i) / a.E, c = 4 * i - r * a.E;
          float* d = s_rows + r * ld + c;
          d[0] = v[u].x;
          d[1] = v[u].y;
          d[2] = v[u].z;
          d[3] = v[u].w;
        }
      }
    } else {
      for (int i = threadIdx.x; i < n; i += RT) {
        const int r = i / a.E;
        s_rows[r * ld + (i - r * a.E)] = __ldg(src + i);
      }
    }
    lg = s_rows + threadIdx.x * ld;
    if (a.bias) {  // logits-bias mode: the staged rows get the bias, and the workspace the sum
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += RT) {
        const int r = i / a.E, c = i - r * a.E;
        const float v = s_rows[r * ld + c] + __ldg(a.bias + t0 * a.E + i);
        s_rows[r * ld + c] = v;
        if (o.logits) o.logits[t0 * a.E + i] = v;
      }
    }
  }
  load_route_state(st, a);  // its barriers also publish s_rows
  if (threadIdx.x < rows) route_one_token(lg, t0 + threadIdx.x, a, o, st);
  flush_block_counts(a, o, st);
}

// route_token over caller-supplied ranked gate choices [T][k]
__global__ void __launch_bounds__(128) route_from_choices_kernel(const int32_t* __restrict__ choices, RouteArgs a,
                                                                 RouteOut o) {
  __shared__ SharedRouteState st;
  load_route_state(st, a);
  const int64_t t = (int64_t)blockIdx.x * RT + threadIdx.x;
  if (t < a.T) {
    int ti[8];
    for (int r = 0; r < a.k; ++r) ti[r] = choices[t * a.k + r];
    route_tail(ti, nullptr, t, a, o, st);
  }
  flush_block_counts(a, o, st);
}

}  // namespace

void launch_route_from_choices(const int32_t* choices, const RouteArgs& a, const RouteOut& o, cudaStream_t s) {
  EMOE_REQUIRE(a.E >= 1 && a.E <= MAX_E, "route: num_experts must be in [1, 128]");
  EMOE_REQUIRE(a.k >= 1 && a.k <= 8, "route: top_k must be in [1, 8]");
  const int nblocks = (int)ceil_div(a.T, RT);
  if (nblocks == 0) return;
  route_from_choices_kernel<<<nblocks, RT, 0, s>>>(choices, a, o);
  EMOE_CUDA(cudaGetLastError());
    count_launch();
}

void launch_gate_route(const void* x, const void* wg, int dtype, const RouteArgs& a, const RouteOut& o,
                       cudaStream_t s) {
  EMOE_REQUIRE(a.E >= 1 && a.E <= MAX_E, "route: num_experts must be in [1, 128]");
  EMOE_REQUIRE(a.k >= 1 && a.k <= 8 && a.k <= a.E, "route: top_k must be in [1, min(8, E)]");
  const int nblocks = (int)ceil_div(a.T, RT);
  if (nblocks == 0) return;
  if (dtype == DT_F32 && o.logits && nblocks < 74) {
    // small T: logits with one warp per token over the whole GPU, then routing
    const int nbx = (int)ceil_div(a.T, 8);
    const int ny = std::max(1, std::min((2 * 148 + nbx - 1) / nbx, (a.E + 1) / 2));  // >= 2 experts per warp
    RouteArgs ra = a;
    ra.bias = nullptr;  // added to the logits by the gate
    const size_t smem = a.sync ? (size_t)RT * (a.E + 1) * sizeof(float) : 0;
    if (smem > 48 * 1024) ensure_max_dynamic_smem(reinterpret_cast<const void*>(gate_logits_f32_kernel), (int)smem);
    EMOE_CUDA(launch_pdl(gate_logits_f32_kernel, dim3(nbx, ny), dim3(256), smem, s, 1, static_cast<const float*>(x),
                         static_cast<const float*>(wg), a.T, a.d, a.E, o.logits, a.bias, ra, o));
    count_launch();
    if (!a.sync) launch_route_from_logits(o.logits, ra, o, s);  // routing in its own kernel
    return;
  } else if (dtype == DT_F32) {
    const size_t smem = (size_t)RT * a.E * sizeof(float);
    EMOE_REQUIRE(smem <= 48 * 1024, "route: fp32 logits tile exceeds 48 KB");
    EMOE_CUDA(launch_pdl(gate_route_f32_kernel, dim3(nblocks), dim3(F32_GATE_THREADS), smem, s, 1,
                         static_cast<const float*>(x), static_cast<const float*>(wg), a, o));
  } else {
    EMOE_REQUIRE(a.d % KC == 0, "route: d_model must be a multiple of 64 for bf16");
    const int nt = (a.E + 7) / 8;
    auto go = [&](auto kernel, int NTv) {
      const int EP = NTv * 8;
      size_t smem = (size_t)2 * RT * 128 + (size_t)2 * EP * 128;
      const size_t lsm = (size_t)RT * (EP + 1) * sizeof(float);
      if (lsm > smem) smem = lsm;
      ensure_max_dynamic_smem(reinterpret_cast<const void*>(kernel), (int)smem);
      EMOE_CUDA(launch_pdl(kernel, dim3(nblocks), dim3(128), smem, s, 1, static_cast<const __nv_bfloat16*>(x),
                           static_cast<const __nv_bfloat16*>(wg), a, o));
    };
    if (nt <= 1)
      go(gate_route_bf16_kernel<1>, 1);
    else if (nt <= 2)
      go(gate_route_bf16_kernel<2>, 2);
    else if (nt <= 4)
      go(gate_route_bf16_kernel<4>, 4);
    else if (nt <= 8)
      go(gate_route_bf16_kernel<8>, 8);
    else
      go(gate_route_bf16_kernel<16>, 16);
  }
  EMOE_CUDA(cudaGetLastError());
    count_launch();
}

void launch_route_from_logits(const float* logits, const RouteArgs& a, const RouteOut& o, cudaStream_t s) {
  EMOE_REQUIRE(a.E >= 1 && a.E <= MAX_E, "route: num_experts must be in [1, 128]");
  EMOE_REQUIRE(a.k >= 1 && a.k <= 8 && a.k <= a.E, "route: top_k must be in [1, min(8, E)]");
  const int nblocks = (int)ceil_div(a.T, RT);
  if (nblocks == 0) return;
  const int smem = a.E >= 32 || a.bias ? RT * (a.E + 1) * (int)sizeof(float) : 0;
  if (smem > 48 * 1024) ensure_max_dynamic_smem(reinterpret_cast<const void*>(route_from_logits_kernel), smem);
  EMOE_CUDA(launch_pdl(route_from_logits_kernel, dim3(nblocks), dim3(RT), (size_t)smem, s, 1, logits, a, o));
  EMOE_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace emoe
