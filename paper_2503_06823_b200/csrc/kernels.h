// Host-side launchers for the emoe sm_100a kernels (internal interface; the
// public boundary is include/emoe.h).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace emoe {

// number of kernels this library launched (reported by bench.py as gpu_launches)
void count_launch(int n = 1);
long long launch_count();
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device: set it once per
// (device, kernel) before a launch needing more than 48 KB (thread-safe)
void ensure_max_dynamic_smem(const void* func, int bytes);

// Programmatic dependent launch for the kernels of one forward (gate -> scan
// -> permute -> GEMM1 -> GEMM2 -> combine): each is launched with
// programmatic stream serialisation, calls pdl_wait() (common.cuh) before its
// first read of anything a preceding kernel wrote, and pdl_trigger() once it
// is running, so the next kernel's launch and prologue (barrier init, TMEM
// allocation, descriptor prefetch) overlap this one's tail.  Every kernel
// launched this way waits unconditionally, so the ordering stays transitive
// along the chain.  Off by default (EMOE_PDL=1 enables it): measured neutral
// in graph replays and slower in the host-buffer pipeline.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              int cluster, Args&&... args) {
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n++].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = (unsigned)cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n++].val.clusterDim.z = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = (unsigned)n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

enum EpiKind { EPI_SWIGLU = 0, EPI_RELU = 1, EPI_STORE = 2, EPI_F32 = 3 };
enum DType { DT_BF16 = 0, DT_F32 = 1 };

constexpr int kRouteBlockTokens = 128;  // tokens per route / permute block
constexpr int kSegPad = 128;            // per-expert segment padding (GEMM BM)

// Outputs of K1 (any pointer except served_idx / served_w / block_counts may be null).
struct RouteOut {
  float* logits;          // [T][E]
  int32_t* topk_idx;      // [T][k]
  int32_t* route_expert;  // [T]
  int32_t* route_rank;    // [T]
  uint8_t* route_hit;     // [T]
  int32_t* served_idx;    // [T][k], -1 = empty slot
  float* served_w;        // [T][k]
  int32_t* block_counts;  // [ceil(T/128)][E]
};

struct RouteArgs {
  int64_t T;
  int d, E, k;
  int weight_mode;          // 0 softmax over served subset, 1 full softmax prob
  int forced_miss;          // engine.cpp:533-537 behaviour when no expert is resident
  const uint8_t* resident;  // [E] device
  const double* scores;     // [E] device or null (empty score vector)
  int* error_flag;          // device int, set to 3 when a token needs a fallback and no expert is resident
  const float* bias = nullptr;  // [T][E] added to the gate's logits before routing (null: none)
  int32_t* sync = nullptr;      // [ceil(T/128)] zeroed counters: the small-T fp32 gate routes in its
                                // last block per 128-token block (null: logits kernel + routing kernel)
};

// K1 from activations: logits = x . wg^T (bf16 x via mma.sync, fp32 x via FFMA) + routing
void launch_gate_route(const void* x, const void* wg, int dtype, const RouteArgs& a, const RouteOut& o,
                       cudaStream_t s);
// K1 from precomputed logits [T][E] fp32 (routing-driven parity mode)
void launch_route_from_logits(const float* logits, const RouteArgs& a, const RouteOut& o, cudaStream_t s);

// A2 route_token over ranked gate choices [T][k] (no logits; served weights uniform)
void launch_route_from_choices(const int32_t* choices, const RouteArgs& a, const RouteOut& o, cudaStream_t s);

// K3a: per-expert totals, padded segment offsets, per-block bases, -1 in the
// padding rows of row_token (nullable); done = a zeroed device counter
void launch_scan(const int32_t* block_counts, int nblocks, int E, int pad, int32_t* counts,
                 int64_t* seg_offsets, int64_t* block_base, int32_t* row_token, int32_t* done, cudaStream_t s);
// K3a + K3b as one call: for small batches (<= 32 token blocks, E <= 128) the
// scan is folded into the permute kernel (one launch), else scan + permute
void launch_scan_permute(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                         const int32_t* block_counts, int pad, int32_t* counts, int64_t* seg_offsets,
                         int64_t* block_base, void* x_perm, int32_t* pos, int32_t* row_token, int32_t* done,
                         cudaStream_t s, float* x_hi = nullptr, float* x_lo = nullptr);
// K3b: stable permutation + row gather into the padded segments
void launch_permute(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                    const int64_t* seg_offsets, const int64_t* block_base, void* x_perm, int32_t* pos,
                    int32_t* row_token, cudaStream_t s, float* x_hi = nullptr, float* x_lo = nullptr);
// Expert-parallel peer-memory addressing: rank q's receive (or expert-output)
// buffer is base[q] (own buffer or a CUDA-IPC mapping).  This rank's padded
// segment of expert e is cut into pieces, one per computing rank q: local
// rows [piece_end[e][q-1], piece_end[e][q]) go to rank q at receive row
// (local row + piece_shift[e][q]).  Device arrays [E][W].
constexpr int kMaxPeers = 8;
struct PeerRows {
  uint8_t* base[kMaxPeers];
  const int64_t* piece_end;
  const int64_t* piece_shift;
  int W;
  int64_t cap;  // rows per buffer: a row outside [0, cap) is not written (pos = -1)
  int pos_remote = 0;  // pos[t][j] = the destination row (1) or the local row (0)
};
// GEMM2 return form: segment i's output rows go to rank seg_rank[i]'s buffer
// base[seg_rank[i]] at row (r + seg_shift[i]) -- the source's own permuted
// layout -- with NVLink stores from the epilogue (device arrays [n_seg])
struct PeerOut {
  uint8_t* base[kMaxPeers];
  const int32_t* seg_rank;
  const int64_t* seg_shift;
};
// K3b dispatch form: rows go straight to the owning rank's receive buffer;
// pos[t][j] stays the local permuted row (where the pushed output returns)
void launch_permute_remote(const void* x, int elem_bytes, int64_t T, int d, int E, int k, const int32_t* served_idx,
                           const int64_t* seg_offsets, const int64_t* block_base, const PeerRows& peers,
                           int32_t* pos, cudaStream_t s);

// K5: gate-weighted combine in fixed slot order
void launch_combine(const void* Y, int dtype, int64_t T, int d, int k, const int32_t* pos, const float* served_w,
                    void* y, cudaStream_t s);

// K4: tcgen05 grouped GEMM (bf16); cta_group 1 (tile 128x256) or 2 (CTA pair, tile 256x256)
CUtensorMap make_tmap_bf16_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
CUtensorMap make_tmap_bf16_store(const void* base, uint64_t rows, uint64_t cols);  // epilogue store target
// mc = 2: 1-CTA MMAs whose weight tile is multicast over a cluster of 2 CTAs
// on adjacent row blocks (segments padded to 256 rows)
int gemm_tile_m(int cta_group, int mc = 1);             // segment padding the kernel needs
int gemm_b_box_rows(int epi, int cta_group, int mc = 1);  // TMA box rows of the weight operand
struct PeerOut;  // expert parallelism: GEMM2 rows pushed to their source ranks (below)
// top-1 combine fused into GEMM2's epilogue: y[row_token[r]] = weight[token] * Y[r]
struct ScatterCombine {
  const int32_t* row_token;  // [R], -1 = padding row
  const float* weight;       // [T][k] served_w
  __nv_bfloat16* y;          // [T][ldo]
  int k = 1;                 // 1 or 2
  const int32_t* pos = nullptr;  // k = 2: [T][2] rows of the served slots (-1 = not served)
  int32_t* arrive = nullptr;     // k = 2: [T][n_blocks][2] zeroed counters (left zeroed)
};
void launch_grouped_gemm(int epi, int cta_group, int mc, const CUtensorMap& ta, const CUtensorMap& tb,
                         const CUtensorMap& tb2, const int64_t* seg_offsets, const int32_t* slot_of_expert,
                         int num_experts, int K, int N_out, int b_rows_per_slot, __nv_bfloat16* out, int64_t ldo,
                         int num_sms, cudaStream_t stream, const int32_t* seg_expert = nullptr,
                         const CUtensorMap* tmap_out = nullptr,  // null: direct st.global epilogue
                         const ScatterCombine* scatter = nullptr, const PeerOut* peer_out = nullptr,
                         const int64_t* seg_a_shift = nullptr,   // [n_seg] A row shift per segment
                         const int64_t* seg_o_shift = nullptr);  // [n_seg] output row shift per segment

// K1 for many experts (E in {32, 64, 96, 128}, bf16): gate GEMM on tcgen05
// with the routing fused into its epilogue (gate_tc.cu).  tmap_gate: W_g [E][d]
// with box rows gate_tc_box_rows(E, d) (the slice of the gate one CTA
// loads).  store_logits: also write o.logits.
int gate_tc_box_rows(int E, int d);
void launch_gate_route_tc(const CUtensorMap& tmap_x, const CUtensorMap& tmap_gate, const RouteArgs& a,
                          const RouteOut& o, bool store_logits, int num_sms, cudaStream_t s);

// K1 for many experts: the gate as one dense tcgen05 GEMM with fp32 output,
// out[M][ldo] = A[M][K] . B[N_out][K]^T, columns >= col_limit (multiple of 32) not stored
void launch_dense_gemm_f32(const CUtensorMap& ta, const CUtensorMap& tb, int64_t M, int K, int N_out, float* out,
                           int64_t ldo, int col_limit, int num_sms, cudaStream_t stream, int cta_group = 1);

// K4 fp32 path on tensor cores (3xTF32, grouped_gemm_tf32.cu): operands
// pre-split into tf32 hi and fp32 lo parts; tensor maps from make_tmap_f32_2d
// (box = 32 fp32 x box_rows, 128-B swizzle)
struct Tf32Operands {
  CUtensorMap a_hi, a_lo, b_hi, b_lo, b2_hi, b2_lo;  // b2: SwiGLU W3 (else = b)
};
CUtensorMap make_tmap_f32_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
bool gemm_tf32x3_supported(int epi, int K, int N_out);
int gemm_tf32x3_b_box_rows(int epi);
int gemm_tf32x3_cta_group();  // 1: 128 x 128 tiles on one CTA; 2: 256 x 128 tiles on a CTA pair
int gemm_tf32x3_tile_m();     // the segment padding the kernel needs (128 or 256)
// x -> tf32(x) in hi (hi may alias x), x - tf32(x) in lo; n % 4 == 0
// rows_dev (optional): device row count bounding the split to rows * row_elems
void launch_split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s,
                       const int64_t* rows_dev = nullptr, int row_elems = 0);
// split-K scratch for small batches: `rows` = the row capacity of the
// operands, `capacity` floats at `partial`
// Stream-K scratch of the 3xTF32 kernel: one raw partial tile per
// co-resident CTA, and an arrival counter per output tile, zero-initialised
// once (every launch leaves them zero)
struct StreamK {
  float* partial;
  size_t partial_floats;
  int32_t* arrive;
  int64_t arrivals;
};
size_t gemm_tf32x3_partial_floats(int num_sms);
int64_t gemm_tf32x3_arrivals(int epi, int N_out, int64_t rows);
// GEMM1 (SwiGLU/ReLU): out_hi/out_lo = split(H); GEMM2 (STORE): out_hi = Y.
// 1-CTA 128 x 128 tiles or CTA-pair 256 x 128 tiles (segments padded to gemm_tf32x3_tile_m())
void launch_grouped_gemm_tf32x3(int epi, const Tf32Operands& ops, const int64_t* seg_offsets,
                                const int32_t* slot_of_expert, const int32_t* seg_expert, int n_seg, int K, int N_out,
                                int b_rows_per_slot, float* out_hi, float* out_lo, int64_t ldo, int64_t max_rows,
                                const StreamK& sk, cudaStream_t stream);

// K4 fp32 path (SIMT FFMA): same grouping/epilogues, fp32 in/out (shapes the
// 3xTF32 kernel does not tile)
void launch_grouped_gemm_f32(int epi, const float* A, int64_t lda, const float* B, const float* B2,
                             const int64_t* seg_offsets, const int32_t* slot_of_expert, int num_experts, int K,
                             int N_out, int b_rows_per_slot, int64_t rows_cap, float* out, int64_t ldo,
                             cudaStream_t stream, const int32_t* seg_expert = nullptr);

// Layer internals the expert-parallel handle (ep.cu) builds on (layer.cu).
struct LayerView {
  int E, d, f, k, dtype, elem, seg_pad;
  int64_t max_tokens, rows_cap;
  const int32_t* served_idx;
  const float* served_w;
  const int64_t* seg_offsets;
  const int64_t* block_base;
  int32_t* pos;
  const int32_t* counts;  // [E] real rows per expert of the last route
};
}  // namespace emoe

struct emoe_layer;
namespace emoe {
LayerView layer_view(emoe_layer* L);
// K1 + K3a (route, per-expert counts, padded local segment offsets); no gather
void layer_route_scan(emoe_layer* L, const void* x, const float* logits_in, int64_t T, cudaStream_t s);
// K4 over caller rows in n_seg segments (device seg offsets / experts);
// after_gemm1 (optional) is recorded on s between the two GEMMs
void layer_ffn_rows(emoe_layer* L, const void* xr, int64_t R, const int64_t* segs, const int32_t* seg_expert,
                    int n_seg, void* hr, void* yr, cudaStream_t s, const PeerOut* peer_out = nullptr,
                    cudaEvent_t after_gemm1 = nullptr);
// K4 over received all-to-all chunks (NCCL EP transport): segment i's A rows
// at r + a_shift[i] of x_chunks, H compact [h_rows][f], Y rows stored at
// r + a_shift[i] of y_chunks (the return chunks mirror the receive chunks)
void layer_ffn_chunks(emoe_layer* L, const void* x_chunks, int64_t x_rows, const int64_t* segs,
                      const int32_t* seg_expert, int n_seg, const int64_t* a_shift, void* h, int64_t h_rows,
                      void* y_chunks, int64_t y_rows, cudaStream_t s, cudaEvent_t after_gemm1 = nullptr);

}  // namespace emoe
