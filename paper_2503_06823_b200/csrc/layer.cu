// C ABI: the MoE layer handle (gate, HBM expert slot pool, two-phase residency
// with side-stream H2D loads, routing/permute/FFN/combine workspace) and the
// batched route_token entry point.  See include/emoe.h for the contract.
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "capi_util.h"
#include "kernels.h"

namespace emoe {

std::string& last_error_slot() {
  static thread_local std::string s;
  return s;
}

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

// off by default: neutral inside the replayed graphs of configs 1 and 3, and
// it slowed the host-buffer (e2e) path of config 2 from 24.5 to 26.8 ms per
// call on the same box (profiles/r02_pdl_fused_scan_ab_L2.txt); EMOE_PDL=1 enables it
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("EMOE_PDL");
    return v && v[0] == '1';
  }();
  return on;
}

void ensure_max_dynamic_smem(const void* func, int bytes) {
  int dev = 0;
  EMOE_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{dev, func}];
  if (have >= bytes) return;
  EMOE_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

namespace {

constexpr int kMaxTableE = 256;

struct TableUpdate {
  int E;
  uint8_t resident[kMaxTableE];
  int32_t slot[kMaxTableE];
};

// Residency tables travel as kernel parameters: captured at launch, ordered
// on the stream, no host staging buffer to race on.
__global__ void set_tables_kernel(TableUpdate u, uint8_t* resident, int32_t* slot) {
  for (int e = threadIdx.x; e < u.E; e += blockDim.x) {
    resident[e] = u.resident[e];
    slot[e] = u.slot[e];
  }
}

struct ScoresUpdate {
  int E;
  double v[kMaxTableE];
};
__global__ void set_scores_kernel(ScoresUpdate u, double* scores) {
  for (int e = threadIdx.x; e < u.E; e += blockDim.x) scores[e] = u.v[e];
}

// engine.cpp:473-478 demand map: tokens per rank-0 gate choice (integer
// atomics: exact and order-independent)
__global__ void gate_demand_kernel(const int32_t* topk, int64_t T, int k, int E, unsigned long long* counts) {
  __shared__ unsigned int h[kMaxTableE];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[topk[t * k]], 1u);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (h[e]) atomicAdd(&counts[e], (unsigned long long)h[e]);
}

template <typename T>
T* dmalloc(size_t count) {
  T* p = nullptr;
  if (count) EMOE_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

}  // namespace
}  // namespace emoe

using namespace emoe;

struct emoe_layer {
  emoe_layer_config cfg{};
  int elem = 2;
  int num_sms = 148;
  int64_t rows_cap = 0;
  int cta_group = 1;  // FFN GEMM CTA group
  int gemm_mc = 1;    // 2: weight tiles multicast over CTA pairs (1-CTA MMAs)
  int seg_pad = kSegPad;
  int route_blocks = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_evict = nullptr, ev_load_start = nullptr, ev_load_done = nullptr;

  void* wg = nullptr;
  void* w1_pool = nullptr;
  void* w3_pool = nullptr;
  void* w2_pool = nullptr;
  int32_t* slot_dev = nullptr;
  uint8_t* resident_dev = nullptr;
  double* scores_dev = nullptr;
  bool have_scores = false;

  std::vector<void*> host_w1, host_w3, host_w2;  // library-owned pinned copies
  std::vector<int> slot_of_expert;               // compute-visible
  std::vector<int> expert_in_slot;
  std::vector<uint8_t> resident;
  std::vector<int> pending_experts, pending_slots;
  double last_load_bytes = 0, last_load_ms = 0, pending_bytes = 0;

  // workspace
  float* logits = nullptr;
  int32_t* topk = nullptr;
  int32_t* r_expert = nullptr;
  int32_t* r_rank = nullptr;
  uint8_t* r_hit = nullptr;
  int32_t* served_idx = nullptr;
  float* served_w = nullptr;
  int32_t* block_counts = nullptr;
  int32_t* counts = nullptr;
  int64_t* seg_offsets = nullptr;
  int64_t* block_base = nullptr;
  int32_t* pos = nullptr;
  int32_t* row_token = nullptr;
  int32_t* route_sync = nullptr;  // [route blocks] zeroed counters (RouteArgs::sync); per layer, never shared
  void* x_perm = nullptr;
  void* h = nullptr;
  void* y_perm = nullptr;
  void* x_in = nullptr;
  void* y_out = nullptr;
  int* err_flag = nullptr;
  int64_t last_T = 0;
  // workspace borrowed from another layer (emoe_layer_share_workspace): the
  // buffers below the routing tables belong to the donor and are not freed here
  bool borrowed_ws = false;
  unsigned long long* demand_dev = nullptr;  // emoe_layer_gate_demand scratch

  CUtensorMap ta1{}, tb1{}, tb3{}, ta2{}, tb2{}, to1{}, to2{};

  // fp32 layers on tensor cores (3xTF32, grouped_gemm_tf32.cu): the slot
  // pools hold tf32(W) in place and W - tf32(W) in the *_lo twins (split on
  // load); GEMM1 reads x split into x_hi / x_lo and writes H as h (hi) + h_lo
  bool tf32 = false;
  void* w1_lo = nullptr;
  void* w3_lo = nullptr;
  void* w2_lo = nullptr;
  float* x_hi = nullptr;
  float* x_lo = nullptr;
  float* h_lo = nullptr;
  Tf32Operands op1{}, op2{};
  // stream-K scratch of the 3xTF32 GEMMs (grouped_gemm_tf32.cu): one raw
  // partial tile per co-resident CTA and per-tile arrival counters
  float* sk_partial = nullptr;
  size_t sk_partial_floats = 0;
  int32_t* sk_arrive = nullptr;
  int64_t sk_arrivals = 0;
  void ensure_sk_arrive(int64_t rows, cudaStream_t s) {
    const int epi1 = swiglu() ? EPI_SWIGLU : EPI_RELU;
    const int64_t need =
        std::max(gemm_tf32x3_arrivals(epi1, cfg.d_ff, rows), gemm_tf32x3_arrivals(EPI_STORE, cfg.d_model, rows));
    if (need <= sk_arrivals) return;
    if (sk_arrive) {
      EMOE_CUDA(cudaStreamSynchronize(s));  // earlier launches may still use the old table
      EMOE_CUDA(cudaFree(sk_arrive));
    }
    sk_arrive = dmalloc<int32_t>((size_t)need);
    EMOE_CUDA(cudaMemsetAsync(sk_arrive, 0, sizeof(int32_t) * need, s));
    sk_arrivals = need;
  }
  // growable scratch for emoe_ffn_segments on caller rows (fp32)
  float* sx_hi = nullptr;
  float* sx_lo = nullptr;
  float* sh_lo = nullptr;
  int64_t s_rows = 0;

  size_t w1_elems() const { return (size_t)cfg.d_ff * cfg.d_model; }
  size_t w2_elems() const { return (size_t)cfg.d_model * cfg.d_ff; }
  bool swiglu() const { return cfg.activation == EMOE_ACT_SWIGLU; }

  void push_tables(cudaStream_t s) {
    TableUpdate u;
    u.E = cfg.num_experts;
    for (int e = 0; e < cfg.num_experts; ++e) {
      u.resident[e] = resident[e];
      u.slot[e] = slot_of_expert[e];
    }
    set_tables_kernel<<<1, 128, 0, s>>>(u, resident_dev, slot_dev);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
  }

  int n_resident() const {
    int n = 0;
    for (uint8_t r : resident) n += r;
    return n;
  }

  void finish_pending(cudaStream_t s) {
    EMOE_CUDA(cudaStreamWaitEvent(s, ev_load_done, 0));
    for (size_t i = 0; i < pending_experts.size(); ++i) {
      resident[pending_experts[i]] = 1;
      slot_of_expert[pending_experts[i]] = pending_slots[i];
    }
    float ms = 0;
    EMOE_CUDA(cudaEventElapsedTime(&ms, ev_load_start, ev_load_done));
    last_load_ms = ms;
    last_load_bytes = pending_bytes;
    pending_experts.clear();
    pending_slots.clear();
    push_tables(s);
  }

  void poll(bool blocking, cudaStream_t s, int* still) {
    if (still) *still = 0;
    if (pending_experts.empty()) return;
    if (blocking) {
      EMOE_CUDA(cudaEventSynchronize(ev_load_done));
    } else {
      cudaError_t q = cudaEventQuery(ev_load_done);
      if (q == cudaErrorNotReady) {
        if (still) *still = 1;
        return;
      }
      EMOE_CUDA(q);
    }
    finish_pending(s);
  }

  // Gate on tcgen05 for E in {32, 64, 96, 128} (bf16): W_g zero-padded to 256 rows.
  void* wg_pad = nullptr;
  CUtensorMap t_gate{}, t_gate2{};  // split path: box 256 rows (1 CTA per MMA) / 128 rows (CTA pair)
  CUtensorMap t_gate_tc{};          // fused gate + route: box E / cluster rows
  bool keep_logits = true;          // fused gate: also store the fp32 logits in the workspace
  static bool split_gate() {
    static const bool split = [] {
      const char* v = getenv("EMOE_GATE_ROUTE");
      return v && std::strcmp(v, "split") == 0;
    }();
    return split;
  }
  bool tc_gate() const {
    return cfg.dtype == EMOE_DTYPE_BF16 && cfg.num_experts >= 32 && cfg.num_experts % 32 == 0 && wg_pad;
  }

  // logits_in of a forward: EMOE_LOGITS_REPLACE (the routing-driven parity
  // mode: no gate) or EMOE_LOGITS_ADD (the gate runs on x and logits_in is
  // added to its logits before routing)
  int logits_mode = EMOE_LOGITS_REPLACE;

  // Expert parallelism: routing sees the GLOBAL resident set (the reference
  // Placement) while this GPU's slots hold only the experts it serves.
  bool route_override = false;
  std::vector<uint8_t> route_resident;
  uint8_t* route_resident_dev = nullptr;

  void route(const void* x, const float* logits_in, int64_t T, cudaStream_t s) {
    EMOE_REQUIRE(T >= 0 && T <= cfg.max_tokens, "moe_forward: T exceeds the layer's max_tokens");
    int n_route = n_resident();
    if (route_override) {
      n_route = 0;
      for (uint8_t r : route_resident) n_route += r;
    }
    if (n_route == 0 && !cfg.forced_miss) throw InvariantError("route_token: no resident experts at layer");
    RouteArgs a;
    a.T = T;
    a.d = cfg.d_model;
    a.E = cfg.num_experts;
    a.k = cfg.top_k;
    a.weight_mode = cfg.weight_mode;
    a.forced_miss = cfg.forced_miss;
    a.resident = route_override ? route_resident_dev : resident_dev;
    a.scores = have_scores ? scores_dev : nullptr;
    a.error_flag = err_flag;
    RouteOut o{logits, topk, r_expert, r_rank, r_hit, served_idx, served_w, block_counts};
    const bool add = logits_in && logits_mode == EMOE_LOGITS_ADD;
    EMOE_REQUIRE(!add || x, "route: the logits-bias mode runs the gate, so x is required");
    a.bias = add ? logits_in : nullptr;
    a.sync = route_sync;
    if (logits_in && !add) {
      launch_route_from_logits(logits_in, a, o, s);
    } else if (tc_gate() && !split_gate()) {
      // many experts: the gate is a real GEMM (T x d x E) on tcgen05 with the
      // routing in its epilogue (x read once, no logits round trip)
      const CUtensorMap tx = make_tmap_bf16_2d(x, (uint64_t)T, cfg.d_model, 128);
      launch_gate_route_tc(tx, t_gate_tc, a, o, keep_logits, num_sms, s);
    } else if (tc_gate()) {
      // EMOE_GATE_ROUTE=split (A/B runs): the dense gate GEMM into the fp32
      // logits buffer, then route from the logits
      const CUtensorMap tx = make_tmap_bf16_2d(x, (uint64_t)T, cfg.d_model, 128);
      static const int gate_cg = [] {  // EMOE_GATE_CG=2: the gate GEMM on CTA pairs (A/B runs)
        const char* v = getenv("EMOE_GATE_CG");
        return v && v[0] == '2' ? 2 : 1;
      }();
      launch_dense_gemm_f32(tx, gate_cg == 2 ? t_gate2 : t_gate, T, cfg.d_model, 256, logits, cfg.num_experts,
                            cfg.num_experts, num_sms, s, gate_cg);
      launch_route_from_logits(logits, a, o, s);
    } else {
      launch_gate_route(x, wg, cfg.dtype, a, o, s);
    }
    last_T = T;
  }

  // stage events for emoe_layer_stage_times (route, scan+permute, gemm1, gemm2, combine);
  // one event set per profiled forward, averaged and recycled by stage_times()
  bool profiling = false;
  cudaEvent_t ext_mark3 = nullptr;  // layer_ffn_rows: the caller's between-GEMMs event
  std::vector<std::array<cudaEvent_t, 6>> ev_pool;
  size_t ev_used = 0;
  void mark(int i, cudaStream_t s) {
    if (!profiling) return;
    if (i == 0 && ev_used == ev_pool.size()) {
      std::array<cudaEvent_t, 6> set;
      for (cudaEvent_t& e : set) EMOE_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(set);
    }
    // inside a stream capture the events must be external record nodes (a
    // plain record would only order the capture)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    EMOE_CUDA(cudaStreamIsCapturing(s, &cap));
    EMOE_CUDA(cudaEventRecordWithFlags(ev_pool[ev_used][i], s,
                                       cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                            : cudaEventRecordDefault));
    if (i == 5) ++ev_used;
  }

  // poll_loads = false: the caller polled already (a chunked host call uses
  // one residency snapshot for all its chunks)
  void forward(const void* x, const float* logits_in, void* y, int64_t T, cudaStream_t s, bool poll_loads = true) {
    if (poll_loads) poll(false, s, nullptr);
    if (T == 0) {
      route(x, logits_in, T, s);
      return;
    }
    mark(0, s);
    route(x, logits_in, T, s);
    mark(1, s);
    permute(x, T, s);
    mark(2, s);
    if (fused_combine()) {  // top-1 / top-2: GEMM2's epilogue writes y directly (K5 fused)
      ScatterCombine sc{row_token, served_w, static_cast<__nv_bfloat16*>(y)};
      if (cfg.top_k == 2) {
        if (!combine_arrive) {  // [max_tokens][d/256][2] counters, zero between forwards
          const size_t n = (size_t)cfg.max_tokens * ceil_div(cfg.d_model, 256) * 2;
          combine_arrive = dmalloc<int32_t>(n);
          EMOE_CUDA(cudaMemsetAsync(combine_arrive, 0, n * sizeof(int32_t), s));
        }
        sc.k = 2;
        sc.pos = pos;
        sc.arrive = combine_arrive;
      }
      ffn(x_perm, rows_cap, seg_offsets, nullptr, cfg.num_experts, h, y_perm, s, true, &sc);
      y_perm_valid = false;
    } else {
      ffn(x_perm, rows_cap, seg_offsets, nullptr, cfg.num_experts, h, y_perm, s, true);
      launch_combine(y_perm, cfg.dtype, T, cfg.d_model, cfg.top_k, pos, served_w, y, s);
      y_perm_valid = true;
    }
    mark(5, s);
  }

  // bf16 layers without forced misses serve every token at least once, so
  // GEMM2's epilogue can produce y: top-1 as a scaled row scatter (default),
  // top-2 by the second of a token's two rows combining both
  // (EMOE_FUSED_COMBINE=2; bit-identical, but its direct-store epilogue costs
  // GEMM2 more than the 0.24 ms combine it removes at the config-2 shape,
  // profiles/r01_fused_top2_combine_ab.jsonl).  EMOE_FUSED_COMBINE=0 keeps
  // the separate K5 for every layer.
  bool fused_combine() const {
    static const int mode = [] {
      const char* v = getenv("EMOE_FUSED_COMBINE");
      return v ? atoi(v) : 1;
    }();
    return cfg.dtype == EMOE_DTYPE_BF16 && !cfg.forced_miss && cfg.top_k <= mode && cfg.top_k <= 2;
  }
  int32_t* combine_arrive = nullptr;
  bool y_perm_valid = true;

  // A3 after route(): per-expert offsets, positions, gathered rows in x_perm
  void permute(const void* x, int64_t T, cudaStream_t s) {
    const int E = cfg.num_experts;
    // 3xTF32 layers: the permute also writes the hi / lo split of every row
    // (the GEMM reads only those), so ffn() skips the separate split pass
    launch_scan_permute(x, elem, T, cfg.d_model, E, cfg.top_k, served_idx, block_counts, seg_pad, counts,
                        seg_offsets, block_base, x_perm, pos, row_token, counts + E, s, tf32 ? x_hi : nullptr,
                        tf32 ? x_lo : nullptr);
    perm_split_done = tf32;
  }
  bool perm_split_done = false;  // x_hi / x_lo hold the split of x_perm's rows

  // A4 over rows [R][d] in n_seg padded segments (seg_expert null: segment i = expert i).
  // workspace = the rows are the layer's own x_perm/h/y_perm (cached tensor maps).
  void ffn(const void* xr, int64_t R, const int64_t* segs, const int32_t* seg_expert, int n_seg, void* hr, void* yr,
           cudaStream_t s, bool workspace, const ScatterCombine* scatter = nullptr,
           const PeerOut* peer_out = nullptr) {
    const int d = cfg.d_model, f = cfg.d_ff;
    if (cfg.dtype == EMOE_DTYPE_BF16) {
      CUtensorMap a1 = ta1, a2 = ta2, o1 = to1, o2 = to2;
      if (!workspace) {
        a1 = make_tmap_bf16_2d(xr, (uint64_t)R, d, 128);
        a2 = make_tmap_bf16_2d(hr, (uint64_t)R, f, 128);
        o1 = make_tmap_bf16_store(hr, (uint64_t)R, f);
        o2 = make_tmap_bf16_store(yr, (uint64_t)R, d);
      }
      launch_grouped_gemm(swiglu() ? EPI_SWIGLU : EPI_RELU, cta_group, gemm_mc, a1, tb1, tb3, segs, slot_dev, n_seg, d, f, f,
                          static_cast<__nv_bfloat16*>(hr), f, num_sms, s, seg_expert, &o1);
      mark(3, s);
      if (ext_mark3) EMOE_CUDA(cudaEventRecord(ext_mark3, s));
      launch_grouped_gemm(EPI_STORE, cta_group, gemm_mc, a2, tb2, tb2, segs, slot_dev, n_seg, f, d, d,
                          static_cast<__nv_bfloat16*>(yr), d, num_sms, s, seg_expert, &o2, scatter, peer_out);
      mark(4, s);
    } else if (tf32) {
      const int epi1 = swiglu() ? EPI_SWIGLU : EPI_RELU;
      float *xh = x_hi, *xl = x_lo, *hl = h_lo;
      Tf32Operands o1 = op1, o2 = op2;
      if (!workspace) {  // caller rows: split into the growable scratch
        if (R > s_rows) {
          for (float* q : {sx_hi, sx_lo, sh_lo})
            if (q) EMOE_CUDA(cudaFree(q));
          sx_hi = dmalloc<float>((size_t)R * d);
          sx_lo = dmalloc<float>((size_t)R * d);
          sh_lo = dmalloc<float>((size_t)R * f);
          s_rows = R;
        }
        xh = sx_hi;
        xl = sx_lo;
        hl = sh_lo;
        o1.a_hi = make_tmap_f32_2d(xh, (uint64_t)R, d, 128);
        o1.a_lo = make_tmap_f32_2d(xl, (uint64_t)R, d, 128);
        o2.a_hi = make_tmap_f32_2d(hr, (uint64_t)R, f, 128);
        o2.a_lo = make_tmap_f32_2d(hl, (uint64_t)R, f, 128);
      }
      if (!(workspace && perm_split_done && xr == x_perm))
        launch_split_tf32(static_cast<const float*>(xr), xh, xl, R * d, s, segs + n_seg, d);
      ensure_sk_arrive(R, s);
      const StreamK sk{sk_partial, sk_partial_floats, sk_arrive, sk_arrivals};
      launch_grouped_gemm_tf32x3(epi1, o1, segs, slot_dev, seg_expert, n_seg, d, f, f, static_cast<float*>(hr), hl,
                                 f, R, sk, s);
      mark(3, s);
      launch_grouped_gemm_tf32x3(EPI_STORE, o2, segs, slot_dev, seg_expert, n_seg, f, d, d, static_cast<float*>(yr),
                                 nullptr, d, R, sk, s);
      mark(4, s);
    } else {
      launch_grouped_gemm_f32(swiglu() ? EPI_SWIGLU : EPI_RELU, static_cast<const float*>(xr), d,
                              static_cast<const float*>(w1_pool), static_cast<const float*>(w3_pool), segs, slot_dev,
                              n_seg, d, f, f, R, static_cast<float*>(hr), f, s, seg_expert);
      mark(3, s);
      launch_grouped_gemm_f32(EPI_STORE, static_cast<const float*>(hr), f, static_cast<const float*>(w2_pool),
                              nullptr, segs, slot_dev, n_seg, f, d, d, R, static_cast<float*>(yr), d, s, seg_expert);
      mark(4, s);
    }
  }

  // Host-buffer forward, pipelined in token chunks: the H2D copy of chunk i+1
  // (in_stream) and the D2H copy of chunk i-1 (out_stream) overlap the forward
  // of chunk i on the compute stream.  bf16: per-token results do not depend
  // on the chunking (every row's GEMM reduction order is fixed), so the output
  // is bit-identical to a single forward over all T tokens.  fp32 (3xTF32
  // stream-K): where a tile's K range is split between CTA pairs depends on
  // the batch's tile count, so chunks agree with one forward to fp32 rounding.
  // Two device staging sets: call i+1's H2D (into set b^1) overlaps call i's
  // compute and D2H (set b).  Reuse of a set waits on events: H2D into x[b]
  // after the compute that last read x[b]; compute into y[b] after the D2H
  // that last read y[b].
  cudaStream_t in_stream = nullptr, out_stream = nullptr;
  void* x_stage[2] = {nullptr, nullptr};
  void* y_stage[2] = {nullptr, nullptr};
  cudaEvent_t x_free[2] = {}, y_free[2] = {}, host_done = nullptr;
  std::vector<cudaEvent_t> chunk_ev[2];
  int stage_next = 0;

  void forward_host_async(const void* x_host, void* y_host, int64_t T, cudaStream_t s) {
    EMOE_REQUIRE(T >= 0 && T <= cfg.max_tokens, "moe_forward: T exceeds the layer's max_tokens");
    const size_t row = (size_t)cfg.d_model * elem;
    if (!x_stage[0]) {
      for (int b = 0; b < 2; ++b) {
        x_stage[b] = dmalloc<uint8_t>((size_t)cfg.max_tokens * row);
        y_stage[b] = dmalloc<uint8_t>((size_t)cfg.max_tokens * row);
        EMOE_CUDA(cudaEventCreateWithFlags(&x_free[b], cudaEventDisableTiming));
        EMOE_CUDA(cudaEventCreateWithFlags(&y_free[b], cudaEventDisableTiming));
      }
      EMOE_CUDA(cudaEventCreateWithFlags(&host_done, cudaEventDisableTiming));
      EMOE_CUDA(cudaStreamCreateWithFlags(&in_stream, cudaStreamNonBlocking));
      EMOE_CUDA(cudaStreamCreateWithFlags(&out_stream, cudaStreamNonBlocking));
      // staging sets start free (events recorded once, complete immediately)
      for (int b = 0; b < 2; ++b) {
        EMOE_CUDA(cudaEventRecord(x_free[b], s));
        EMOE_CUDA(cudaEventRecord(y_free[b], s));
      }
    }
    static const int n_chunks = [] {  // EMOE_H2D_CHUNKS overrides for tuning
      const char* v = getenv("EMOE_H2D_CHUNKS");
      // 2: best of {1, 2, 4} with the async two-staging-set pipeline over 20
      // calls (profiles/r01_e2e_chunks_s40.jsonl; 1-4 are within 1.5 %)
      return v ? std::max(1, atoi(v)) : 2;
    }();
    int64_t chunk = std::max<int64_t>(8192, ceil_div(T, n_chunks));
    chunk = ceil_div(chunk, kRouteBlockTokens) * kRouteBlockTokens;
    const int n = (int)std::max<int64_t>(1, ceil_div(T, chunk));
    const int b = stage_next;
    stage_next ^= 1;
    auto& ev = chunk_ev[b];
    while ((int)ev.size() < 2 * n) {
      cudaEvent_t e;
      EMOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    EMOE_CUDA(cudaStreamWaitEvent(in_stream, x_free[b], 0));
    EMOE_CUDA(cudaStreamWaitEvent(s, y_free[b], 0));
    poll(false, s, nullptr);  // one residency snapshot for every chunk of this call
    for (int i = 0; i < n; ++i) {
      const int64_t t0 = i * chunk, tn = std::min<int64_t>(chunk, T - t0);
      uint8_t* xd = static_cast<uint8_t*>(x_stage[b]) + t0 * row;
      uint8_t* yd = static_cast<uint8_t*>(y_stage[b]) + t0 * row;
      EMOE_CUDA(cudaMemcpyAsync(xd, static_cast<const uint8_t*>(x_host) + t0 * row, tn * row,
                                cudaMemcpyHostToDevice, in_stream));
      EMOE_CUDA(cudaEventRecord(ev[2 * i], in_stream));
      EMOE_CUDA(cudaStreamWaitEvent(s, ev[2 * i], 0));
      forward(xd, nullptr, yd, tn, s, false);
      EMOE_CUDA(cudaEventRecord(ev[2 * i + 1], s));
      EMOE_CUDA(cudaStreamWaitEvent(out_stream, ev[2 * i + 1], 0));
      EMOE_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(y_host) + t0 * row, yd, tn * row, cudaMemcpyDeviceToHost,
                                out_stream));
    }
    EMOE_CUDA(cudaEventRecord(x_free[b], s));
    EMOE_CUDA(cudaEventRecord(y_free[b], out_stream));
    EMOE_CUDA(cudaEventRecord(host_done, out_stream));
  }

  void wait_host() {
    if (host_done) EMOE_CUDA(cudaEventSynchronize(host_done));
  }

  void forward_host(const void* x_host, void* y_host, int64_t T, cudaStream_t s) {
    forward_host_async(x_host, y_host, T, s);
    wait_host();
  }

  void begin_load(const int32_t* ev, int nev, const int32_t* ld, int nld, cudaStream_t s) {
    const int E = cfg.num_experts;
    if (!pending_experts.empty()) poll(true, s, nullptr);  // plans apply in order
    std::vector<uint8_t> evicting(E, 0), loading(E, 0);
    for (int i = 0; i < nev; ++i) {
      EMOE_REQUIRE(ev[i] >= 0 && ev[i] < E, "begin_load: eviction index out of range");
      if (!resident[ev[i]] || evicting[ev[i]]) throw InvariantError("placement: evicting non-resident expert");
      evicting[ev[i]] = 1;
    }
    int after = n_resident() - nev;
    for (int i = 0; i < nld; ++i) {
      EMOE_REQUIRE(ld[i] >= 0 && ld[i] < E, "begin_load: load index out of range");
      if ((resident[ld[i]] && !evicting[ld[i]]) || loading[ld[i]])
        throw InvariantError("placement: loading resident expert");
      if (!host_w1[ld[i]]) throw ValidationError("begin_load: expert weights were never registered");
      loading[ld[i]] = 1;
      if (++after > cfg.num_slots) throw InvariantError("placement: layer budget exceeded");
    }
    // phase 1 (load start): evictions take effect for compute enqueued after this point
    for (int i = 0; i < nev; ++i) {
      resident[ev[i]] = 0;
      expert_in_slot[slot_of_expert[ev[i]]] = -1;
      slot_of_expert[ev[i]] = -1;
    }
    push_tables(s);
    if (nld == 0) return;
    // the freed slots may still be read by compute already enqueued on `s`
    cudaStream_t cs = load_stream();
    EMOE_CUDA(cudaEventRecord(ev_evict, s));
    EMOE_CUDA(cudaStreamWaitEvent(cs, ev_evict, 0));
    EMOE_CUDA(cudaEventRecord(ev_load_start, cs));
    pending_bytes = 0;
    for (int i = 0; i < nld; ++i) {
      int slot = -1;
      for (int q = 0; q < cfg.num_slots; ++q)
        if (expert_in_slot[q] < 0) {
          slot = q;
          break;
        }
      if (slot < 0) throw InvariantError("placement: layer budget exceeded");
      expert_in_slot[slot] = ld[i];
      const int e = ld[i];
      const size_t b1 = w1_elems() * elem, b2 = w2_elems() * elem;
      EMOE_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(w1_pool) + slot * b1, host_w1[e], b1, cudaMemcpyHostToDevice,
                                cs));
      pending_bytes += (double)b1;
      if (swiglu()) {
        EMOE_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(w3_pool) + slot * b1, host_w3[e], b1,
                                  cudaMemcpyHostToDevice, cs));
        pending_bytes += (double)b1;
      }
      EMOE_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(w2_pool) + slot * b2, host_w2[e], b2, cudaMemcpyHostToDevice,
                                cs));
      pending_bytes += (double)b2;
      if (tf32) {  // tf32 hi in place + fp32 lo twin, on the copy stream before the load event
        auto split = [&](void* pool, void* lo, size_t elems) {
          float* w = reinterpret_cast<float*>(static_cast<uint8_t*>(pool) + slot * elems * 4);
          launch_split_tf32(w, w, reinterpret_cast<float*>(static_cast<uint8_t*>(lo) + slot * elems * 4),
                            (int64_t)elems, cs);
        };
        split(w1_pool, w1_lo, w1_elems());
        if (swiglu()) split(w3_pool, w3_lo, w1_elems());
        split(w2_pool, w2_lo, w2_elems());
      }
      pending_experts.push_back(e);
      pending_slots.push_back(slot);
    }
    EMOE_CUDA(cudaEventRecord(ev_load_done, cs));
  }

  cudaStream_t ext_copy_stream = nullptr;  // shared copy stream (layer-sequential loads)
  std::vector<uint8_t> host_owned;         // 1 = library-owned pinned copy, 0 = caller pointer
  cudaStream_t load_stream() const { return ext_copy_stream ? ext_copy_stream : copy_stream; }

  // the per-forward workspace (routing outputs, permutation, FFN rows)
  std::vector<void*> workspace_buffers() const {
    return {(void*)logits,       (void*)topk,   (void*)r_expert,    (void*)r_rank,    (void*)r_hit,
            (void*)served_idx,   (void*)served_w, (void*)block_counts, (void*)counts, (void*)seg_offsets,
            (void*)block_base,   (void*)pos,    (void*)row_token,   x_perm,           h,
            y_perm,              (void*)x_hi,   (void*)x_lo,        (void*)h_lo};
  }

  void destroy() {
    auto f = [](void* p) {
      if (p) cudaFree(p);
    };
    if (!borrowed_ws)
      for (void* p : workspace_buffers()) f(p);
    for (void* p : {(void*)wg, w1_pool, w3_pool, w2_pool, (void*)slot_dev, (void*)resident_dev, (void*)scores_dev,
                    (void*)route_resident_dev, wg_pad, (void*)demand_dev, x_in, y_out, (void*)err_flag, x_stage[0],
                    x_stage[1], y_stage[0], y_stage[1], w1_lo, w3_lo, w2_lo, (void*)sx_hi, (void*)sx_lo,
                    (void*)sh_lo, (void*)combine_arrive, (void*)sk_partial,
                    (void*)sk_arrive, (void*)route_sync})
      f(p);
    for (auto* v : {&host_w1, &host_w3, &host_w2})
      for (size_t e = 0; e < v->size(); ++e)
        if ((*v)[e] && e < host_owned.size() && host_owned[e]) cudaFreeHost((*v)[e]);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (in_stream) cudaStreamDestroy(in_stream);
    if (out_stream) cudaStreamDestroy(out_stream);
    for (auto& v : chunk_ev)
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    for (cudaEvent_t e : {x_free[0], x_free[1], y_free[0], y_free[1], host_done})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {ev_evict, ev_load_start, ev_load_done})
      if (e) cudaEventDestroy(e);
    for (auto& set : ev_pool)
      for (cudaEvent_t e : set) cudaEventDestroy(e);
  }
};

extern "C" {

const char* emoe_last_error(void) { return last_error_slot().c_str(); }
int emoe_version(void) { return 1; }

int emoe_layer_create(const emoe_layer_config* cfg, emoe_layer** out) {
  return guard([&] {
    EMOE_REQUIRE(cfg && out, "layer_create: null argument");
    const emoe_layer_config& c = *cfg;
    EMOE_REQUIRE(c.num_experts >= 1 && c.num_experts <= 128, "layer.num_experts: must be in [1, 128]");
    EMOE_REQUIRE(c.top_k >= 1 && c.top_k <= 8 && c.top_k <= c.num_experts, "layer.top_k: must be in [1, min(8, E)]");
    EMOE_REQUIRE(c.num_slots >= 1 && c.num_slots <= c.num_experts, "layer.num_slots: must be in [1, E]");
    EMOE_REQUIRE(c.max_tokens >= 1, "layer.max_tokens: must be >= 1");
    EMOE_REQUIRE(c.dtype == EMOE_DTYPE_BF16 || c.dtype == EMOE_DTYPE_F32, "layer.dtype: unknown");
    EMOE_REQUIRE(c.activation == EMOE_ACT_SWIGLU || c.activation == EMOE_ACT_RELU, "layer.activation: unknown");
    if (c.dtype == EMOE_DTYPE_BF16) {
      EMOE_REQUIRE(c.d_model % 256 == 0, "layer.d_model: bf16 path needs a multiple of 256");
      EMOE_REQUIRE(c.d_ff % 256 == 0, "layer.d_ff: bf16 path needs a multiple of 256");
    } else {
      EMOE_REQUIRE(c.d_model % 64 == 0 && c.d_ff % 64 == 0, "layer: fp32 path needs d_model, d_ff % 64 == 0");
    }
    auto* L = new emoe_layer();
    try {
      L->cfg = c;
      L->elem = c.dtype == EMOE_DTYPE_BF16 ? 2 : 4;
      int dev = 0;
      EMOE_CUDA(cudaGetDevice(&dev));
      EMOE_CUDA(cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, dev));
      const int E = c.num_experts, k = c.top_k;
      const int64_t T = c.max_tokens;
      EMOE_REQUIRE(c.gemm_cta_group >= 0 && c.gemm_cta_group <= 2, "layer.gemm_cta_group: must be 0, 1 or 2");
      // auto: short-K layers (d_model <= 2048) are fed from L2 at ~96 B/clk/SM by the
      // 128x256 tile and gain from the CTA pair's halved operand traffic (Switch shape
      // +6%); large layers run at the power cap, where 1-CTA is 9% faster (Mixtral
      // shape) — profiles/r01_cta_group_ab.jsonl
      const int auto_cg = c.d_model <= 2048 ? 2 : 1;
      L->cta_group = c.dtype == EMOE_DTYPE_BF16 ? (c.gemm_cta_group ? c.gemm_cta_group : auto_cg) : 1;
      // EMOE_GEMM_MC=2: 1-CTA GEMMs with the weight tile multicast over CTA pairs (A/B runs)
      L->gemm_mc = c.dtype == EMOE_DTYPE_BF16 && L->cta_group == 1 && getenv("EMOE_GEMM_MC") &&
                           atoi(getenv("EMOE_GEMM_MC")) == 2
                       ? 2
                       : 1;
      L->seg_pad = c.dtype == EMOE_DTYPE_BF16 ? gemm_tile_m(L->cta_group, L->gemm_mc) : gemm_tf32x3_tile_m();
      L->rows_cap = T * k + (int64_t)E * L->seg_pad;
      L->route_blocks = (int)ceil_div(T, kRouteBlockTokens);
      EMOE_CUDA(cudaStreamCreateWithFlags(&L->copy_stream, cudaStreamNonBlocking));
      EMOE_CUDA(cudaEventCreateWithFlags(&L->ev_evict, cudaEventDisableTiming));
      EMOE_CUDA(cudaEventCreate(&L->ev_load_start));
      EMOE_CUDA(cudaEventCreate(&L->ev_load_done));
      const size_t el = L->elem;
      L->wg = dmalloc<uint8_t>((size_t)E * c.d_model * el);
      L->w1_pool = dmalloc<uint8_t>((size_t)c.num_slots * L->w1_elems() * el);
      if (L->swiglu()) L->w3_pool = dmalloc<uint8_t>((size_t)c.num_slots * L->w1_elems() * el);
      L->w2_pool = dmalloc<uint8_t>((size_t)c.num_slots * L->w2_elems() * el);
      L->slot_dev = dmalloc<int32_t>(E);
      L->resident_dev = dmalloc<uint8_t>(E);
      L->scores_dev = dmalloc<double>(E);
      L->logits = dmalloc<float>((size_t)T * E);
      L->topk = dmalloc<int32_t>((size_t)T * k);
      L->r_expert = dmalloc<int32_t>(T);
      L->r_rank = dmalloc<int32_t>(T);
      L->r_hit = dmalloc<uint8_t>(T);
      L->served_idx = dmalloc<int32_t>((size_t)T * k);
      L->served_w = dmalloc<float>((size_t)T * k);
      L->block_counts = dmalloc<int32_t>((size_t)L->route_blocks * E);
      L->route_sync = dmalloc<int32_t>((size_t)L->route_blocks);  // the small-T fp32 gate's counters
      EMOE_CUDA(cudaMemset(L->route_sync, 0, sizeof(int32_t) * L->route_blocks));
      L->counts = dmalloc<int32_t>(E + 1);  // [E] = the scan kernel's last-block counter
      EMOE_CUDA(cudaMemset(L->counts, 0, (E + 1) * sizeof(int32_t)));
      L->seg_offsets = dmalloc<int64_t>(E + 1);
      L->block_base = dmalloc<int64_t>((size_t)L->route_blocks * E);
      L->pos = dmalloc<int32_t>((size_t)T * k);
      L->row_token = dmalloc<int32_t>(L->rows_cap);
      L->x_perm = dmalloc<uint8_t>((size_t)L->rows_cap * c.d_model * el);
      L->h = dmalloc<uint8_t>((size_t)L->rows_cap * c.d_ff * el);
      L->y_perm = dmalloc<uint8_t>((size_t)L->rows_cap * c.d_model * el);
      L->err_flag = dmalloc<int>(1);
      EMOE_CUDA(cudaMemset(L->x_perm, 0, (size_t)L->rows_cap * c.d_model * el));
      EMOE_CUDA(cudaMemset(L->h, 0, (size_t)L->rows_cap * c.d_ff * el));
      EMOE_CUDA(cudaMemset(L->y_perm, 0, (size_t)L->rows_cap * c.d_model * el));
      EMOE_CUDA(cudaMemset(L->err_flag, 0, sizeof(int)));
      EMOE_CUDA(cudaMemset(L->w1_pool, 0, (size_t)c.num_slots * L->w1_elems() * el));
      if (L->w3_pool) EMOE_CUDA(cudaMemset(L->w3_pool, 0, (size_t)c.num_slots * L->w1_elems() * el));
      EMOE_CUDA(cudaMemset(L->w2_pool, 0, (size_t)c.num_slots * L->w2_elems() * el));
      L->host_w1.assign(E, nullptr);
      L->host_w3.assign(E, nullptr);
      L->host_w2.assign(E, nullptr);
      L->host_owned.assign(E, 1);
      L->slot_of_expert.assign(E, -1);
      L->expert_in_slot.assign(c.num_slots, -1);
      L->resident.assign(E, 0);
      L->push_tables(0);
      if (c.dtype == EMOE_DTYPE_BF16) {
        const uint64_t d = c.d_model, f = c.d_ff;
        const int epi1 = L->swiglu() ? EPI_SWIGLU : EPI_RELU;
        const uint32_t b1_box = gemm_b_box_rows(epi1, L->cta_group, L->gemm_mc);
        L->ta1 = make_tmap_bf16_2d(L->x_perm, L->rows_cap, d, 128);
        L->tb1 = make_tmap_bf16_2d(L->w1_pool, (uint64_t)c.num_slots * f, d, b1_box);
        L->tb3 = L->swiglu() ? make_tmap_bf16_2d(L->w3_pool, (uint64_t)c.num_slots * f, d, b1_box) : L->tb1;
        L->ta2 = make_tmap_bf16_2d(L->h, L->rows_cap, f, 128);
        L->tb2 = make_tmap_bf16_2d(L->w2_pool, (uint64_t)c.num_slots * d, f, gemm_b_box_rows(EPI_STORE, L->cta_group, L->gemm_mc));
        L->to1 = make_tmap_bf16_store(L->h, L->rows_cap, f);
        L->to2 = make_tmap_bf16_store(L->y_perm, L->rows_cap, d);
      } else {
        // fp32: 3xTF32 on tcgen05 where the shape tiles (EMOE_F32_GEMM=ffma keeps the SIMT kernel)
        const char* mode = getenv("EMOE_F32_GEMM");
        const int epi1 = L->swiglu() ? EPI_SWIGLU : EPI_RELU;
        const uint64_t d = c.d_model, f = c.d_ff, slots = c.num_slots;
        L->tf32 = !(mode && std::strcmp(mode, "ffma") == 0) && gemm_tf32x3_supported(epi1, (int)d, (int)f) &&
                  gemm_tf32x3_supported(EPI_STORE, (int)f, (int)d);
        if (L->tf32) {
          const size_t pw1 = slots * L->w1_elems() * 4, pw2 = slots * L->w2_elems() * 4;
          L->w1_lo = dmalloc<uint8_t>(pw1);
          EMOE_CUDA(cudaMemset(L->w1_lo, 0, pw1));
          if (L->swiglu()) {
            L->w3_lo = dmalloc<uint8_t>(pw1);
            EMOE_CUDA(cudaMemset(L->w3_lo, 0, pw1));
          }
          L->w2_lo = dmalloc<uint8_t>(pw2);
          EMOE_CUDA(cudaMemset(L->w2_lo, 0, pw2));
          L->x_hi = dmalloc<float>((size_t)L->rows_cap * d);
          L->x_lo = dmalloc<float>((size_t)L->rows_cap * d);
          L->h_lo = dmalloc<float>((size_t)L->rows_cap * f);
          const uint32_t bb = gemm_tf32x3_b_box_rows(epi1), bb2 = gemm_tf32x3_b_box_rows(EPI_STORE);
          L->op1.a_hi = make_tmap_f32_2d(L->x_hi, L->rows_cap, d, 128);
          L->op1.a_lo = make_tmap_f32_2d(L->x_lo, L->rows_cap, d, 128);
          L->op1.b_hi = make_tmap_f32_2d(L->w1_pool, slots * f, d, bb);
          L->op1.b_lo = make_tmap_f32_2d(L->w1_lo, slots * f, d, bb);
          L->op1.b2_hi = L->swiglu() ? make_tmap_f32_2d(L->w3_pool, slots * f, d, bb) : L->op1.b_hi;
          L->op1.b2_lo = L->swiglu() ? make_tmap_f32_2d(L->w3_lo, slots * f, d, bb) : L->op1.b_lo;
          L->op2.a_hi = make_tmap_f32_2d(L->h, L->rows_cap, f, 128);
          L->op2.a_lo = make_tmap_f32_2d(L->h_lo, L->rows_cap, f, 128);
          L->op2.b_hi = make_tmap_f32_2d(L->w2_pool, slots * d, f, bb2);
          L->op2.b_lo = make_tmap_f32_2d(L->w2_lo, slots * d, f, bb2);
          L->op2.b2_hi = L->op2.b_hi;
          L->op2.b2_lo = L->op2.b_lo;
          // stream-K scratch (one partial tile per co-resident CTA, ~10-19 MB)
          L->sk_partial_floats = gemm_tf32x3_partial_floats(L->num_sms);
          L->sk_partial = dmalloc<float>(L->sk_partial_floats);
          L->ensure_sk_arrive(L->rows_cap, 0);
        }
      }
      EMOE_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      L->destroy();
      delete L;
      throw;
    }
    *out = L;
  });
}

int emoe_layer_destroy(emoe_layer* layer) {
  return guard([&] {
    if (!layer) return;
    cudaDeviceSynchronize();
    layer->destroy();
    delete layer;
  });
}

int emoe_layer_share_workspace(emoe_layer* L, const emoe_layer* donor) {
  return guard([&] {
    EMOE_REQUIRE(L && donor && L != donor, "share_workspace: need two distinct layers");
    EMOE_REQUIRE(!donor->borrowed_ws, "share_workspace: the donor must own its workspace");
    const emoe_layer_config &a = L->cfg, &b = donor->cfg;
    EMOE_REQUIRE(a.d_model == b.d_model && a.d_ff == b.d_ff && a.num_experts == b.num_experts &&
                     a.top_k == b.top_k && a.dtype == b.dtype && a.max_tokens == b.max_tokens &&
                     L->rows_cap == donor->rows_cap && L->tf32 == donor->tf32,
                 "share_workspace: layers differ in shape, dtype, max_tokens or GEMM tiling");
    EMOE_CUDA(cudaDeviceSynchronize());  // nothing in flight on the buffers being released
    if (!L->borrowed_ws)
      for (void* p : L->workspace_buffers())
        if (p) EMOE_CUDA(cudaFree(p));
    L->logits = donor->logits;
    L->topk = donor->topk;
    L->r_expert = donor->r_expert;
    L->r_rank = donor->r_rank;
    L->r_hit = donor->r_hit;
    L->served_idx = donor->served_idx;
    L->served_w = donor->served_w;
    L->block_counts = donor->block_counts;
    L->counts = donor->counts;
    L->seg_offsets = donor->seg_offsets;
    L->block_base = donor->block_base;
    L->pos = donor->pos;
    L->row_token = donor->row_token;
    L->x_perm = donor->x_perm;
    L->h = donor->h;
    L->y_perm = donor->y_perm;
    L->x_hi = donor->x_hi;
    L->x_lo = donor->x_lo;
    L->h_lo = donor->h_lo;
    // tensor maps over the (now shared) activation buffers; the weight maps stay
    L->ta1 = donor->ta1;
    L->ta2 = donor->ta2;
    L->to1 = donor->to1;
    L->to2 = donor->to2;
    L->op1.a_hi = donor->op1.a_hi;
    L->op1.a_lo = donor->op1.a_lo;
    L->op2.a_hi = donor->op2.a_hi;
    L->op2.a_lo = donor->op2.a_lo;
    L->borrowed_ws = true;
  });
}

int emoe_layer_set_gate_host(emoe_layer* L, const void* wg) {
  return guard([&] {
    EMOE_REQUIRE(L && wg, "set_gate: null argument");
    const size_t bytes = (size_t)L->cfg.num_experts * L->cfg.d_model * L->elem;
    EMOE_CUDA(cudaMemcpy(L->wg, wg, bytes, cudaMemcpyHostToDevice));
    const int E = L->cfg.num_experts;
    if (L->cfg.dtype == EMOE_DTYPE_BF16 && E >= 32 && E % 32 == 0 && E <= 256) {
      if (!L->wg_pad) {
        L->wg_pad = dmalloc<uint8_t>((size_t)256 * L->cfg.d_model * 2);
        EMOE_CUDA(cudaMemset(L->wg_pad, 0, (size_t)256 * L->cfg.d_model * 2));
        // the map covers the E real rows only: the rest of the 256-row B box is
        // out of bounds, zero-filled by the TMA without reading memory (mapping
        // all 256 padded rows doubled the gate's operand bytes at E = 128)
        L->t_gate = make_tmap_bf16_2d(L->wg_pad, E, L->cfg.d_model, 256);
        L->t_gate2 = make_tmap_bf16_2d(L->wg_pad, E, L->cfg.d_model, 128);
        if (E <= 128) L->t_gate_tc = make_tmap_bf16_2d(L->wg_pad, E, L->cfg.d_model, gate_tc_box_rows(E, L->cfg.d_model));
      }
      EMOE_CUDA(cudaMemcpy(L->wg_pad, wg, bytes, cudaMemcpyHostToDevice));
    }
  });
}

int emoe_layer_register_expert_host(emoe_layer* L, int e, const void* w1, const void* w3, const void* w2) {
  return guard([&] {
    EMOE_REQUIRE(L && w1 && w2, "register_expert: null weights");
    EMOE_REQUIRE(e >= 0 && e < L->cfg.num_experts, "register_expert: expert index out of range");
    EMOE_REQUIRE(!L->swiglu() || w3, "register_expert: SwiGLU needs w3");
    const size_t b1 = L->w1_elems() * L->elem, b2 = L->w2_elems() * L->elem;
    if (!L->host_owned[e]) {  // previously a caller pointer: start owning fresh copies
      L->host_w1[e] = L->host_w3[e] = L->host_w2[e] = nullptr;
      L->host_owned[e] = 1;
    }
    auto put = [&](std::vector<void*>& v, const void* src, size_t bytes) {
      if (!v[e]) EMOE_CUDA(cudaHostAlloc(&v[e], bytes, cudaHostAllocDefault));
      std::memcpy(v[e], src, bytes);
    };
    put(L->host_w1, w1, b1);
    if (L->swiglu()) put(L->host_w3, w3, b1);
    put(L->host_w2, w2, b2);
  });
}

int emoe_layer_register_expert_pinned(emoe_layer* L, int e, const void* w1, const void* w3, const void* w2) {
  return guard([&] {
    EMOE_REQUIRE(L && w1 && w2, "register_expert: null weights");
    EMOE_REQUIRE(e >= 0 && e < L->cfg.num_experts, "register_expert: expert index out of range");
    EMOE_REQUIRE(!L->swiglu() || w3, "register_expert: SwiGLU needs w3");
    if (L->host_owned[e])
      for (auto* v : {&L->host_w1, &L->host_w3, &L->host_w2})
        if ((*v)[e]) EMOE_CUDA(cudaFreeHost((*v)[e]));
    L->host_owned[e] = 0;
    L->host_w1[e] = const_cast<void*>(w1);
    L->host_w3[e] = const_cast<void*>(w3);
    L->host_w2[e] = const_cast<void*>(w2);
  });
}

int emoe_layer_set_copy_stream(emoe_layer* L, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L, "set_copy_stream: null layer");
    if (!L->pending_experts.empty()) L->poll(true, L->load_stream(), nullptr);
    L->ext_copy_stream = static_cast<cudaStream_t>(stream);
  });
}

int emoe_layer_set_scores(emoe_layer* L, const double* scores, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L, "set_scores: null layer");
    if (!scores) {  // later route launches pass a null score pointer
      L->have_scores = false;
      return;
    }
    ScoresUpdate u;
    u.E = L->cfg.num_experts;
    for (int e = 0; e < u.E; ++e) u.v[e] = scores[e];
    set_scores_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(u, L->scores_dev);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    L->have_scores = true;
  });
}

int emoe_layer_set_scores_host(emoe_layer* L, const double* scores) {
  const int rc = emoe_layer_set_scores(L, scores, nullptr);
  if (rc != 0) return rc;
  return guard([&] { EMOE_CUDA(cudaStreamSynchronize(nullptr)); });
}

int emoe_layer_begin_load(emoe_layer* L, const int32_t* evictions, int n_ev, const int32_t* loads, int n_ld,
                          void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L, "begin_load: null layer");
    L->begin_load(evictions, n_ev, loads, n_ld, static_cast<cudaStream_t>(stream));
  });
}

int emoe_layer_poll_loads(emoe_layer* L, int blocking, void* stream, int* still_pending) {
  return guard([&] {
    EMOE_REQUIRE(L, "poll_loads: null layer");
    L->poll(blocking != 0, static_cast<cudaStream_t>(stream), still_pending);
  });
}

int emoe_layer_residency(const emoe_layer* L, uint8_t* out) {
  return guard([&] {
    EMOE_REQUIRE(L && out, "residency: null argument");
    std::copy(L->resident.begin(), L->resident.end(), out);
  });
}

int emoe_layer_last_load_stats(const emoe_layer* L, double* bytes, double* ms) {
  return guard([&] {
    EMOE_REQUIRE(L, "last_load_stats: null layer");
    if (bytes) *bytes = L->last_load_bytes;
    if (ms) *ms = L->last_load_ms;
  });
}

int emoe_moe_forward(emoe_layer* L, const void* x, const float* logits_in, void* y, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && y && (x || logits_in), "moe_forward: null argument");
    EMOE_REQUIRE(x, "moe_forward: x is required (the FFN consumes it)");
    L->forward(x, logits_in, y, T, static_cast<cudaStream_t>(stream));
  });
}

int emoe_moe_forward_host(emoe_layer* L, const void* x_host, void* y_host, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && x_host && y_host, "moe_forward_host: null argument");
    EMOE_REQUIRE(T >= 0 && T <= L->cfg.max_tokens, "moe_forward: T exceeds the layer's max_tokens");
    L->forward_host(x_host, y_host, T, static_cast<cudaStream_t>(stream));
  });
}

int emoe_moe_forward_host_async(emoe_layer* L, const void* x_host, void* y_host, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && x_host && y_host, "moe_forward_host_async: null argument");
    L->forward_host_async(x_host, y_host, T, static_cast<cudaStream_t>(stream));
  });
}

int emoe_layer_wait_host(emoe_layer* L) {
  return guard([&] {
    EMOE_REQUIRE(L, "wait_host: null layer");
    L->wait_host();
  });
}

int emoe_route(emoe_layer* L, const void* x, const float* logits_in, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && (x || logits_in), "route: null argument");
    L->poll(false, static_cast<cudaStream_t>(stream), nullptr);
    L->route(x, logits_in, T, static_cast<cudaStream_t>(stream));
  });
}

int emoe_layer_gate_demand(emoe_layer* L, int64_t* counts_host, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && counts_host, "gate_demand: null argument");
    const int E = L->cfg.num_experts;
    EMOE_REQUIRE(E <= kMaxTableE, "gate_demand: too many experts");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!L->demand_dev) L->demand_dev = dmalloc<unsigned long long>(E);
    EMOE_CUDA(cudaMemsetAsync(L->demand_dev, 0, sizeof(unsigned long long) * E, s));
    if (L->last_T > 0) {
      const int blocks = (int)std::min<int64_t>(ceil_div(L->last_T, (int64_t)256), (int64_t)L->num_sms * 4);
      gate_demand_kernel<<<blocks, 256, 0, s>>>(L->topk, L->last_T, L->cfg.top_k, E, L->demand_dev);
      EMOE_CUDA(cudaGetLastError());
      count_launch();
    }
    std::vector<unsigned long long> h(E);
    EMOE_CUDA(cudaMemcpyAsync(h.data(), L->demand_dev, sizeof(unsigned long long) * E, cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
    for (int e = 0; e < E; ++e) counts_host[e] = (int64_t)h[e];
  });
}

int emoe_layer_set_keep_logits(emoe_layer* L, int keep) {
  return guard([&] {
    EMOE_REQUIRE(L, "set_keep_logits: null layer");
    L->keep_logits = keep != 0;
  });
}

int emoe_layer_set_logits_mode(emoe_layer* L, int mode) {
  return guard([&] {
    EMOE_REQUIRE(L, "set_logits_mode: null layer");
    EMOE_REQUIRE(mode == EMOE_LOGITS_REPLACE || mode == EMOE_LOGITS_ADD, "set_logits_mode: unknown mode");
    L->logits_mode = mode;
  });
}

int emoe_layer_set_route_residency(emoe_layer* L, const uint8_t* resident, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L, "set_route_residency: null layer");
    if (!resident) {
      L->route_override = false;
      return;
    }
    const int E = L->cfg.num_experts;
    if (!L->route_resident_dev) L->route_resident_dev = dmalloc<uint8_t>(E);
    L->route_resident.assign(resident, resident + E);
    TableUpdate u;
    u.E = E;
    for (int e = 0; e < E; ++e) {
      u.resident[e] = resident[e] ? 1 : 0;
      u.slot[e] = L->slot_of_expert[e];
    }
    // same parameter-carried update as the slot tables; slot table rewritten unchanged
    set_tables_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(u, L->route_resident_dev, L->slot_dev);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    L->route_override = true;
  });
}

int emoe_route_permute(emoe_layer* L, const void* x, const float* logits_in, int64_t T, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && x, "route_permute: null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    L->poll(false, s, nullptr);
    L->route(x, logits_in, T, s);
    if (T > 0) L->permute(x, T, s);
  });
}

int emoe_ffn_segments(emoe_layer* L, const void* x_rows, int64_t R, const int64_t* seg_offsets, const int32_t* seg_expert,
                      int n_seg, void* h_scratch, void* y_rows, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && seg_offsets && seg_expert, "ffn_segments: null argument");
    EMOE_REQUIRE(n_seg >= 0 && n_seg <= 256, "ffn_segments: n_seg must be in [0, 256]");
    if (n_seg == 0 || R == 0) return;
    EMOE_REQUIRE(x_rows && h_scratch && y_rows, "ffn_segments: null buffer");
    EMOE_REQUIRE(R % L->seg_pad == 0, "ffn_segments: R must be a multiple of the layer's seg_pad");
    const bool was = L->profiling;
    L->profiling = false;  // stage events belong to forward()
    L->ffn(x_rows, R, seg_offsets, seg_expert, n_seg, h_scratch, y_rows, static_cast<cudaStream_t>(stream), false);
    L->profiling = was;
  });
}

int emoe_combine(emoe_layer* L, const void* y_rows, const int32_t* pos, const float* served_w, int64_t T, void* y,
                 void* stream) {
  return guard([&] {
    EMOE_REQUIRE(L && y_rows && pos && served_w && y, "combine: null argument");
    launch_combine(y_rows, L->cfg.dtype, T, L->cfg.d_model, L->cfg.top_k, pos, served_w, y,
                   static_cast<cudaStream_t>(stream));
  });
}

int emoe_layer_workspace(emoe_layer* L, emoe_workspace* w) {
  return guard([&] {
    EMOE_REQUIRE(L && w, "workspace: null argument");
    w->T = L->last_T;
    w->rows_cap = L->rows_cap;
    w->seg_pad = L->seg_pad;
    w->gemm_cta_group = L->cta_group;
    w->logits = L->logits;
    w->topk_idx = L->topk;
    w->route_expert = L->r_expert;
    w->route_rank = L->r_rank;
    w->route_hit = L->r_hit;
    w->served_idx = L->served_idx;
    w->served_w = L->served_w;
    w->counts = L->counts;
    w->seg_offsets = L->seg_offsets;
    w->pos = L->pos;
    w->row_token = L->row_token;
    w->x_perm = L->x_perm;
    w->h = L->h;
    w->y_perm = L->y_perm_valid ? L->y_perm : nullptr;  // null: GEMM2 wrote y directly (top-1 fused combine)
    w->slot_of_expert = L->slot_dev;
    w->resident = L->resident_dev;
    w->fp32_tensor_core = L->tf32 ? 1 : 0;
  });
}

int emoe_layer_set_profiling(emoe_layer* L, int enable) {
  return guard([&] {
    EMOE_REQUIRE(L, "set_profiling: null layer");
    L->profiling = enable != 0;
    L->ev_used = 0;
  });
}

int emoe_layer_stage_times(emoe_layer* L, float* ms) {
  return guard([&] {
    EMOE_REQUIRE(L && ms, "stage_times: null argument");
    EMOE_REQUIRE(L->ev_used > 0, "stage_times: no profiled forward since the last call");
    for (int i = 0; i < 5; ++i) ms[i] = 0.0f;
    for (size_t n = 0; n < L->ev_used; ++n) {
      auto& set = L->ev_pool[n];
      EMOE_CUDA(cudaEventSynchronize(set[5]));
      for (int i = 0; i < 5; ++i) {
        float v = 0;
        EMOE_CUDA(cudaEventElapsedTime(&v, set[i], set[i + 1]));
        ms[i] += v / (float)L->ev_used;
      }
    }
    L->ev_used = 0;
  });
}

int emoe_layer_stage_times_last(emoe_layer* L, float* ms) {
  return guard([&] {
    EMOE_REQUIRE(L && ms, "stage_times: null argument");
    EMOE_REQUIRE(!L->ev_pool.empty(), "stage_times: no profiled forward");
    auto& set = L->ev_pool[0];
    EMOE_CUDA(cudaEventSynchronize(set[5]));
    for (int i = 0; i < 5; ++i) EMOE_CUDA(cudaEventElapsedTime(&ms[i], set[i], set[i + 1]));
  });
}

long long emoe_kernel_launches(void) { return launch_count(); }

int emoe_route_tokens_host(const int32_t* choices, int64_t T, int k, const uint8_t* resident, int E,
                           const double* scores, int32_t* out_expert, int32_t* out_rank, uint8_t* out_hit) {
  return guard([&] {
    EMOE_REQUIRE(E >= 1 && E <= 128, "route_tokens: E must be in [1, 128]");
    EMOE_REQUIRE(k >= 1 && k <= 8, "route_tokens: k must be in [1, 8]");
    for (int64_t i = 0; i < T * k; ++i)
      EMOE_REQUIRE(choices[i] >= 0 && choices[i] < E, "route_tokens: gate choice out of range");
    if (T == 0) return;
    // Per-thread scratch reused across calls (the engine calls route_token per
    // request per layer, engine.cpp:538): one pinned staging block, one device
    // block, one H2D + one D2H copy per call.
    //   in  = [flag i32 | pad | scores f64 x128 | resident u8 x128 | choices i32 x T*k]
    //   out = [expert i32 x T | rank i32 x T | hit u8 x T]
    struct Scratch {
      uint8_t* host = nullptr;
      uint8_t* dev = nullptr;
      size_t cap = 0;
      cudaStream_t s = nullptr;
      ~Scratch() {
        if (host) cudaFreeHost(host);
        if (dev) cudaFree(dev);
        if (s) cudaStreamDestroy(s);
      }
    };
    static thread_local Scratch sc;
    const size_t in_bytes = 16 + 128 * 8 + 128 + (size_t)T * k * 4;
    const size_t in_pad = (in_bytes + 15) / 16 * 16;
    const size_t total = in_pad + (size_t)T * 9;
    if (total > sc.cap) {
      if (sc.host) EMOE_CUDA(cudaFreeHost(sc.host));
      if (sc.dev) EMOE_CUDA(cudaFree(sc.dev));
      const size_t cap = std::max<size_t>(total * 2, 1 << 16);
      EMOE_CUDA(cudaHostAlloc(&sc.host, cap, cudaHostAllocDefault));
      EMOE_CUDA(cudaMalloc(&sc.dev, cap));
      sc.cap = cap;
    }
    if (!sc.s) EMOE_CUDA(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    uint8_t* h = sc.host;
    std::memset(h, 0, 16);
    if (scores) std::memcpy(h + 16, scores, sizeof(double) * E);
    std::memcpy(h + 16 + 1024, resident, E);
    std::memcpy(h + 16 + 1024 + 128, choices, (size_t)T * k * 4);
    EMOE_CUDA(cudaMemcpyAsync(sc.dev, h, in_bytes, cudaMemcpyHostToDevice, sc.s));
    RouteArgs a;
    a.T = T;
    a.d = 0;
    a.E = E;
    a.k = k;
    a.weight_mode = 0;
    a.forced_miss = 0;
    a.resident = sc.dev + 16 + 1024;
    a.scores = scores ? reinterpret_cast<const double*>(sc.dev + 16) : nullptr;
    a.error_flag = reinterpret_cast<int*>(sc.dev);
    uint8_t* out = sc.dev + in_pad;
    RouteOut o{nullptr, nullptr, reinterpret_cast<int32_t*>(out), reinterpret_cast<int32_t*>(out + 4 * T),
               out + 8 * T, nullptr, nullptr, nullptr};
    launch_route_from_choices(reinterpret_cast<const int32_t*>(sc.dev + 16 + 1024 + 128), a, o, sc.s);
    EMOE_CUDA(cudaMemcpyAsync(h, sc.dev, 4, cudaMemcpyDeviceToHost, sc.s));
    EMOE_CUDA(cudaMemcpyAsync(h + in_pad, out, (size_t)T * 9, cudaMemcpyDeviceToHost, sc.s));
    EMOE_CUDA(cudaStreamSynchronize(sc.s));
    int f = 0;
    std::memcpy(&f, h, 4);
    if (f == 3) throw InvariantError("route_token: no resident experts at layer");
    std::memcpy(out_expert, h + in_pad, (size_t)T * 4);
    std::memcpy(out_rank, h + in_pad + 4 * T, (size_t)T * 4);
    std::memcpy(out_hit, h + in_pad + 8 * T, (size_t)T);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// internal interface for the expert-parallel handle (ep.cu)
// ---------------------------------------------------------------------------
namespace emoe {

LayerView layer_view(emoe_layer* L) {
  LayerView v;
  v.E = L->cfg.num_experts;
  v.d = L->cfg.d_model;
  v.f = L->cfg.d_ff;
  v.k = L->cfg.top_k;
  v.dtype = L->cfg.dtype;
  v.elem = L->elem;
  v.seg_pad = L->seg_pad;
  v.max_tokens = L->cfg.max_tokens;
  v.rows_cap = L->rows_cap;
  v.served_idx = L->served_idx;
  v.served_w = L->served_w;
  v.seg_offsets = L->seg_offsets;
  v.block_base = L->block_base;
  v.pos = L->pos;
  v.counts = L->counts;
  return v;
}

void layer_route_scan(emoe_layer* L, const void* x, const float* logits_in, int64_t T, cudaStream_t s) {
  L->poll(false, s, nullptr);
  L->route(x, logits_in, T, s);
  if (T > 0)
    launch_scan(L->block_counts, (int)ceil_div(T, kRouteBlockTokens), L->cfg.num_experts, L->seg_pad, L->counts,
                L->seg_offsets, L->block_base, nullptr, L->counts + L->cfg.num_experts, s);
}

void layer_ffn_chunks(emoe_layer* L, const void* x_chunks, int64_t x_rows, const int64_t* segs,
                      const int32_t* seg_expert, int n_seg, const int64_t* a_shift, void* h, int64_t h_rows,
                      void* y_chunks, int64_t y_rows, cudaStream_t s, cudaEvent_t after_gemm1) {
  EMOE_REQUIRE(L->cfg.dtype == EMOE_DTYPE_BF16, "ffn_chunks: the NCCL EP transport runs the bf16 path");
  const int d = L->cfg.d_model, f = L->cfg.d_ff;
  const CUtensorMap a1 = make_tmap_bf16_2d(x_chunks, (uint64_t)x_rows, d, 128);
  const CUtensorMap o1 = make_tmap_bf16_store(h, (uint64_t)h_rows, f);
  const CUtensorMap a2 = make_tmap_bf16_2d(h, (uint64_t)h_rows, f, 128);
  const CUtensorMap o2 = make_tmap_bf16_store(y_chunks, (uint64_t)y_rows, d);
  // GEMM1: A rows from the receive chunks, H compact; GEMM2: H compact, Y into the return chunks
  launch_grouped_gemm(L->swiglu() ? EPI_SWIGLU : EPI_RELU, L->cta_group, L->gemm_mc, a1, L->tb1, L->tb3, segs,
                      L->slot_dev, n_seg, d, f, f, static_cast<__nv_bfloat16*>(h), f, L->num_sms, s, seg_expert, &o1,
                      nullptr, nullptr, a_shift, nullptr);
  if (after_gemm1) EMOE_CUDA(cudaEventRecord(after_gemm1, s));
  launch_grouped_gemm(EPI_STORE, L->cta_group, L->gemm_mc, a2, L->tb2, L->tb2, segs, L->slot_dev, n_seg, f, d, d,
                      static_cast<__nv_bfloat16*>(y_chunks), d, L->num_sms, s, seg_expert, &o2, nullptr, nullptr,
                      nullptr, a_shift);
}

void layer_ffn_rows(emoe_layer* L, const void* xr, int64_t R, const int64_t* segs, const int32_t* seg_expert,
                    int n_seg, void* hr, void* yr, cudaStream_t s, const PeerOut* peer_out, cudaEvent_t after_gemm1) {
  const bool was = L->profiling;
  L->profiling = false;
  L->ext_mark3 = after_gemm1;
  L->ffn(xr, R, segs, seg_expert, n_seg, hr, yr, s, false, nullptr, peer_out);
  L->ext_mark3 = nullptr;
  L->profiling = was;
}

}  // namespace emoe
