/* emoe.h -- C ABI of the B200-native predicted-residency MoE layer.
 *
 * This is the drop-in boundary for the hot path of the reference `moesim`
 * library (/root/reference/proj/core).  Every entry point names the reference
 * interface it replaces (file:line, relative to /root/reference/proj/core).
 * Signatures are plain C: pointers, sizes and opaque handles; no C++ or torch
 * types.  A C++ compat layer with the exact `moesim::` signatures and the
 * ctypes binding used by the Python host mirror sit on top.
 *
 * Conventions
 *   - Return codes mirror the reference's exception split:
 *       EMOE_OK                 0
 *       EMOE_ERR_RUNTIME        1  CUDA / driver / allocation failure
 *       EMOE_ERR_VALIDATION     2  moesim::ValidationError (types.hpp:11-14)
 *       EMOE_ERR_INVARIANT      3  std::logic_error (expert_store.cpp:47-54, :213)
 *     emoe_last_error() returns the thread-local message of the last failure.
 *   - `_dev` pointers are device pointers and the call is stream-ordered on
 *     `stream` (a cudaStream_t, NULL = legacy default stream).  `_host`
 *     pointers are host memory and the call returns after results are on the
 *     host.
 *   - Element types: `dtype` 0 = bf16, 1 = fp32 for activations and weights;
 *     routing outputs are int32 / uint8 / fp32; predictor state is fp64/int64.
 *   - Threading: one handle per owning thread/stream (Placement mutation is
 *     single-owner); distinct handles are independent.
 */
#ifndef EMOE_H
#define EMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMOE_OK 0
#define EMOE_ERR_RUNTIME 1
#define EMOE_ERR_VALIDATION 2
#define EMOE_ERR_INVARIANT 3

#define EMOE_DTYPE_BF16 0
#define EMOE_DTYPE_F32 1
#define EMOE_ACT_SWIGLU 0
#define EMOE_ACT_RELU 1
#define EMOE_WEIGHTS_TOPK_SOFTMAX 0 /* Mixtral: softmax over the served top-k logits */
#define EMOE_WEIGHTS_FULL_SOFTMAX 1 /* Switch: full-softmax probability of the served expert */

const char* emoe_last_error(void);
int emoe_version(void);

/* ========================================================================
 * A2  route_token  (expert_store.hpp:101-111, expert_store.cpp:206-220)
 * Batched: token t's ranked gate choices are choices[t*k .. t*k+k).
 * resident: [E] 0/1 residency of the layer (Placement::resident_, :41).
 * scores: [E] layer scores or NULL for the empty score vector.
 * Returns EMOE_ERR_INVARIANT when a token needs the fallback and no expert is
 * resident ("route_token: no resident experts at layer").
 * ====================================================================== */
int emoe_route_tokens_host(const int32_t* choices, int64_t T, int k, const uint8_t* resident, int E,
                           const double* scores, int32_t* out_expert, int32_t* out_rank, uint8_t* out_hit);

/* ========================================================================
 * MoE layer handle: gate weights, HBM expert slot pool (budget L), residency
 * table, pinned host copies of every expert, routing/permute workspace.
 * ====================================================================== */
typedef struct emoe_layer emoe_layer;

typedef struct {
  int d_model;     /* d */
  int d_ff;        /* f */
  int num_experts; /* E (ModelShape::experts_per_layer, types.hpp:19) */
  int top_k;       /* k (ModelShape::top_k, types.hpp:20) */
  int activation;  /* EMOE_ACT_* */
  int dtype;       /* EMOE_DTYPE_* */
  int weight_mode; /* EMOE_WEIGHTS_* */
  int num_slots;   /* HBM expert slots = resident budget L (Placement::budget) */
  int64_t max_tokens;
  int forced_miss; /* 1: a layer with no resident expert serves nothing (engine.cpp:533-537) */
  int gemm_cta_group; /* bf16 FFN GEMM: 1 = one CTA per 128x256 tile, 2 = CTA pair per 256x256
                         tile (segments padded to 256 rows), 0 = auto (2 when d_model <= 2048:
                         short-K GEMMs are L2-feed bound; else 1: faster under the 1 kW power
                         cap; profiles/r01_cta_group_ab.jsonl) */
} emoe_layer_config;

int emoe_layer_create(const emoe_layer_config* cfg, emoe_layer** out);
int emoe_layer_destroy(emoe_layer* layer);

/* gate weights W_g [E][d] (layer dtype), host memory */
int emoe_layer_set_gate_host(emoe_layer* layer, const void* wg);
/* expert e's weights, host memory, copied into library-owned pinned buffers:
 * w1, w3: [f][d] (w3 ignored for ReLU), w2: [d][f]  (layer dtype) */
int emoe_layer_register_expert_host(emoe_layer* layer, int expert, const void* w1, const void* w3, const void* w2);

/* Same, but the library keeps the caller's host pointers (no copy): they must
 * stay valid and should be pinned (cudaHostAlloc / cudaHostRegister) for the
 * side-stream copies to overlap compute.  Lets a stack of layers share one
 * pinned copy of the weights. */
int emoe_layer_register_expert_pinned(emoe_layer* layer, int expert, const void* w1, const void* w3, const void* w2);
/* H2D expert loads go to `stream` (NULL = the layer's own copy stream).
 * Layers sharing one copy stream load layer-sequentially, as the engine
 * schedules them (engine.cpp:431-440). */
int emoe_layer_set_copy_stream(emoe_layer* layer, void* stream);

/* What a forward does with caller logits (logits_in of emoe_moe_forward,
 * emoe_route, emoe_route_permute, emoe_ep_forward):
 *   EMOE_LOGITS_REPLACE (default)  routing-driven parity mode: logits_in
 *       replaces the gate (x is still the FFN's input);
 *   EMOE_LOGITS_ADD  the gate runs on x and logits_in [T][E] fp32 is added to
 *       its fp32 logits before top-k (a serving trace imposed as a bias on a
 *       real gate computation); the workspace logits hold the sum. */
/* keep != 0 (default): a forward that computes the gate also stores the fp32
 * logits [T][E] in the workspace (emoe_layer_workspace().logits).  0: the
 * fused tcgen05 gate (E >= 32) routes from its accumulators and skips that
 * store (33.5 MB at the Switch shape); routing outputs are identical. */
int emoe_layer_set_keep_logits(emoe_layer* layer, int keep);

#define EMOE_LOGITS_REPLACE 0
#define EMOE_LOGITS_ADD 1
int emoe_layer_set_logits_mode(emoe_layer* layer, int mode);

/* Layer scores used by the route_token fallback (the engine's last aggregate
 * row, set when an invocation completes: engine.cpp:424, :529-531).
 * scores == NULL sets the empty score vector.  Stream-ordered: the [E]
 * scores travel as the arguments of a kernel enqueued on `stream`, so
 * forwards enqueued earlier on `stream` still route with the old scores and
 * later ones with the new (no host staging buffer, no device-wide sync). */
int emoe_layer_set_scores(emoe_layer* layer, const double* scores, void* stream);
/* Same, then synchronises the legacy default stream (kept for callers of the
 * blocking form). */
int emoe_layer_set_scores_host(emoe_layer* layer, const double* scores);

/* ========================================================================
 * A8  apply_plan_layer / engine load schedule (expert_store.cpp:197-200,
 * engine.cpp:431-464).  Two-phase residency exactly as the engine:
 * evictions take effect at load start (stream-ordered on `stream`), loads
 * become resident at load completion.  The H2D copies of the loaded experts
 * run on the layer's side copy stream from pinned host memory and overlap
 * compute; emoe_layer_poll_loads() flips them resident once complete
 * (blocking = 1 waits).  Loading a resident expert, evicting a non-resident
 * one or exceeding the slot budget returns EMOE_ERR_INVARIANT
 * (Placement::load/evict, expert_store.cpp:46-57).
 * ====================================================================== */
int emoe_layer_begin_load(emoe_layer* layer, const int32_t* evictions, int n_evictions, const int32_t* loads,
                          int n_loads, void* stream);
int emoe_layer_poll_loads(emoe_layer* layer, int blocking, void* stream, int* still_pending);
/* residency as seen by compute: out[E] 0/1 (Placement::residents, :24) */
int emoe_layer_residency(const emoe_layer* layer, uint8_t* out);
/* bytes of the last completed load batch and its H2D time in ms */
int emoe_layer_last_load_stats(const emoe_layer* layer, double* bytes, double* ms);

/* ========================================================================
 * A1-A5  MoE layer forward (replaces the engine iteration's route loop and
 * cost model, engine.cpp:524-546).  x, y: [T][d] in the layer dtype.
 * logits_in (optional): [T][E] fp32 precomputed gate logits (routing-driven
 * parity mode); when NULL the gate is computed from x.
 * ====================================================================== */
int emoe_moe_forward(emoe_layer* layer, const void* x_dev, const float* logits_in_dev, void* y_dev, int64_t T,
                     void* stream);
/* Same through host buffers: H2D of x, forward, D2H of y; returns after y is on the host.
 * Copies and compute are pipelined in token chunks (pinned buffers overlap). */
int emoe_moe_forward_host(emoe_layer* layer, const void* x_host, void* y_host, int64_t T, void* stream);
/* Asynchronous form for serving loops: enqueues H2D, forward and D2H and
 * returns; consecutive calls alternate two device staging sets, so call i+1's
 * H2D overlaps call i's compute and D2H.  x_host must stay unchanged and y_host
 * unread until emoe_layer_wait_host() returns (it waits for every call made).
 * Loads are polled once per call: every chunk of a call sees the same
 * residency, as one emoe_moe_forward over all T tokens would. */
int emoe_moe_forward_host_async(emoe_layer* layer, const void* x_host, void* y_host, int64_t T, void* stream);
int emoe_layer_wait_host(emoe_layer* layer);

/* Route only (A1 + A2): fills the workspace routing fields. */
int emoe_route(emoe_layer* layer, const void* x_dev, const float* logits_in_dev, int64_t T, void* stream);

/* Demand of the last route / forward: counts_host[E] = tokens whose rank-0
 * gate choice is e (the per-layer demand map of the on-demand baseline,
 * engine.cpp:469-478 dynamic_transfers).  Synchronous on `stream`. */
int emoe_layer_gate_demand(emoe_layer* layer, int64_t* counts_host, void* stream);

/* ========================================================================
 * Stage entry points used by expert parallelism: the forward
 * split at its two exchange points.
 *   emoe_route_permute  A1-A3 into the workspace (x_perm, counts,
 *                       seg_offsets, pos, served_w).
 *   emoe_ffn_segments   A4 over caller rows x_rows [R][d]: n_seg segments
 *                       starting at seg_offsets_dev[i] (multiples of the
 *                       layer's seg_pad; seg_offsets_dev[n_seg] = R) served by
 *                       resident expert seg_expert_dev[i]; h_scratch [R][f];
 *                       writes y_rows [R][d].  n_seg <= 256.
 *   emoe_combine        A5: y[t] = sum_j w[t][j] * y_rows[pos[t][j]].
 * ====================================================================== */
int emoe_route_permute(emoe_layer* layer, const void* x_dev, const float* logits_in_dev, int64_t T, void* stream);
/* Expert parallelism: route against the GLOBAL resident set resident[E]
 * (the reference Placement) while this GPU's slots hold only the experts it
 * serves; NULL restores routing against the local slots. */
int emoe_layer_set_route_residency(emoe_layer* layer, const uint8_t* resident, void* stream);
int emoe_ffn_segments(emoe_layer* layer, const void* x_rows_dev, int64_t R, const int64_t* seg_offsets_dev,
                      const int32_t* seg_expert_dev, int n_seg, void* h_scratch_dev, void* y_rows_dev, void* stream);
int emoe_combine(emoe_layer* layer, const void* y_rows_dev, const int32_t* pos_dev, const float* served_w_dev,
                 int64_t T, void* y_dev, void* stream);

/* ========================================================================
 * Expert parallelism over peer memory (replaces the
 * all-to-all exchange of emoe_route_permute / emoe_ffn_segments /
 * emoe_combine with stores and loads into IPC-mapped peer buffers).  The
 * reference has no counterpart (multi-GPU is a non-goal); the
 * forward it extends is the engine's per-layer serve step, engine.cpp:524-546.
 *   emoe_ep_create      one per rank over that rank's layer (its slots hold
 *                       the experts it computes; routing residency set with
 *                       emoe_layer_set_route_residency).  cum_shares[E][world]
 *                       (int64, fixed point 2^24 = 1): cumulative share of
 *                       expert e's rows computed on ranks <= q, non-decreasing
 *                       over q and ending at 2^24; a row of -1 = not resident.
 *                       Each forward splits e's rows (all sources, in source
 *                       order) at those shares, rounded to the segment padding,
 *                       so a hot expert is shared token by token.  recv_rows_cap
 *                       0 = the worst case, world x the layer's rows_cap.
 *                       share_with (NULL or another rank-local handle of the
 *                       same world/rank and layer shape): reuse its symmetric
 *                       region, IPC mappings and epoch -- the layers of a stack
 *                       share one region (open peers once, on the first).
 *                       world <= 8, bf16.
 *   emoe_ep_ipc_handle  this rank's symmetric buffer as an IPC handle
 *                       (EMOE_IPC_HANDLE_BYTES bytes) for the caller to
 *                       all-gather; emoe_ep_open_peers maps the others
 *                       (handles[world][EMOE_IPC_HANDLE_BYTES], own ignored).
 *   emoe_ep_forward     route -> dispatch (permute stores into the computing
 *                       ranks' buffers) -> grouped FFN on the received rows,
 *                       GEMM2 pushing outputs back -> local combine, with three
 *                       device-side barriers; every rank must call it the
 *                       same number of times.  Output bit-identical to the
 *                       single-GPU forward.  No host synchronisation.
 *   emoe_ep_status      synchronises `stream`; *status 0 = ok, 1 = a peer
 *                       barrier timed out (EMOE_EP_TIMEOUT_S, default 60 s),
 *                       2 = a receive buffer overflowed (rows dropped);
 *                       *recv_rows = rows this rank computed last forward.
 *   emoe_ep_stats       synchronises `stream`; out[5] of the last forward:
 *                       rows this rank computed (padded), real rows it sent
 *                       to peers, real rows it received from peers, real rows
 *                       it routed, real rows it computed.
 *   emoe_ep_layout      synchronises `stream`; the last forward's send pieces
 *                       piece_end / piece_shift [E][world] and receive layout
 *                       recv_segs [world*n_owned+1] / out_shift [world*n_owned]
 *                       (any pointer may be NULL; for tests).
 *   emoe_ep_set_profiling / emoe_ep_stage_times   per-forward CUDA events;
 *                       ms[8] averaged over the profiled forwards: route,
 *                       count exchange (bar0), dispatch, dispatch wait,
 *                       gemm1, gemm2 + return pushes, return wait, combine.
 * ====================================================================== */
#define EMOE_IPC_HANDLE_BYTES 64
typedef struct emoe_ep emoe_ep;
int emoe_ep_create(emoe_layer* layer, int world, int rank, const int64_t* cum_shares, int64_t recv_rows_cap,
                   emoe_ep* share_with, emoe_ep** out);
int emoe_ep_ipc_handle(emoe_ep* ep, void* handle_out);
int emoe_ep_open_peers(emoe_ep* ep, const void* handles);
int emoe_ep_forward(emoe_ep* ep, const void* x_dev, const float* logits_in_dev, void* y_dev, int64_t T,
                    void* stream);
int emoe_ep_status(emoe_ep* ep, void* stream, int* status, int64_t* recv_rows);
int emoe_ep_stats(emoe_ep* ep, void* stream, int64_t* out);
int emoe_ep_layout(emoe_ep* ep, void* stream, int64_t* piece_end, int64_t* piece_shift, int64_t* recv_segs,
                   int64_t* out_shift);
int emoe_ep_set_profiling(emoe_ep* ep, int enable);
int emoe_ep_stage_times(emoe_ep* ep, float* ms);
int emoe_ep_destroy(emoe_ep* ep);

/* ========================================================================
 * Expert parallelism over NCCL all-to-all without host synchronisation (the
 * capacity-padded form; the baseline the peer-memory form
 * replaces).  Every (source, destination) pair owns a fixed chunk of cap
 * rows in the caller's send / receive / return buffers ([world][cap][d]
 * bf16), so the caller's all-to-alls take equal splits and no host-side
 * sizes.  Same split (cum_shares) and bit-identical outputs as emoe_ep_*.
 * Per forward, all on one stream:
 *   emoe_epx_route      route + counts (the layer workspace's counts [E] i32);
 *                       the caller all-gathers them into table [world][E]
 *   emoe_epx_dispatch   split layout from the table + permute into the send
 *                       chunks (a pair over cap rows drops the forward's rows on
 *                       every rank: status 2)
 *   (caller: all_to_all send -> receive)
 *   emoe_epx_ffn        grouped FFN over the received chunks, outputs into
 *                       the return chunks (same rows)
 *   (caller: all_to_all return -> returned)
 *   emoe_epx_combine    local combine from the returned chunks
 * cap_rows 0 = the layer's rows_cap (every pair may carry all of a source's
 * rows); emoe_epx_cap_rows reads the padded value back. */
typedef struct emoe_epx emoe_epx;
int emoe_epx_create(emoe_layer* layer, int world, int rank, const int64_t* cum_shares, int64_t cap_rows,
                    emoe_epx** out);
int emoe_epx_cap_rows(const emoe_epx* x, int64_t* cap_rows);
int emoe_epx_route(emoe_epx* x, const void* x_dev, const float* logits_in_dev, int64_t T, void* stream);
int emoe_epx_dispatch(emoe_epx* x, const int32_t* table_dev, const void* x_dev, int64_t T, void* send_chunks_dev,
                      void* stream);
int emoe_epx_ffn(emoe_epx* x, const void* recv_chunks_dev, void* return_chunks_dev, void* stream);
int emoe_epx_combine(emoe_epx* x, const void* returned_chunks_dev, void* y_dev, int64_t T, void* stream);
int emoe_epx_status(emoe_epx* x, void* stream, int* status, int64_t* rows_computed);
int emoe_epx_destroy(emoe_epx* x);

/* Device pointers of the last forward's intermediates (valid until the next
 * call on the layer).  Sizes: T tokens, R = rows_cap permuted rows. */
typedef struct {
  int64_t T;
  int64_t rows_cap;
  int64_t seg_pad;        /* per-expert segment padding (rows) */
  int64_t gemm_cta_group; /* CTA group the FFN GEMMs run with */
  float* logits;          /* [T][E] */
  int32_t* topk_idx;      /* [T][k] gate choices, rank order */
  int32_t* route_expert;  /* [T] RouteResult.expert */
  int32_t* route_rank;    /* [T] RouteResult.rank (-1 = fallback) */
  uint8_t* route_hit;     /* [T] RouteResult.hit */
  int32_t* served_idx;    /* [T][k] served experts, -1 = empty slot */
  float* served_w;        /* [T][k] served gate weights */
  int32_t* counts;        /* [E] served rows per expert */
  int64_t* seg_offsets;   /* [E+1] padded segment starts */
  int32_t* pos;           /* [T][k] permuted row of each served slot, -1 = none */
  int32_t* row_token;     /* [R] source token of each permuted row, -1 = padding */
  void* x_perm;           /* [R][d] */
  void* h;                /* [R][f] */
  void* y_perm;           /* [R][d]; NULL after a top-1 bf16 forward, whose
                             GEMM2 epilogue writes y directly (fused combine) */
  int32_t* slot_of_expert; /* [E] HBM slot, -1 = not resident */
  uint8_t* resident;      /* [E] */
  int64_t fp32_tensor_core; /* fp32 layer: 1 = FFN GEMMs on tcgen05 (3xTF32), 0 = SIMT FFMA */
} emoe_workspace;
int emoe_layer_workspace(emoe_layer* layer, emoe_workspace* out);

/* Run `layer` on `donor`'s workspace (routing outputs, permutation and the
 * FFN row buffers: ~6.5 GB for a Mixtral-shaped layer at 65,536 tokens)
 * instead of its own, which is released: a stack of layers executed one
 * after another on one stream needs one workspace, not one per layer.  Same
 * shape, dtype, max_tokens and GEMM tiling required; the donor must outlive
 * the borrower and the two must not run concurrently.  The workspace views
 * (emoe_layer_workspace) of both then describe whichever ran last. */
int emoe_layer_share_workspace(emoe_layer* layer, const emoe_layer* donor);

/* Measurement hooks (no reference counterpart): CUDA events between the
 * forward's stages on the forward's stream; ms[5] = route, scan+permute,
 * FFN GEMM1, FFN GEMM2, combine, averaged over the profiled forwards since
 * the previous emoe_layer_stage_times call. */
int emoe_layer_set_profiling(emoe_layer* layer, int enable);
int emoe_layer_stage_times(emoe_layer* layer, float* ms);
/* The stage times of the first profiled forward's event set without
 * recycling it: for a forward captured once (profiling on) into a CUDA graph,
 * read after each replay -- the events are record nodes of the graph, so every
 * replay re-stamps them with no host launch gaps between the stages. */
int emoe_layer_stage_times_last(emoe_layer* layer, float* ms);
/* kernels launched by this library since load (gpu_launches evidence) */
long long emoe_kernel_launches(void);

/* ========================================================================
 * A6-A8  predictor: popularity histograms over routing history, prediction,
 * Eq. 2, resident-set selection and load planning.
 * ====================================================================== */
typedef struct emoe_predictor emoe_predictor;

/* TransitionModel (predictor.hpp:25-38): m layers, E experts, top_k,
 * smoothing; num_tasks labels (indices into the caller's lexicographically
 * sorted task ids = std::map order). */
int emoe_predictor_create(int num_layers, int num_experts, int top_k, int num_tasks, double smoothing,
                          emoe_predictor** out);
int emoe_predictor_destroy(emoe_predictor* pred);
int emoe_predictor_reset(emoe_predictor* pred);
/* End the prompt chain: the next emoe_hist_update does not count a
 * transition from the last prompt seen (an empty prompt in the reference
 * breaks the chain, predictor.cpp:176-178). */
int emoe_predictor_break_chain(emoe_predictor* pred);

/* fit (predictor.cpp:137-185) as an incremental histogram on the GPU.
 * trace_dev: [P][m][T][k] int32 routing history, task_ids_dev: [P] or NULL.
 * Successive calls continue the prompt chain, so fit over a concatenation
 * equals the sum of the calls (counts commute, test_predictor.cpp:284-296). */
int emoe_hist_update(emoe_predictor* pred, const int32_t* trace_dev, int P, int T, const int32_t* task_ids_dev,
                     void* stream);
/* Same from host memory (copied to the device; returns when the update is done). */
int emoe_hist_update_host(emoe_predictor* pred, const int32_t* trace_host, int P, int T, const int32_t* task_ids_host);
/* Export the tallies (exact integers as doubles): layer [(m-1)][E][E],
 * prompt [m][E][E], task [num_tasks][m][E]. */
int emoe_predictor_counts_host(emoe_predictor* pred, double* layer_counts, double* prompt_counts,
                               double* task_counts);
/* Load tallies (e.g. from a saved TransitionModel). */
int emoe_predictor_set_counts_host(emoe_predictor* pred, const double* layer_counts, const double* prompt_counts,
                                   const double* task_counts);

/* The tallies as one int64 device vector [layer | prompt | task] of
 * emoe_predictor_count_size() entries, stream-ordered after pending
 * histogram updates.  Multi-GPU: each rank fits its own prompts and the
 * ranks sum their deltas with one all-reduce (counts commute,
 * test_predictor.cpp:284-296), so A7/A8 then run identically
 * on every rank (paper_2503_06823_b200/ep.py HistogramSync). */
int emoe_predictor_count_size(emoe_predictor* pred, int64_t* n);
int emoe_predictor_counts_dev(emoe_predictor* pred, int64_t* dst_dev, void* stream);
int emoe_predictor_set_counts_dev(emoe_predictor* pred, const int64_t* src_dev, void* stream);

/* dominant_expert / prompt_expert_sets (workload.cpp:350-377) for one prompt
 * of a device trace [P][m][T][k]: dominant [m], sets [m][k] (-1 padded), sizes [m]. */
int emoe_prompt_expert_sets(const int32_t* trace_dev, int P, int m, int T, int k, int prompt, int32_t* dominant_host,
                            int32_t* sets_host, int32_t* sizes_host, void* stream);
/* Same for one prompt in host memory [m][T][k] (T = 0 allowed: dominant 0,
 * empty sets, as the reference); expert indices must be < 1024. */
int emoe_prompt_expert_sets_host(const int32_t* trace_prompt_host, int m, int T, int k, int32_t* dominant_host,
                                 int32_t* sets_host, int32_t* sizes_host);

/* predict_all_layers (mode 0) / predict_chained (mode 1) / predict_layerwise
 * (mode 2, `layer`) (predictor.cpp:187-220).  prev_sets [m][k] + sizes [m].
 * Outputs scores [m][E] and experts [m][k] (+ counts [m]). */
int emoe_predict_host(emoe_predictor* pred, int mode, const int32_t* prev_sets, const int32_t* prev_sizes, int layer,
                      double* scores, int32_t* experts, int32_t* n_experts);
/* predicted_frequencies (predictor.cpp:222-238); task = -1 for an unseen task */
int emoe_predicted_frequencies_host(emoe_predictor* pred, int task, double* out);

/* expected_tokens Eq. 2 (expert_store.cpp:59-106).  Tasks are indices into
 * the sorted profile list: wo [n_tasks], sensitivity [n_tasks][m] with
 * has_sens[i] = 0 for an empty vector; requests (running then incoming) as
 * task index + input tokens; freqs [n_tasks][m][E] with freq_present[i]. */
int emoe_expected_tokens_host(int m, int E, int n_tasks, const double* wo, const int32_t* sensitivity,
                              const uint8_t* has_sens, int n_requests, const int32_t* req_task,
                              const int32_t* req_tokens, const uint8_t* freq_present, const double* freqs,
                              int task_aware, double* aggregate);
/* select_experts / loading_targets (expert_store.cpp:111-157): out [m][E] */
int emoe_select_experts_host(const double* aggregate, int m, int E, const int32_t* budgets, int32_t* out);
int emoe_loading_targets_host(const double* aggregate, int m, int E, const uint8_t* resident, const int32_t* budgets,
                              int32_t* out, int32_t* sizes);
/* plan_loading (expert_store.cpp:159-195) */
int emoe_plan_loading_host(const uint8_t* resident, const int32_t* budgets, int m, int E, const int32_t* target,
                           const int32_t* target_sizes, const double* aggregate, double per_expert_seconds,
                           int32_t* evictions, int32_t* n_evict, int32_t* loads, int32_t* n_load, double* duration,
                           double* delta_e, int32_t* total_loads);

/* One predictor invocation of the engine (engine.cpp:367-446) on the GPU:
 * predict from the previous prompt's expert sets (mode 0 all-layers, 1
 * chained), modulate by each profile's fitted frequencies, Eq. 2 over the
 * requests, loading_targets against `resident` and plan_loading.  Outputs
 * the aggregate [m][E] and the plan (evictions/loads [m][E] + counts). */
int emoe_invocation_host(emoe_predictor* pred, int mode, const int32_t* prev_sets, const int32_t* prev_sizes,
                         int n_tasks, const double* wo, const int32_t* sensitivity, const uint8_t* has_sens,
                         int n_requests, const int32_t* req_task, const int32_t* req_tokens, int task_aware,
                         const uint8_t* resident, const int32_t* budgets, double per_expert_seconds,
                         double* aggregate, int32_t* evictions, int32_t* n_evict, int32_t* loads, int32_t* n_load,
                         double* delta_e);

/* ========================================================================
 * Workload generator (workload.cpp:242-286, :455): the reference's Markov
 * routing trace, bit-identical (std::mt19937_64), used for synthetic inputs.
 * out: [P][m][T][k] host int32.
 * ====================================================================== */
int emoe_gen_routing_trace(int m, int E, int k, double layer_lambda, double prompt_lambda, int initial_expert,
                           uint64_t seed, int P, int T, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* EMOE_H */
