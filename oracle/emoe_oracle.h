/* emoe CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithm for the predicted-residency
 * MoE layer.  Only tests/, the smoke() check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may
 * load this library, and only as the checker or the timed CPU baseline --
 * never as the product path.  The product (paper_2503_06823_b200/) never links
 * or loads it and fails loudly when its CUDA library is missing.
 *
 * Parity pinning: rows A2, A6, A7, A8 restate reference functions
 * (file:line cited per function in emoe_oracle.c) and are checked bit for bit
 * against the reference itself built here (oracle/_ref/libmoesim_ref.so) and
 * against the golden fixtures in tests/golden/.  Rows A1, A3, A4, A5 have no
 * reference arithmetic (the reference reads routing from a trace and models the
 * FFN as a cost): their semantics are defined in DESIGN.md and parity for them
 * is "unpinned" by construction.
 *
 * Return codes: 0 ok, 2 validation error, 3 invariant (logic) error.
 */
#ifndef EMOE_ORACLE_H
#define EMOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* host threads used by the FP oracle loops (0 = all online cores) */
void oracle_set_threads(int n);
int oracle_get_threads(void);

/* ---- A2: route_token (expert_store.cpp:206-220) ---- */
int oracle_route_tokens(const int32_t* choices, int64_t T, int k, const uint8_t* resident, int E,
                        const double* scores, int n_scores, int32_t* out_expert, int32_t* out_rank,
                        uint8_t* out_hit);

/* ---- A1 + A2 k-slot extension (builder-defined) ----
 * weight_mode 0 = softmax over the served subset of the top-k logits (Mixtral)
 * weight_mode 1 = full-softmax probability of each served expert (Switch)
 * forced_miss: when the layer has no residents, RouteResult = {choice0,-1,0}
 * and no slot is served (engine.cpp:533-537) instead of an invariant error. */
int oracle_gate_route(const float* logits, int64_t T, int E, int k, int weight_mode,
                      const uint8_t* resident, const double* scores, int n_scores, int forced_miss,
                      int32_t* topk_idx, float* topk_logit, int32_t* route_expert,
                      int32_t* route_rank, uint8_t* route_hit, int32_t* served_idx,
                      float* served_w, int32_t* counts);

/* ---- A1 gate logits: logits[t][e] = sum_i x[t][i] * wg[e][i] (double accumulate) ---- */
void oracle_gate_logits_f32(const float* x, const float* wg, int64_t T, int d, int E, float* logits);

/* ---- A3 permutation (builder-defined): segments padded to `pad` rows ---- */
int oracle_permute(const int32_t* served_idx, int64_t T, int k, int E, int pad, int32_t* counts,
                   int64_t* offsets, int64_t* pos, int32_t* perm_src, int64_t rows_cap,
                   int64_t* rows_used);

/* ---- A4 expert FFN for a batch of rows (double accumulate).
 * act 0 = SwiGLU (w1,w3: [f][d], w2: [d][f]); act 1 = ReLU (w1: [f][d], w2: [d][f]).
 * round_bf16: round H and Y to bf16 (mirrors the bf16 kernels' rounding points). */
void oracle_expert_ffn(const float* x, int64_t rows, int d, int f, const float* w1, const float* w3,
                       const float* w2, int act, int round_bf16, float* y, int threads);

/* ---- A5 combine: y[t] = sum_j w_j * Y[pos(t,j)], fixed slot order, fp32 ---- */
void oracle_combine(const float* Y, int d, const int64_t* pos, const float* served_w, int64_t T,
                    int k, int round_bf16, float* y);

/* ---- A6 fit (predictor.cpp:137-185), dominant_expert / prompt_expert_sets
 * (workload.cpp:350-377).  trace is [P][m][T][k]. task_ids: per-prompt index
 * into the caller's sorted task list or NULL. */
int oracle_fit(const int32_t* trace, int P, int m, int T, int k, const int32_t* task_ids,
               int n_tasks, int num_experts, int32_t* out_E, double* layer_counts,
               double* prompt_counts, double* task_counts);
int oracle_dominant_expert(const int32_t* trace, int P, int m, int T, int k, int prompt, int layer);
int oracle_prompt_expert_sets(const int32_t* trace, int P, int m, int T, int k, int prompt,
                              int32_t* sets, int32_t* set_sizes);

/* ---- A7 predictor query (predictor.cpp:13-238) ---- */
int oracle_predict(int m, int E, int k, double smoothing, const double* layer_counts,
                   const double* prompt_counts, int mode, const int32_t* prev_sets,
                   const int32_t* prev_sizes, int layer, double* scores, int32_t* experts,
                   int32_t* n_experts);
int oracle_predicted_frequencies(int m, int E, int n_tasks, const double* task_counts,
                                 double smoothing, int task, double* out);

/* ---- A7 Eq. 2 expected_tokens (expert_store.cpp:59-106): tasks are indices
 * into the caller's lexicographically sorted profile list; freq_present[i]==0
 * means task i has no frequency rows (uniform 1/E). Request task -1 = unknown. */
int oracle_expected_tokens(int m, int E, int n_tasks, const double* wo, const int32_t* sensitivity,
                           const uint8_t* has_sens, int n_requests, const int32_t* req_task,
                           const int32_t* req_tokens, const uint8_t* freq_present,
                           const double* freqs, int task_aware, double* aggregate);

/* ---- A7 select_experts / loading_targets (expert_store.cpp:111-157) ---- */
int oracle_select_experts(const double* aggregate, int m, int E, const int32_t* budgets, int32_t* out);
int oracle_loading_targets(const double* aggregate, int m, int E, const uint8_t* resident,
                           const int32_t* budgets, int32_t* out, int32_t* sizes);

/* ---- A8 plan_loading (expert_store.cpp:159-195) ---- */
int oracle_plan_loading(const uint8_t* resident, const int32_t* budgets, int m, int E,
                        const int32_t* target, const int32_t* target_sizes, const double* aggregate,
                        double per_expert_seconds, int32_t* evictions, int32_t* n_evict,
                        int32_t* loads, int32_t* n_load, double* duration, double* delta_e,
                        int32_t* total_loads);

/* ---- engine invocation_aggregate (engine.cpp:367-417) for predictor modes:
 * pred_scores [m][E] (prediction score rows), fitted [n_tasks][m][E]
 * (predicted_frequencies per profile), then Eq. 2. ---- */
int oracle_invocation_aggregate(int m, int E, int n_tasks, const double* pred_scores,
                                const double* fitted, const double* wo, const int32_t* sensitivity,
                                const uint8_t* has_sens, int n_requests, const int32_t* req_task,
                                const int32_t* req_tokens, int task_aware, double* aggregate);

#ifdef __cplusplus
}
#endif
#endif
