/* emoe CPU oracle -- TEST INFRASTRUCTURE ONLY (see emoe_oracle.h).
 *
 * Compiled with -ffp-contract=off and no -march so fp64 expressions evaluate
 * exactly as the reference's ISO C++20 Release build does (no FMA contraction,
 * SURVEY.md section 2 build row).  Every function cites the reference lines it
 * restates; loop and summation orders follow the reference literally.
 */
#include "emoe_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

/* Minimal pthread parallel-for (libgomp is not available in this image). */
typedef void (*range_fn)(int64_t lo, int64_t hi, void* ctx);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t lo, hi;
} range_job;

static void* range_worker(void* p) {
  range_job* j = (range_job*)p;
  j->fn(j->lo, j->hi, j->ctx);
  return NULL;
}

static int g_threads = 0;

static int oracle_threads(void) {
  if (g_threads > 0) return g_threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void parallel_for(int64_t n, range_fn fn, void* ctx) {
  int nt = oracle_threads();
  if (nt > n) nt = (int)(n > 0 ? n : 1);
  if (nt <= 1) {
    fn(0, n, ctx);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
  range_job* jobs = (range_job*)malloc(sizeof(range_job) * (size_t)nt);
  for (int i = 0; i < nt; ++i) {
    jobs[i].fn = fn;
    jobs[i].ctx = ctx;
    jobs[i].lo = n * i / nt;
    jobs[i].hi = n * (i + 1) / nt;
    pthread_create(&th[i], NULL, range_worker, &jobs[i]);
  }
  for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  free(th);
  free(jobs);
}

void oracle_set_threads(int n) { g_threads = n; }
int oracle_get_threads(void) { return oracle_threads(); }

static _Thread_local char g_err[256];

const char* oracle_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

#define VALIDATION 2
#define INVARIANT 3

static inline int64_t tidx(int m, int T, int k, int p, int l, int t, int r) {
  return (((int64_t)p * m + l) * T + t) * k + r;
}

/* ------------------------------------------------------------------------ */
/* A2: route_token, expert_store.cpp:206-220                                 */
/* ------------------------------------------------------------------------ */
static int route_one(const int32_t* choice, int k, const uint8_t* resident, int E,
                     const double* scores, int n_scores, int32_t* ex, int32_t* rk, uint8_t* hit) {
  for (int r = 0; r < k; ++r) {
    if (resident[choice[r]]) { /* first resident gate choice wins (:207-210) */
      *ex = choice[r];
      *rk = r;
      *hit = (uint8_t)(r == 0);
      return 0;
    }
  }
  int best = -1; /* residents[0] = smallest resident index (:211-213) */
  for (int e = 0; e < E; ++e)
    if (resident[e]) {
      best = e;
      break;
    }
  if (best < 0) return fail(INVARIANT, "route_token: no resident experts at layer");
  if (n_scores > 0) /* strict '>' keeps the smallest index on ties (:214-217) */
    for (int e = 0; e < E; ++e)
      if (resident[e] && scores[e] > scores[best]) best = e;
  *ex = best;
  *rk = -1;
  *hit = 0;
  return 0;
}

int oracle_route_tokens(const int32_t* choices, int64_t T, int k, const uint8_t* resident, int E,
                        const double* scores, int n_scores, int32_t* out_expert, int32_t* out_rank,
                        uint8_t* out_hit) {
  for (int64_t t = 0; t < T; ++t) {
    int rc = route_one(choices + t * k, k, resident, E, scores, n_scores, out_expert + t,
                       out_rank + t, out_hit + t);
    if (rc) return rc;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* A1 + A2: gate top-k on logits + residency remap + weights (builder rule)  */
/* ------------------------------------------------------------------------ */
int oracle_gate_route(const float* logits, int64_t T, int E, int k, int weight_mode,
                      const uint8_t* resident, const double* scores, int n_scores, int forced_miss,
                      int32_t* topk_idx, float* topk_logit, int32_t* route_expert,
                      int32_t* route_rank, uint8_t* route_hit, int32_t* served_idx,
                      float* served_w, int32_t* counts) {
  if (k < 1 || k > E || k > 8) return fail(VALIDATION, "gate_route: k must be in [1, min(E, 8)]");
  int n_res = 0;
  for (int e = 0; e < E; ++e) n_res += resident[e] ? 1 : 0;
  for (int e = 0; e < E; ++e) counts[e] = 0;
  for (int64_t t = 0; t < T; ++t) {
    const float* lg = logits + t * E;
    int32_t* ti = topk_idx + t * k;
    /* top-k by descending logit, ascending index on ties */
    for (int r = 0; r < k; ++r) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        int used = 0;
        for (int q = 0; q < r; ++q) used |= (ti[q] == e);
        if (used) continue;
        if (best < 0 || lg[e] > lg[best]) best = e;
      }
      ti[r] = best;
      topk_logit[t * k + r] = lg[best];
    }
    int32_t ex, rk;
    uint8_t hit;
    if (n_res == 0) {
      if (!forced_miss) return fail(INVARIANT, "route_token: no resident experts at layer");
      ex = ti[0]; /* engine forced miss, engine.cpp:533-537 */
      rk = -1;
      hit = 0;
    } else {
      int rc = route_one(ti, k, resident, E, scores, n_scores, &ex, &rk, &hit);
      if (rc) return rc;
    }
    route_expert[t] = ex;
    route_rank[t] = rk;
    route_hit[t] = hit;
    /* served set: resident choices in rank order, else the fallback expert */
    int32_t* si = served_idx + t * k;
    float* sw = served_w + t * k;
    int ns = 0;
    for (int r = 0; r < k; ++r) {
      si[r] = -1;
      sw[r] = 0.0f;
    }
    if (n_res > 0) {
      if (rk >= 0) {
        for (int r = 0; r < k; ++r)
          if (resident[ti[r]]) si[ns++] = ti[r];
      } else {
        si[ns++] = ex;
      }
    }
    if (weight_mode == 0) {
      /* softmax over the served subset; its max is the first served logit */
      if (ns > 0) {
        float mx = lg[si[0]];
        float den = 0.0f;
        float ev[8];
        for (int j = 0; j < ns; ++j) {
          ev[j] = expf(lg[si[j]] - mx);
          den += ev[j];
        }
        for (int j = 0; j < ns; ++j) sw[j] = ev[j] / den;
      }
    } else {
      float mx = lg[ti[0]];
      float den = 0.0f;
      for (int e = 0; e < E; ++e) den += expf(lg[e] - mx);
      for (int j = 0; j < ns; ++j) sw[j] = expf(lg[si[j]] - mx) / den;
    }
    for (int j = 0; j < ns; ++j) counts[si[j]] += 1;
  }
  return 0;
}

typedef struct {
  const float *x, *wg;
  int d, E;
  float* logits;
} logits_ctx;

static void logits_range(int64_t lo, int64_t hi, void* p) {
  logits_ctx* c = (logits_ctx*)p;
  for (int64_t t = lo; t < hi; ++t)
    for (int e = 0; e < c->E; ++e) {
      double acc = 0.0;
      for (int i = 0; i < c->d; ++i) acc += (double)c->x[t * c->d + i] * (double)c->wg[(int64_t)e * c->d + i];
      c->logits[t * c->E + e] = (float)acc;
    }
}

void oracle_gate_logits_f32(const float* x, const float* wg, int64_t T, int d, int E, float* logits) {
  logits_ctx c = {x, wg, d, E, logits};
  parallel_for(T, logits_range, &c);
}

/* ------------------------------------------------------------------------ */
/* A3: stable permutation into padded per-expert segments (builder-defined)  */
/* ------------------------------------------------------------------------ */
int oracle_permute(const int32_t* served_idx, int64_t T, int k, int E, int pad, int32_t* counts,
                   int64_t* offsets, int64_t* pos, int32_t* perm_src, int64_t rows_cap,
                   int64_t* rows_used) {
  if (pad < 1) return fail(VALIDATION, "permute: pad must be >= 1");
  for (int e = 0; e < E; ++e) counts[e] = 0;
  for (int64_t i = 0; i < T * k; ++i)
    if (served_idx[i] >= 0) counts[served_idx[i]] += 1;
  offsets[0] = 0;
  for (int e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + ((int64_t)(counts[e] + pad - 1) / pad) * pad;
  *rows_used = offsets[E];
  if (offsets[E] > rows_cap) return fail(VALIDATION, "permute: rows exceed capacity");
  for (int64_t r = 0; r < offsets[E]; ++r) perm_src[r] = -1;
  int64_t* cursor = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  for (int64_t t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) {
      int e = served_idx[t * k + j];
      if (e < 0) {
        pos[t * k + j] = -1;
        continue;
      }
      int64_t row = offsets[e] + cursor[e]++;
      pos[t * k + j] = row;
      perm_src[row] = (int32_t)t;
    }
  free(cursor);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* A4: expert FFN rows; A5: combine                                          */
/* ------------------------------------------------------------------------ */
static inline float bf16_round(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return v; /* inf / nan pass through */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

typedef struct {
  const float *x, *w1, *w3, *w2;
  int d, f, act, round_bf16;
  float *h, *y;
} ffn_ctx;

static void ffn_h_range(int64_t lo, int64_t hi, void* p) { /* index = r * f + j */
  ffn_ctx* c = (ffn_ctx*)p;
  for (int64_t idx = lo; idx < hi; ++idx) {
    int64_t r = idx / c->f;
    int j = (int)(idx % c->f);
    const float* xr = c->x + r * c->d;
    const float* a = c->w1 + (int64_t)j * c->d;
    double g = 0.0;
    for (int i = 0; i < c->d; ++i) g += (double)xr[i] * (double)a[i];
    float hv;
    if (c->act == 0) {
      const float* b = c->w3 + (int64_t)j * c->d;
      double u = 0.0;
      for (int i = 0; i < c->d; ++i) u += (double)xr[i] * (double)b[i];
      float gf = (float)g, uf = (float)u;
      hv = gf / (1.0f + expf(-gf)) * uf;
    } else {
      float gf = (float)g;
      hv = gf > 0.0f ? gf : 0.0f;
    }
    c->h[idx] = c->round_bf16 ? bf16_round(hv) : hv;
  }
}

static void ffn_y_range(int64_t lo, int64_t hi, void* p) { /* index = r * d + o */
  ffn_ctx* c = (ffn_ctx*)p;
  for (int64_t idx = lo; idx < hi; ++idx) {
    int64_t r = idx / c->d;
    int o = (int)(idx % c->d);
    const float* hr = c->h + r * c->f;
    const float* w = c->w2 + (int64_t)o * c->f;
    double acc = 0.0;
    for (int j = 0; j < c->f; ++j) acc += (double)hr[j] * (double)w[j];
    float yv = (float)acc;
    c->y[idx] = c->round_bf16 ? bf16_round(yv) : yv;
  }
}

void oracle_expert_ffn(const float* x, int64_t rows, int d, int f, const float* w1, const float* w3,
                       const float* w2, int act, int round_bf16, float* y, int threads) {
  int saved = g_threads;
  if (threads > 0) g_threads = threads;
  ffn_ctx c = {x, w1, w3, w2, d, f, act, round_bf16, NULL, y};
  c.h = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)f);
  parallel_for(rows * f, ffn_h_range, &c);
  parallel_for(rows * d, ffn_y_range, &c);
  free(c.h);
  g_threads = saved;
}

void oracle_combine(const float* Y, int d, const int64_t* pos, const float* served_w, int64_t T,
                    int k, int round_bf16, float* y) {
  for (int64_t t = 0; t < T; ++t)
    for (int i = 0; i < d; ++i) {
      float acc = 0.0f;
      for (int j = 0; j < k; ++j) {
        int64_t p = pos[t * k + j];
        if (p < 0) continue;
        acc += served_w[t * k + j] * Y[p * d + i];
      }
      y[t * d + i] = round_bf16 ? bf16_round(acc) : acc;
    }
}

/* ------------------------------------------------------------------------ */
/* A6: fit (predictor.cpp:137-185), dominant/sets (workload.cpp:350-377)     */
/* ------------------------------------------------------------------------ */
int oracle_dominant_expert(const int32_t* trace, int P, int m, int T, int k, int prompt, int layer) {
  (void)P;
  /* count vector grows to the largest rank-0 index seen (:351-356) */
  int size = 0;
  for (int t = 0; t < T; ++t) {
    int e = trace[tidx(m, T, k, prompt, layer, t, 0)];
    if (e + 1 > size) size = e + 1;
  }
  if (size == 0) return 0;
  int* count = (int*)calloc((size_t)size, sizeof(int));
  for (int t = 0; t < T; ++t) ++count[trace[tidx(m, T, k, prompt, layer, t, 0)]];
  int best = 0;
  for (int e = 1; e < size; ++e)
    if (count[e] > count[best]) best = e; /* strict: smallest index on ties */
  free(count);
  return best;
}

int oracle_prompt_expert_sets(const int32_t* trace, int P, int m, int T, int k, int prompt,
                              int32_t* sets, int32_t* set_sizes) {
  (void)P;
  for (int l = 0; l < m; ++l) {
    int size = 0;
    for (int t = 0; t < T; ++t) {
      int e = trace[tidx(m, T, k, prompt, l, t, 0)];
      if (e + 1 > size) size = e + 1;
    }
    int* count = (int*)calloc((size_t)(size > 0 ? size : 1), sizeof(int));
    for (int t = 0; t < T; ++t) ++count[trace[tidx(m, T, k, prompt, l, t, 0)]];
    /* items sorted by count desc, index asc (:368-372); take up to top_k */
    int n = 0;
    for (int r = 0; r < k; ++r) {
      int best = -1;
      for (int e = 0; e < size; ++e) {
        if (count[e] <= 0) continue;
        int used = 0;
        for (int q = 0; q < n; ++q) used |= (sets[l * k + q] == e);
        if (used) continue;
        if (best < 0 || count[e] > count[best]) best = e;
      }
      if (best < 0) break;
      sets[l * k + n++] = best;
    }
    for (int r = n; r < k; ++r) sets[l * k + r] = -1;
    set_sizes[l] = n;
    free(count);
  }
  return 0;
}

int oracle_fit(const int32_t* trace, int P, int m, int T, int k, const int32_t* task_ids,
               int n_tasks, int num_experts, int32_t* out_E, double* layer_counts,
               double* prompt_counts, double* task_counts) {
  if (P == 0 || m < 1) return fail(VALIDATION, "predictor.trace: empty");
  int E = num_experts;
  if (E <= 0) /* infer from the largest index seen (:144-150) */
    for (int64_t i = 0; i < (int64_t)P * m * T * k; ++i)
      if (trace[i] + 1 > E) E = trace[i] + 1;
  if (E < 1) return fail(VALIDATION, "predictor.trace: no experts");
  *out_E = E;
  memset(layer_counts, 0, sizeof(double) * (size_t)(m > 1 ? m - 1 : 0) * E * E);
  memset(prompt_counts, 0, sizeof(double) * (size_t)m * E * E);
  if (task_ids) memset(task_counts, 0, sizeof(double) * (size_t)n_tasks * m * E);
  for (int p = 0; p < P; ++p) {
    for (int l = 0; l + 1 < m; ++l) /* rank-0 layer transitions (:164-166) */
      for (int t = 0; t < T; ++t) {
        int a = trace[tidx(m, T, k, p, l, t, 0)];
        int b = trace[tidx(m, T, k, p, l + 1, t, 0)];
        layer_counts[((int64_t)l * E + a) * E + b] += 1.0;
      }
    if (task_ids) { /* every rank of every token (:167-173) */
      double* rows = task_counts + (int64_t)task_ids[p] * m * E;
      for (int l = 0; l < m; ++l)
        for (int t = 0; t < T; ++t)
          for (int r = 0; r < k; ++r) rows[(int64_t)l * E + trace[tidx(m, T, k, p, l, t, r)]] += 1.0;
    }
  }
  if (T > 0) /* prompt transitions of dominant experts (:176-183) */
    for (int p = 0; p + 1 < P; ++p)
      for (int l = 0; l < m; ++l) {
        int a = oracle_dominant_expert(trace, P, m, T, k, p, l);
        int b = oracle_dominant_expert(trace, P, m, T, k, p + 1, l);
        prompt_counts[((int64_t)l * E + a) * E + b] += 1.0;
      }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* A7: smoothed / rank_scores / mean_rows / predict_* (predictor.cpp:13-220) */
/* ------------------------------------------------------------------------ */
static void smoothed(const double* counts, int e, double s, double* row) {
  double sum = 0.0; /* std::accumulate, left to right (:15) */
  for (int j = 0; j < e; ++j) sum += counts[j];
  double denom = sum + s * e;
  if (denom <= 0.0) {
    for (int j = 0; j < e; ++j) row[j] = 1.0 / e;
    return;
  }
  for (int j = 0; j < e; ++j) row[j] = (counts[j] + s) / denom;
}

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* stable order by descending score, ascending index on exact ties */
static void ranked_indices(const double* row, int e, int* order) {
  for (int i = 0; i < e; ++i) order[i] = i;
  for (int i = 1; i < e; ++i) { /* insertion sort == stable_sort with this comparator */
    int v = order[i];
    int j = i - 1;
    while (j >= 0) {
      int u = order[j];
      int before = (row[v] != row[u]) ? (row[v] > row[u]) : (v < u);
      if (!before) break;
      order[j + 1] = u;
      --j;
    }
    order[j + 1] = v;
  }
}

/* rank_scores (:30-58): relative tie band grouped by leader */
static int rank_scores(const double* scores, int e, int k, int32_t* experts) {
  int* order = (int*)malloc(sizeof(int) * (size_t)(e > 0 ? e : 1));
  ranked_indices(scores, e, order);
  int group_start = 0;
  double leader = e > 0 ? scores[order[0]] : 0.0;
  for (int i = 0; i <= e; ++i) {
    int close_group = (i == e) || (leader - scores[order[i]] > 1e-12 + 1e-3 * fabs(leader));
    if (close_group) {
      qsort(order + group_start, (size_t)(i - group_start), sizeof(int), cmp_int);
      if (i < e) {
        group_start = i;
        leader = scores[order[i]];
      }
    }
  }
  int n = k < e ? k : e;
  for (int r = 0; r < n; ++r) experts[r] = order[r];
  free(order);
  return n;
}

static int mean_rows(int E, double smoothing, const double* counts_base, const int32_t* from,
                     int n_from, double* scores) {
  if (n_from <= 0) return fail(VALIDATION, "predictor: empty expert set");
  double* row = (double*)malloc(sizeof(double) * (size_t)E);
  for (int j = 0; j < E; ++j) scores[j] = 0.0;
  for (int i = 0; i < n_from; ++i) {
    int e = from[i];
    if (e < 0 || e >= E) {
      free(row);
      return fail(VALIDATION, "predictor: expert index out of range");
    }
    smoothed(counts_base + (int64_t)e * E, E, smoothing, row);
    for (int j = 0; j < E; ++j) scores[j] += row[j];
  }
  for (int j = 0; j < E; ++j) scores[j] /= (double)n_from;
  free(row);
  return 0;
}

int oracle_predict(int m, int E, int k, double smoothing, const double* layer_counts,
                   const double* prompt_counts, int mode, const int32_t* prev_sets,
                   const int32_t* prev_sizes, int layer, double* scores, int32_t* experts,
                   int32_t* n_experts) {
  int rc;
  if (mode == 0) { /* predict_all_layers (:195-206) */
    for (int l = 0; l < m; ++l) {
      rc = mean_rows(E, smoothing, prompt_counts + (int64_t)l * E * E, prev_sets + l * k,
                     prev_sizes[l], scores + (int64_t)l * E);
      if (rc) return rc;
      n_experts[l] = rank_scores(scores + (int64_t)l * E, E, k, experts + l * k);
    }
    return 0;
  }
  if (mode == 1) { /* predict_chained (:208-220) */
    rc = mean_rows(E, smoothing, prompt_counts, prev_sets, prev_sizes[0], scores);
    if (rc) return rc;
    n_experts[0] = rank_scores(scores, E, k, experts);
    for (int l = 1; l < m; ++l) {
      rc = mean_rows(E, smoothing, layer_counts + (int64_t)(l - 1) * E * E, experts + (l - 1) * k,
                     n_experts[l - 1], scores + (int64_t)l * E);
      if (rc) return rc;
      n_experts[l] = rank_scores(scores + (int64_t)l * E, E, k, experts + l * k);
    }
    return 0;
  }
  /* predict_layerwise (:187-193) */
  if (layer < 1 || layer >= m) return fail(VALIDATION, "predictor.layer: must be in [1, num_layers)");
  rc = mean_rows(E, smoothing, layer_counts + (int64_t)(layer - 1) * E * E, prev_sets, prev_sizes[0],
                 scores);
  if (rc) return rc;
  n_experts[0] = rank_scores(scores, E, k, experts);
  return 0;
}

int oracle_predicted_frequencies(int m, int E, int n_tasks, const double* task_counts,
                                 double smoothing, int task, double* out) {
  /* (:222-238): seen task -> its tallies; unseen -> sum in std::map order */
  double* raw = (double*)calloc((size_t)m * E, sizeof(double));
  if (task >= 0 && task < n_tasks) {
    memcpy(raw, task_counts + (int64_t)task * m * E, sizeof(double) * (size_t)m * E);
  } else {
    for (int t = 0; t < n_tasks; ++t)
      for (int l = 0; l < m; ++l)
        for (int e = 0; e < E; ++e) raw[l * E + e] += task_counts[((int64_t)t * m + l) * E + e];
  }
  for (int l = 0; l < m; ++l) smoothed(raw + l * E, E, smoothing, out + l * E);
  free(raw);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* A7: Eq. 2 expected_tokens (expert_store.cpp:59-106)                       */
/* ------------------------------------------------------------------------ */
int oracle_expected_tokens(int m, int E, int n_tasks, const double* wo, const int32_t* sensitivity,
                           const uint8_t* has_sens, int n_requests, const int32_t* req_task,
                           const int32_t* req_tokens, const uint8_t* freq_present,
                           const double* freqs, int task_aware, double* aggregate) {
  double* tok = (double*)calloc((size_t)(n_tasks > 0 ? n_tasks : 1), sizeof(double));
  int* cnt = (int*)calloc((size_t)(n_tasks > 0 ? n_tasks : 1), sizeof(int));
  for (int i = 0; i < n_requests; ++i) { /* running then incoming (:80-81) */
    int t = req_task[i];
    if (t < 0 || t >= n_tasks) {
      free(tok);
      free(cnt);
      return fail(VALIDATION, "expected_tokens.request: unknown task_id");
    }
    tok[t] += (double)req_tokens[i];
    cnt[t] += 1;
  }
  for (int64_t i = 0; i < (int64_t)m * E; ++i) aggregate[i] = 0.0;
  for (int t = 0; t < n_tasks; ++t) { /* std::map key order == sorted task ids */
    if (cnt[t] == 0) continue;
    const double volume = tok[t] + cnt[t] * wo[t];
    for (int l = 0; l < m; ++l) {
      int sensitive = task_aware ? (!has_sens[t] || sensitivity[t * m + l] != 0) : 1;
      if (!sensitive) continue;
      for (int e = 0; e < E; ++e) {
        double f = 1.0 / E;
        if (freq_present[t]) f = freqs[((int64_t)t * m + l) * E + e];
        double grid = volume * f;
        aggregate[(int64_t)l * E + e] += grid;
      }
    }
  }
  free(tok);
  free(cnt);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* A7: select_experts / loading_targets (expert_store.cpp:111-157)           */
/* ------------------------------------------------------------------------ */
int oracle_select_experts(const double* aggregate, int m, int E, const int32_t* budgets, int32_t* out) {
  int* order = (int*)malloc(sizeof(int) * (size_t)E);
  for (int l = 0; l < m; ++l) {
    if (budgets[l] < 0 || budgets[l] > E) {
      free(order);
      return fail(VALIDATION, "select_experts.budgets: entries must be in [0, experts_per_layer]");
    }
    ranked_indices(aggregate + (int64_t)l * E, E, order);
    for (int i = 0; i < budgets[l]; ++i) out[l * E + i] = order[i];
  }
  free(order);
  return 0;
}

int oracle_loading_targets(const double* aggregate, int m, int E, const uint8_t* resident,
                           const int32_t* budgets, int32_t* out, int32_t* sizes) {
  int rc = oracle_select_experts(aggregate, m, E, budgets, out);
  if (rc) return rc;
  for (int l = 0; l < m; ++l) {
    sizes[l] = budgets[l];
    int all_zero = 1;
    for (int e = 0; e < E; ++e)
      if (aggregate[(int64_t)l * E + e] != 0.0) {
        all_zero = 0;
        break;
      }
    if (!all_zero) continue;
    int n = 0; /* masked layer keeps current residents, lowest indices first */
    for (int e = 0; e < E && n < budgets[l]; ++e)
      if (resident[l * E + e]) out[l * E + n++] = e;
    sizes[l] = n;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* A8: plan_loading (expert_store.cpp:159-195)                               */
/* ------------------------------------------------------------------------ */
int oracle_plan_loading(const uint8_t* resident, const int32_t* budgets, int m, int E,
                        const int32_t* target, const int32_t* target_sizes, const double* aggregate,
                        double per_expert_seconds, int32_t* evictions, int32_t* n_evict,
                        int32_t* loads, int32_t* n_load, double* duration, double* delta_e,
                        int32_t* total_loads) {
  uint8_t* wanted = (uint8_t*)malloc((size_t)E);
  int* order = (int*)malloc(sizeof(int) * (size_t)E);
  *delta_e = 0.0;
  *total_loads = 0;
  int rc = 0;
  for (int l = 0; l < m && !rc; ++l) {
    if (target_sizes[l] > budgets[l]) {
      rc = fail(VALIDATION, "plan_loading.target: exceeds layer budget");
      break;
    }
    memset(wanted, 0, (size_t)E);
    for (int i = 0; i < target_sizes[l]; ++i) {
      int e = target[l * E + i];
      if (e < 0 || e >= E) {
        rc = fail(VALIDATION, "plan_loading.target: expert index out of range");
        break;
      }
      if (wanted[e]) {
        rc = fail(VALIDATION, "plan_loading.target: duplicate expert index");
        break;
      }
      wanted[e] = 1;
    }
    if (rc) break;
    int ne = 0, nl = 0;
    for (int e = 0; e < E; ++e) /* evictions ascending (:172-173) */
      if (resident[l * E + e] && !wanted[e]) evictions[l * E + ne++] = e;
    ranked_indices(aggregate + (int64_t)l * E, E, order); /* loads by priority (:174-178) */
    for (int i = 0; i < E; ++i) {
      int e = order[i];
      if (wanted[e] && !resident[l * E + e]) loads[l * E + nl++] = e;
    }
    n_evict[l] = ne;
    n_load[l] = nl;
    duration[l] = (double)nl * per_expert_seconds;
    *delta_e += duration[l];
    *total_loads += nl;
  }
  free(wanted);
  free(order);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* engine invocation_aggregate (engine.cpp:367-417), predictor modes         */
/* ------------------------------------------------------------------------ */
int oracle_invocation_aggregate(int m, int E, int n_tasks, const double* pred_scores,
                                const double* fitted, const double* wo, const int32_t* sensitivity,
                                const uint8_t* has_sens, int n_requests, const int32_t* req_task,
                                const int32_t* req_tokens, int task_aware, double* aggregate) {
  double* freqs = (double*)malloc(sizeof(double) * (size_t)(n_tasks > 0 ? n_tasks : 1) * m * E);
  uint8_t* present = (uint8_t*)malloc((size_t)(n_tasks > 0 ? n_tasks : 1));
  for (int t = 0; t < n_tasks; ++t) {
    present[t] = 1;
    for (int l = 0; l < m; ++l) {
      double* rows = freqs + ((int64_t)t * m + l) * E;
      const double* fit = fitted + ((int64_t)t * m + l) * E;
      double sum = 0.0;
      for (int e = 0; e < E; ++e) {
        rows[e] = pred_scores[(int64_t)l * E + e] * fit[e];
        sum += rows[e];
      }
      if (sum <= 0.0) {
        for (int e = 0; e < E; ++e) rows[e] = 1.0 / E;
      } else {
        for (int e = 0; e < E; ++e) rows[e] /= sum;
      }
    }
  }
  int rc = oracle_expected_tokens(m, E, n_tasks, wo, sensitivity, has_sens, n_requests, req_task,
                                  req_tokens, present, freqs, task_aware, aggregate);
  free(freqs);
  free(present);
  return rc;
}
