// K2: popularity histograms over routing history (A6) and the predictor /
// Eq. 2 / resident-set selection / load planning (A7, A8) on the GPU.
//
// A6 is the data-parallel part: one block per (prompt, layer) builds the
// rank-0 and all-rank expert histograms and the layer-transition histogram of
// that slice in shared memory and folds them into exact 64-bit global tallies
// (the reference stores the same integers as doubles, predictor.cpp:164-183;
// counts commute, so block order does not matter).  Dominant experts per
// (prompt, layer) are reduced on the fly, and the last block to finish
// tallies the prompt transitions, continuing the chain across calls (one
// launch per update).
//
// A7/A8 are latency-bound fp64 control logic over m x E numbers.  They run as
// single-block kernels whose every floating-point expression and summation
// order matches the reference line for line; this file is compiled with
// --fmad=false so no multiply-add is contracted (the reference's ISO C++
// build has -ffp-contract=off).  Ranking uses a parallel stable rank
// (position = number of elements that precede it under "score desc, index
// asc"), which is exactly std::stable_sort's order for a strict total order.
#include <algorithm>
#include <vector>

#include <cstring>

#include "capi_util.h"
#include "kernels.h"

namespace emoe {
namespace {

using u64 = unsigned long long;

// ---------------------------------------------------------------------------
// A6 histograms
// ---------------------------------------------------------------------------
// The last block to finish (a device counter in last[m], reset by that
// block) also tallies the prompt n -> n+1 transitions of the dominant
// experts (predictor.cpp:176-183), continuing the chain from the previous
// call through last[] when has_last, and saves the last prompt's dominant
// experts for the next call: one launch per update.
__global__ void hist_kernel(const int32_t* __restrict__ trace, int P, int m, int T, int k, int E,
                            const int32_t* __restrict__ task_ids, u64* __restrict__ layer_counts,
                            u64* __restrict__ task_counts, int32_t* __restrict__ dom, int32_t* __restrict__ last,
                            int has_last, u64* __restrict__ prompt_counts) {
  extern __shared__ int sh[];
  int* h0 = sh;          // [E] rank-0 counts
  int* hall = sh + E;    // [E] all-rank counts
  int* htr = sh + 2 * E;  // [E*E] layer transitions l -> l+1
  const int p = blockIdx.x / m, l = blockIdx.x % m;
  const bool do_trans = l + 1 < m;
  const int nbins = 2 * E + (do_trans ? E * E : 0);
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int32_t* base = trace + ((int64_t)p * m + l) * T * k;
  const int32_t* next = trace + ((int64_t)p * m + l + 1) * T * k;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int a = base[(int64_t)t * k];
    atomicAdd(&h0[a], 1);
    if (task_ids)
      for (int r = 0; r < k; ++r) atomicAdd(&hall[base[(int64_t)t * k + r]], 1);
    if (do_trans) atomicAdd(&htr[a * E + next[(int64_t)t * k]], 1);
  }
  __syncthreads();
  if (task_ids) {
    u64* dst = task_counts + ((int64_t)task_ids[p] * m + l) * E;
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      if (hall[e]) atomicAdd(&dst[e], (u64)hall[e]);
  }
  if (do_trans) {
    u64* dst = layer_counts + (int64_t)l * E * E;
    for (int i = threadIdx.x; i < E * E; i += blockDim.x)
      if (htr[i]) atomicAdd(&dst[i], (u64)htr[i]);
  }
  if (threadIdx.x < 32) {  // dominant_expert: modal rank-0, smallest index on ties (workload.cpp:350-361)
    int bc = -1, be = 0;     // this lane's best over e = lane, lane + 32, ... (ascending: first max kept)
    for (int e = threadIdx.x; e < E; e += 32)
      if (h0[e] > bc) {
        bc = h0[e];
        be = e;
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {  // (count desc, index asc) is a total order: the reduction is exact
      const int oc = __shfl_down_sync(0xffffffffu, bc, off), oe = __shfl_down_sync(0xffffffffu, be, off);
      if (oc > bc || (oc == bc && oe < be)) {
        bc = oc;
        be = oe;
      }
    }
    if (threadIdx.x == 0) dom[(int64_t)p * m + l] = be;
  }
  __shared__ int is_last;
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(&last[m], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int total = (P - 1 + (has_last ? 1 : 0)) * m;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int ll = i % m;
    const int pi = i / m - (has_last ? 1 : 0);  // -1 = chain from the previous call
    const int a = pi < 0 ? last[ll] : __ldcg(dom + (int64_t)pi * m + ll);
    const int b = __ldcg(dom + (int64_t)(pi + 1) * m + ll);
    atomicAdd(&prompt_counts[((int64_t)ll * E + a) * E + b], 1ull);
  }
  __syncthreads();  // every read of last[] above precedes the overwrite
  for (int ll = threadIdx.x; ll < m; ll += blockDim.x) last[ll] = __ldcg(dom + (int64_t)(P - 1) * m + ll);
  if (threadIdx.x == 0) last[m] = 0;
}

// prompt_expert_sets (workload.cpp:363-377): one block per layer
__global__ void prompt_sets_kernel(const int32_t* __restrict__ trace, int m, int T, int k, int E, int prompt,
                                   int32_t* __restrict__ dom, int32_t* __restrict__ sets, int32_t* __restrict__ sizes) {
  extern __shared__ int cnt[];
  const int l = blockIdx.x;
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int32_t* base = trace + ((int64_t)prompt * m + l) * T * k;
  for (int t = threadIdx.x; t < T; t += blockDim.x) atomicAdd(&cnt[base[(int64_t)t * k]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int best = 0;
    for (int e = 1; e < E; ++e)
      if (cnt[e] > cnt[best]) best = e;
    dom[l] = best;
    int n = 0;
    for (int r = 0; r < k; ++r) {  // by count desc, index asc, only experts that occur
      int b = -1;
      for (int e = 0; e < E; ++e) {
        if (cnt[e] <= 0) continue;
        bool used = false;
        for (int q = 0; q < n; ++q) used |= sets[l * k + q] == e;
        if (used) continue;
        if (b < 0 || cnt[e] > cnt[b]) b = e;
      }
      if (b < 0) break;
      sets[l * k + n++] = b;
    }
    for (int r = n; r < k; ++r) sets[l * k + r] = -1;
    sizes[l] = n;
  }
}

// ---------------------------------------------------------------------------
// A7 / A8 device helpers (single block, blockDim >= 32)
// ---------------------------------------------------------------------------
constexpr int MAXE = 1024;

// smoothed(counts)[j] for a u64 count row (predictor.cpp:13-24).  The sum is
// computed left to right by every calling thread (identical value).
__device__ double smoothed_at(const u64* row, int E, double s, int j) {
  double sum = 0.0;
  for (int q = 0; q < E; ++q) sum += (double)row[q];
  const double denom = sum + s * E;
  if (denom <= 0.0) return 1.0 / E;
  return ((double)row[j] + s) / denom;
}
__device__ double smoothed_at_d(const double* row, int E, double s, int j) {
  double sum = 0.0;
  for (int q = 0; q < E; ++q) sum += row[q];
  const double denom = sum + s * E;
  if (denom <= 0.0) return 1.0 / E;
  return (row[j] + s) / denom;
}

// stable rank under (score desc, index asc): order[pos] = i
__device__ void ranked_indices_block(const double* row, int E, int* order) {
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const double si = row[i];
    int pos = 0;
    for (int j = 0; j < E; ++j) {
      const double sj = row[j];
      pos += (sj != si) ? (sj > si) : (j < i);
    }
    order[pos] = i;
  }
  __syncthreads();
}

// rank_scores (predictor.cpp:30-58) on a shared scores row; writes experts[0..min(k,E))
__device__ int rank_scores_block(const double* scores, int E, int k, int* order, int32_t* experts) {
  ranked_indices_block(scores, E, order);
  __shared__ int n_out;
  if (threadIdx.x == 0) {
    int group_start = 0;
    double leader = E > 0 ? scores[order[0]] : 0.0;
    for (int i = 0; i <= E; ++i) {
      const bool close = i == E || leader - scores[order[i]] > 1e-12 + 1e-3 * fabs(leader);
      if (close) {
        for (int a = group_start + 1; a < i; ++a) {  // sort the group by index
          const int v = order[a];
          int b = a - 1;
          while (b >= group_start && order[b] > v) {
            order[b + 1] = order[b];
            --b;
          }
          order[b + 1] = v;
        }
        if (i < E) {
          group_start = i;
          leader = scores[order[i]];
        }
      }
    }
    const int n = k < E ? k : E;
    for (int r = 0; r < n; ++r) experts[r] = order[r];
    n_out = n;
  }
  __syncthreads();
  return n_out;
}

// mean_rows (predictor.cpp:60-72) of u64 count rows `base[e]` over `from`
__device__ void mean_rows_block(const u64* base, int E, double s, const int32_t* from, int n_from, double* scores) {
  for (int j = threadIdx.x; j < E; j += blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < n_from; ++i) acc += smoothed_at(base + (int64_t)from[i] * E, E, s, j);
    scores[j] = acc / (double)n_from;
  }
  __syncthreads();
}

struct PredictArgs {
  int mode, layer, m, E, k;
  double s;
  const u64* layer_counts;
  const u64* prompt_counts;
  const int32_t* prev_sets;
  const int32_t* prev_sizes;
  double* scores;   // [m][E]
  int32_t* experts;  // [m][k]
  int32_t* n_experts;  // [m]
};

// l0/l1: the layers of predict_all_layers this block handles (layers are
// independent in that mode; chained / layerwise ignore the range)
__device__ void predict_block(const PredictArgs& a, int* order, double* row, int l0 = 0, int l1 = -1) {
  const int E = a.E, k = a.k;
  if (l1 < 0) l1 = a.m;
  if (a.mode == 0) {  // predict_all_layers
    for (int l = l0; l < l1; ++l) {
      mean_rows_block(a.prompt_counts + (int64_t)l * E * E, E, a.s, a.prev_sets + l * k, a.prev_sizes[l], row);
      for (int j = threadIdx.x; j < E; j += blockDim.x) a.scores[(int64_t)l * E + j] = row[j];
      const int n = rank_scores_block(row, E, k, order, a.experts + l * k);
      if (threadIdx.x == 0) a.n_experts[l] = n;
      __syncthreads();
    }
  } else if (a.mode == 1) {  // predict_chained
    mean_rows_block(a.prompt_counts, E, a.s, a.prev_sets, a.prev_sizes[0], row);
    for (int j = threadIdx.x; j < E; j += blockDim.x) a.scores[j] = row[j];
    int n = rank_scores_block(row, E, k, order, a.experts);
    if (threadIdx.x == 0) a.n_experts[0] = n;
    __syncthreads();
    for (int l = 1; l < a.m; ++l) {
      mean_rows_block(a.layer_counts + (int64_t)(l - 1) * E * E, E, a.s, a.experts + (l - 1) * k, n, row);
      for (int j = threadIdx.x; j < E; j += blockDim.x) a.scores[(int64_t)l * E + j] = row[j];
      n = rank_scores_block(row, E, k, order, a.experts + l * k);
      if (threadIdx.x == 0) a.n_experts[l] = n;
      __syncthreads();
    }
  } else {  // predict_layerwise
    mean_rows_block(a.layer_counts + (int64_t)(a.layer - 1) * E * E, E, a.s, a.prev_sets, a.prev_sizes[0], row);
    for (int j = threadIdx.x; j < E; j += blockDim.x) a.scores[j] = row[j];
    const int n = rank_scores_block(row, E, k, order, a.experts);
    if (threadIdx.x == 0) a.n_experts[0] = n;
  }
}

__global__ void predict_kernel(PredictArgs a) {
  __shared__ int order[MAXE];
  __shared__ double row[MAXE];
  predict_block(a, order, row);
}

// predicted_frequencies (predictor.cpp:222-238)
__device__ void freq_block(const u64* task_counts, int n_tasks, int m, int E, double s, int task, double* out,
                           double* raw, int l0 = 0, int l1 = -1) {
  if (l1 < 0) l1 = m;
  for (int l = l0; l < l1; ++l) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      double v = 0.0;
      if (task >= 0 && task < n_tasks) {
        v = (double)task_counts[((int64_t)task * m + l) * E + e];
      } else {
        for (int t = 0; t < n_tasks; ++t) v += (double)task_counts[((int64_t)t * m + l) * E + e];
      }
      raw[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) out[(int64_t)l * E + e] = smoothed_at_d(raw, E, s, e);
    __syncthreads();
  }
}

__global__ void freq_kernel(const u64* task_counts, int n_tasks, int m, int E, double s, int task, double* out) {
  __shared__ double raw[MAXE];
  freq_block(task_counts, n_tasks, m, E, s, task, out, raw);
}

struct Eq2Args {
  int m, E, n_tasks;
  const double* wo;
  const int32_t* sens;
  const uint8_t* has_sens;
  int n_req;
  const int32_t* req_task;
  const int32_t* req_tokens;
  const uint8_t* freq_present;
  const double* freqs;  // [n_tasks][m][E]
  int task_aware;
  double* aggregate;  // [m][E]
};

// expected_tokens (expert_store.cpp:59-106): thread per (l, e), tasks in sorted order
__device__ void eq2_block(const Eq2Args& a, double* tok, int* cnt, int l0 = 0, int l1 = -1) {
  if (l1 < 0) l1 = a.m;
  for (int t = threadIdx.x; t < a.n_tasks; t += blockDim.x) {
    double s = 0.0;
    int c = 0;
    for (int i = 0; i < a.n_req; ++i)
      if (a.req_task[i] == t) {
        s += (double)a.req_tokens[i];
        ++c;
      }
    tok[t] = s;
    cnt[t] = c;
  }
  __syncthreads();
  const int ME = (l1 - l0) * a.E;
  for (int i = threadIdx.x; i < ME; i += blockDim.x) {
    const int l = l0 + i / a.E, e = i % a.E;
    double agg = 0.0;
    for (int t = 0; t < a.n_tasks; ++t) {
      if (cnt[t] == 0) continue;
      const double volume = tok[t] + cnt[t] * a.wo[t];
      const bool sensitive = a.task_aware ? (!a.has_sens[t] || a.sens[t * a.m + l] != 0) : true;
      if (!sensitive) continue;
      double f = 1.0 / a.E;
      if (a.freq_present[t]) f = a.freqs[((int64_t)t * a.m + l) * a.E + e];
      const double grid = volume * f;
      agg += grid;
    }
    a.aggregate[(int64_t)l * a.E + e] = agg;
  }
  __syncthreads();
}

constexpr int MAX_TASKS = 256;

__global__ void eq2_kernel(Eq2Args a) {
  __shared__ double tok[MAX_TASKS];
  __shared__ int cnt[MAX_TASKS];
  eq2_block(a, tok, cnt);
}

struct PlanArgs {
  int m, E;
  const double* aggregate;
  const uint8_t* resident;  // [m][E]
  const int32_t* budgets;
  double per_expert;
  int32_t* targets;  // [m][E]
  int32_t* target_sizes;
  int32_t* evictions;
  int32_t* n_evict;
  int32_t* loads;
  int32_t* n_load;
  double* duration;
  double* delta_e;
  int32_t* total_loads;
  int targets_given;  // 1: use targets as input (plan_loading only)
  int select_only;    // 1: select_experts only (no zero-row keep, no plan)
};

// select_experts + loading_targets + plan_loading (expert_store.cpp:111-195)
// l0/l1: layer range; accumulate = 0 leaves delta_e / total_loads to
// plan_finalize_kernel (several blocks, one layer each)
__device__ void plan_block(const PlanArgs& a, int* order, int l0 = 0, int l1 = -1, bool accumulate = true) {
  const int E = a.E;
  __shared__ int wanted[MAXE];
  if (l1 < 0) l1 = a.m;
  for (int l = l0; l < l1; ++l) {
    const double* row = a.aggregate + (int64_t)l * E;
    ranked_indices_block(row, E, order);
    if (!a.targets_given && threadIdx.x == 0) {
      int n = a.budgets[l];
      for (int i = 0; i < n; ++i) a.targets[l * E + i] = order[i];
      if (!a.select_only) {
        bool all_zero = true;
        for (int e = 0; e < E; ++e)
          if (row[e] != 0.0) {
            all_zero = false;
            break;
          }
        if (all_zero) {  // masked layer keeps current residents, lowest indices first
          n = 0;
          for (int e = 0; e < E && n < a.budgets[l]; ++e)
            if (a.resident[l * E + e]) a.targets[l * E + n++] = e;
        }
      }
      a.target_sizes[l] = n;
    }
    __syncthreads();
    if (a.select_only) continue;
    for (int e = threadIdx.x; e < E; e += blockDim.x) wanted[e] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < a.target_sizes[l]; ++i) wanted[a.targets[l * E + i]] = 1;
      int ne = 0, nl = 0;
      for (int e = 0; e < E; ++e)
        if (a.resident[l * E + e] && !wanted[e]) a.evictions[l * E + ne++] = e;
      for (int i = 0; i < E; ++i) {
        const int e = order[i];
        if (wanted[e] && !a.resident[l * E + e]) a.loads[l * E + nl++] = e;
      }
      a.n_evict[l] = ne;
      a.n_load[l] = nl;
      a.duration[l] = (double)nl * a.per_expert;
      if (accumulate) {
        if (l == 0) {
          *a.delta_e = 0.0;
          *a.total_loads = 0;
        }
        *a.delta_e += a.duration[l];
        *a.total_loads += nl;
      }
    }
    __syncthreads();
  }
}

__global__ void plan_kernel(PlanArgs a) {
  __shared__ int order[MAXE];
  plan_block(a, order);
}

// engine invocation (engine.cpp:367-446): predict -> per-task modulation ->
// Eq. 2 -> loading_targets -> plan_loading, all in one block
struct InvocationArgs {
  PredictArgs pred;
  const u64* task_counts;  // fitted frequencies come from these
  int n_tasks;
  double* fitted;  // scratch [n_tasks][m][E]
  double* freqs;   // scratch [n_tasks][m][E]
  Eq2Args eq2;
  PlanArgs plan;
};

// predict_all_layers (mode 0): one block per layer -- every step below is
// per layer -- and plan_finalize_kernel sums delta_e in layer order (the
// reference's sequential sum, bit for bit); predict_chained (mode 1): one
// block over all layers (layer l's prediction feeds layer l + 1).
__global__ void invocation_kernel(InvocationArgs a) {
  __shared__ int order[MAXE];
  __shared__ double row[MAXE];
  __shared__ double tok[MAX_TASKS];
  __shared__ int cnt[MAX_TASKS];
  const int m = a.pred.m, E = a.pred.E;
  const bool per_layer = gridDim.x > 1;
  const int l0 = per_layer ? (int)blockIdx.x : 0, l1 = per_layer ? l0 + 1 : m;
  predict_block(a.pred, order, row, l0, l1);
  __syncthreads();
  for (int t = 0; t < a.n_tasks; ++t)  // fitted_freq_ per profile (engine.cpp:256-257)
    freq_block(a.task_counts, a.n_tasks, m, E, a.pred.s, t, a.fitted + (int64_t)t * m * E, row, l0, l1);
  // rows[l][e] = score * fitted, normalised (engine.cpp:394-411)
  for (int i = threadIdx.x; i < a.n_tasks * (l1 - l0); i += blockDim.x) {
    const int t = i / (l1 - l0), l = l0 + i % (l1 - l0);
    const double* sc = a.pred.scores + (int64_t)l * E;
    const double* fit = a.fitted + ((int64_t)t * m + l) * E;
    double* rows = a.freqs + ((int64_t)t * m + l) * E;
    double sum = 0.0;
    for (int e = 0; e < E; ++e) {
      rows[e] = sc[e] * fit[e];
      sum += rows[e];
    }
    if (sum <= 0.0) {
      for (int e = 0; e < E; ++e) rows[e] = 1.0 / E;
    } else {
      for (int e = 0; e < E; ++e) rows[e] /= sum;
    }
  }
  __syncthreads();
  eq2_block(a.eq2, tok, cnt, l0, l1);
  plan_block(a.plan, order, l0, l1, !per_layer);
}

__global__ void plan_finalize_kernel(PlanArgs a) {
  if (threadIdx.x != 0) return;
  double de = 0.0;
  int nl = 0;
  for (int l = 0; l < a.m; ++l) {
    de += a.duration[l];
    nl += a.n_load[l];
  }
  *a.delta_e = de;
  *a.total_loads = nl;
}

}  // namespace
}  // namespace emoe

using namespace emoe;

struct emoe_predictor {
  int m = 0, E = 0, k = 0, n_tasks = 0;
  double smoothing = 0.01;
  u64* layer_counts = nullptr;
  u64* prompt_counts = nullptr;
  u64* task_counts = nullptr;
  int32_t* last_dom = nullptr;
  bool has_last = false;
  int32_t* dom = nullptr;
  size_t dom_cap = 0;

  // Invocation path (emoe_invocation_host, called every p prompts while the
  // layers compute): its own stream, ordered after the last histogram update
  // by an event, and one persistent device arena + pinned host staging block
  // (inputs packed and uploaded with one copy, outputs downloaded with one), so
  // an invocation allocates nothing and never synchronises the whole device.
  cudaStream_t inv_stream = nullptr;
  cudaEvent_t hist_done = nullptr;
  bool hist_recorded = false;
  uint8_t* arena_dev = nullptr;
  uint8_t* arena_host = nullptr;
  size_t arena_cap = 0;
  void arena_reserve(size_t bytes) {
    if (bytes <= arena_cap) return;
    if (arena_dev) {
      EMOE_CUDA(cudaStreamSynchronize(inv_stream));
      EMOE_CUDA(cudaFree(arena_dev));
      EMOE_CUDA(cudaFreeHost(arena_host));
      arena_dev = arena_host = nullptr;
    }
    const size_t cap = std::max<size_t>(bytes, 2 * arena_cap);
    EMOE_CUDA(cudaMalloc(&arena_dev, cap));
    EMOE_CUDA(cudaHostAlloc(&arena_host, cap, cudaHostAllocDefault));
    arena_cap = cap;
  }

  size_t n_layer() const { return (size_t)(m > 1 ? m - 1 : 0) * E * E; }
  size_t n_prompt() const { return (size_t)m * E * E; }
  size_t n_task() const { return (size_t)n_tasks * m * E; }
  void zero() {
    if (n_layer()) EMOE_CUDA(cudaMemset(layer_counts, 0, n_layer() * sizeof(u64)));
    EMOE_CUDA(cudaMemset(prompt_counts, 0, n_prompt() * sizeof(u64)));
    if (n_task()) EMOE_CUDA(cudaMemset(task_counts, 0, n_task() * sizeof(u64)));
    EMOE_CUDA(cudaDeviceSynchronize());  // visible to the invocation stream (not ordered with the legacy stream)
    has_last = false;
  }
};

namespace {

void check_sets(const int32_t* sets, const int32_t* sizes, int rows, int k, int E, const char* field) {
  for (int l = 0; l < rows; ++l) {
    if (sizes[l] <= 0) throw ValidationError(std::string(field) + ": empty expert set");
    EMOE_REQUIRE(sizes[l] <= k, std::string(field) + ": set larger than top_k");
    for (int i = 0; i < sizes[l]; ++i)
      if (sets[l * k + i] < 0 || sets[l * k + i] >= E)
        throw ValidationError(std::string(field) + ": expert index out of range");
  }
}

PredictArgs make_predict_args(emoe_predictor* P, int mode, int layer, const int32_t* d_sets, const int32_t* d_sizes,
                              double* d_scores, int32_t* d_experts, int32_t* d_n) {
  PredictArgs a;
  a.mode = mode;
  a.layer = layer;
  a.m = P->m;
  a.E = P->E;
  a.k = P->k;
  a.s = P->smoothing;
  a.layer_counts = P->layer_counts;
  a.prompt_counts = P->prompt_counts;
  a.prev_sets = d_sets;
  a.prev_sizes = d_sizes;
  a.scores = d_scores;
  a.experts = d_experts;
  a.n_experts = d_n;
  return a;
}

void validate_predict(emoe_predictor* P, int mode, int layer, const int32_t* sets, const int32_t* sizes) {
  EMOE_REQUIRE(mode >= 0 && mode <= 2, "predict: unknown mode");
  if (mode == 2) EMOE_REQUIRE(layer >= 1 && layer < P->m, "predictor.layer: must be in [1, num_layers)");
  check_sets(sets, sizes, mode == 0 ? P->m : 1, P->k, P->E, mode == 0 ? "predictor.prev_prompt" : "predictor.prev_experts");
}

void validate_eq2(int m, int E, int n_tasks, int n_req, const int32_t* req_task) {
  EMOE_REQUIRE(m >= 1 && E >= 1 && E <= MAXE, "expected_tokens: invalid shape");
  EMOE_REQUIRE(n_tasks <= MAX_TASKS, "expected_tokens: too many tasks");
  for (int i = 0; i < n_req; ++i)
    if (req_task[i] < 0 || req_task[i] >= n_tasks) throw ValidationError("expected_tokens.request: unknown task_id");
}

void validate_budgets(int m, int E, const int32_t* budgets) {
  for (int l = 0; l < m; ++l)
    EMOE_REQUIRE(budgets[l] >= 0 && budgets[l] <= E,
                 "select_experts.budgets: entries must be in [0, experts_per_layer]");
}

}  // namespace

extern "C" {

int emoe_predictor_create(int m, int E, int k, int n_tasks, double smoothing, emoe_predictor** out) {
  return guard([&] {
    EMOE_REQUIRE(out, "predictor_create: null out");
    EMOE_REQUIRE(m >= 1, "predictor.num_layers: must be >= 1");
    EMOE_REQUIRE(E >= 1 && E <= MAXE, "predictor.num_experts: must be in [1, 1024]");
    EMOE_REQUIRE(k >= 1 && k <= E, "predictor.top_k: must be in [1, num_experts]");
    EMOE_REQUIRE(smoothing >= 0.0, "predictor.smoothing: must be >= 0");
    EMOE_REQUIRE(n_tasks >= 0 && n_tasks <= MAX_TASKS, "predictor.num_tasks: out of range");
    auto* P = new emoe_predictor();
    P->m = m;
    P->E = E;
    P->k = k;
    P->n_tasks = n_tasks;
    P->smoothing = smoothing;
    EMOE_CUDA(cudaMalloc(&P->layer_counts, std::max<size_t>(1, P->n_layer()) * sizeof(u64)));
    EMOE_CUDA(cudaMalloc(&P->prompt_counts, P->n_prompt() * sizeof(u64)));
    EMOE_CUDA(cudaMalloc(&P->task_counts, std::max<size_t>(1, P->n_task()) * sizeof(u64)));
    EMOE_CUDA(cudaMalloc(&P->last_dom, (m + 1) * sizeof(int32_t)));  // [m] = hist_kernel's last-block counter
    EMOE_CUDA(cudaMemset(P->last_dom, 0, (m + 1) * sizeof(int32_t)));
    EMOE_CUDA(cudaStreamCreateWithFlags(&P->inv_stream, cudaStreamNonBlocking));
    EMOE_CUDA(cudaEventCreateWithFlags(&P->hist_done, cudaEventDisableTiming));
    P->zero();
    *out = P;
  });
}

int emoe_predictor_destroy(emoe_predictor* P) {
  return guard([&] {
    if (!P) return;
    cudaDeviceSynchronize();
    for (void* p : {(void*)P->layer_counts, (void*)P->prompt_counts, (void*)P->task_counts, (void*)P->last_dom,
                    (void*)P->dom, (void*)P->arena_dev})
      if (p) cudaFree(p);
    if (P->arena_host) cudaFreeHost(P->arena_host);
    if (P->inv_stream) cudaStreamDestroy(P->inv_stream);
    if (P->hist_done) cudaEventDestroy(P->hist_done);
    delete P;
  });
}

int emoe_predictor_reset(emoe_predictor* P) {
  return guard([&] {
    EMOE_REQUIRE(P, "predictor_reset: null");
    P->zero();
  });
}

int emoe_predictor_break_chain(emoe_predictor* P) {
  return guard([&] {
    EMOE_REQUIRE(P, "predictor_break_chain: null");
    P->has_last = false;
  });
}

int emoe_hist_update(emoe_predictor* P, const int32_t* trace, int nP, int T, const int32_t* task_ids, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(P && trace, "hist_update: null argument");
    if (nP == 0) return;
    EMOE_REQUIRE(T >= 1, "hist_update: tokens_per_prompt must be >= 1");
    EMOE_REQUIRE(!task_ids || P->n_tasks > 0, "hist_update: task ids given but the predictor has no tasks");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t need = (size_t)nP * P->m;
    if (need > P->dom_cap) {
      if (P->dom) EMOE_CUDA(cudaFree(P->dom));
      EMOE_CUDA(cudaMalloc(&P->dom, need * sizeof(int32_t)));
      P->dom_cap = need;
    }
    const int E = P->E;
    const size_t smem = (size_t)(2 * E + (P->m > 1 ? E * E : 0)) * sizeof(int);
    EMOE_REQUIRE(smem <= 200 * 1024, "hist_update: E too large for the shared-memory histogram");
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(hist_kernel), (int)smem);
    hist_kernel<<<nP * P->m, 512, smem, s>>>(trace, nP, P->m, T, P->k, E, task_ids, P->layer_counts, P->task_counts,
                                             P->dom, P->last_dom, P->has_last ? 1 : 0, P->prompt_counts);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    EMOE_CUDA(cudaEventRecord(P->hist_done, s));  // the next invocation reads the counts after this
    P->hist_recorded = true;
    P->has_last = true;
  });
}

int emoe_hist_update_host(emoe_predictor* P, const int32_t* trace, int nP, int T, const int32_t* task_ids) {
  return guard([&] {
    EMOE_REQUIRE(P && (trace || nP == 0), "hist_update_host: null argument");
    if (nP == 0) return;
    EMOE_REQUIRE(T >= 1, "hist_update: tokens_per_prompt must be >= 1");
    const size_t n = (size_t)nP * P->m * T * P->k;
    for (size_t i = 0; i < n; ++i)
      EMOE_REQUIRE(trace[i] >= 0 && trace[i] < P->E, "predictor.trace: expert index out of range");
    if (task_ids)
      for (int p = 0; p < nP; ++p)
        EMOE_REQUIRE(task_ids[p] >= 0 && task_ids[p] < P->n_tasks, "predictor.task_ids: index out of range");
    DevBuf<int32_t> dt(trace, n);
    DevBuf<int32_t> di(task_ids ? (size_t)nP : 0);
    if (task_ids) EMOE_CUDA(cudaMemcpy(di.p, task_ids, nP * sizeof(int32_t), cudaMemcpyHostToDevice));
    const int rc = emoe_hist_update(P, dt.p, nP, T, task_ids ? di.p : nullptr, nullptr);
    if (rc != EMOE_OK) throw CudaError(last_error_slot());
    EMOE_CUDA(cudaDeviceSynchronize());
  });
}

int emoe_predictor_counts_host(emoe_predictor* P, double* lc, double* pc, double* tc) {
  return guard([&] {
    EMOE_REQUIRE(P, "predictor_counts: null");
    EMOE_CUDA(cudaDeviceSynchronize());
    auto dump = [](const u64* d, size_t n, double* out) {
      if (!n || !out) return;
      std::vector<u64> h(n);
      EMOE_CUDA(cudaMemcpy(h.data(), d, n * sizeof(u64), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i) out[i] = (double)h[i];
    };
    dump(P->layer_counts, P->n_layer(), lc);
    dump(P->prompt_counts, P->n_prompt(), pc);
    dump(P->task_counts, P->n_task(), tc);
  });
}

int emoe_predictor_set_counts_host(emoe_predictor* P, const double* lc, const double* pc, const double* tc) {
  return guard([&] {
    EMOE_REQUIRE(P, "predictor_set_counts: null");
    auto load = [](u64* d, size_t n, const double* in) {
      if (!n || !in) return;
      std::vector<u64> h(n);
      for (size_t i = 0; i < n; ++i) {
        EMOE_REQUIRE(in[i] >= 0.0 && in[i] == (double)(u64)in[i], "predictor counts must be non-negative integers");
        h[i] = (u64)in[i];
      }
      EMOE_CUDA(cudaMemcpy(d, h.data(), n * sizeof(u64), cudaMemcpyHostToDevice));
    };
    load(P->layer_counts, P->n_layer(), lc);
    load(P->prompt_counts, P->n_prompt(), pc);
    load(P->task_counts, P->n_task(), tc);
    EMOE_CUDA(cudaDeviceSynchronize());  // copies complete before the invocation stream reads them
  });
}

int emoe_predictor_count_size(emoe_predictor* P, int64_t* n) {
  return guard([&] {
    EMOE_REQUIRE(P && n, "predictor_count_size: null");
    *n = (int64_t)(P->n_layer() + P->n_prompt() + P->n_task());
  });
}

// Stream-ordered device copies of the tallies as one int64 vector
// [layer | prompt | task]: the all-reduce of per-rank histogram deltas
// runs on these without a host round trip.
int emoe_predictor_counts_dev(emoe_predictor* P, int64_t* dst, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(P && dst, "predictor_counts_dev: null");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (P->hist_recorded) EMOE_CUDA(cudaStreamWaitEvent(s, P->hist_done, 0));
    size_t off = 0;
    for (auto [d, n] : {std::pair<const u64*, size_t>{P->layer_counts, P->n_layer()},
                        {P->prompt_counts, P->n_prompt()}, {P->task_counts, P->n_task()}}) {
      if (n) EMOE_CUDA(cudaMemcpyAsync(dst + off, d, n * sizeof(u64), cudaMemcpyDeviceToDevice, s));
      off += n;
    }
  });
}

int emoe_predictor_set_counts_dev(emoe_predictor* P, const int64_t* src, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(P && src, "predictor_set_counts_dev: null");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (P->hist_recorded) EMOE_CUDA(cudaStreamWaitEvent(s, P->hist_done, 0));
    size_t off = 0;
    for (auto [d, n] : {std::pair<u64*, size_t>{P->layer_counts, P->n_layer()}, {P->prompt_counts, P->n_prompt()},
                        {P->task_counts, P->n_task()}}) {
      if (n) EMOE_CUDA(cudaMemcpyAsync(d, src + off, n * sizeof(u64), cudaMemcpyDeviceToDevice, s));
      off += n;
    }
    EMOE_CUDA(cudaEventRecord(P->hist_done, s));  // invocations read the merged counts after this
    P->hist_recorded = true;
  });
}

int emoe_prompt_expert_sets(const int32_t* trace, int nP, int m, int T, int k, int prompt, int32_t* dominant,
                            int32_t* sets, int32_t* sizes, void* stream) {
  return guard([&] {
    EMOE_REQUIRE(trace && prompt >= 0 && prompt < nP && m >= 1 && T >= 1 && k >= 1, "prompt_expert_sets: bad args");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // E is bounded by the largest index seen; scan on the device is cheap but the
    // caller's trace is device memory, so bound E by the predictor maximum.
    const int E = MAXE;
    DevBuf<int32_t> dd(m), ds((size_t)m * k), dz(m);
    prompt_sets_kernel<<<m, 256, E * sizeof(int), s>>>(trace, m, T, k, E, prompt, dd.p, ds.p, dz.p);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    EMOE_CUDA(cudaStreamSynchronize(s));
    dd.to_host(dominant);
    ds.to_host(sets);
    dz.to_host(sizes);
  });
}

int emoe_prompt_expert_sets_host(const int32_t* trace_prompt, int m, int T, int k, int32_t* dominant, int32_t* sets,
                                 int32_t* sizes) {
  return guard([&] {
    EMOE_REQUIRE(m >= 1 && T >= 0 && k >= 1 && dominant && sets && sizes, "prompt_expert_sets: bad args");
    EMOE_REQUIRE(T == 0 || trace_prompt, "prompt_expert_sets: null trace");
    if (T == 0) {  // no tokens: the reference's empty count vector gives expert 0 and empty sets
      for (int l = 0; l < m; ++l) {
        dominant[l] = 0;
        sizes[l] = 0;
        for (int r = 0; r < k; ++r) sets[(size_t)l * k + r] = -1;
      }
      return;
    }
    // the count vector spans the largest rank-0 index seen (workload.cpp:351-356)
    int E = 1;
    for (size_t i = 0; i < (size_t)m * T; ++i) {
      const int32_t e = trace_prompt[i * k];
      EMOE_REQUIRE(e >= 0 && e < MAXE, "prompt_expert_sets: expert index out of range [0, 1024)");
      E = std::max(E, e + 1);
    }
    DevBuf<int32_t> dt(trace_prompt, (size_t)m * T * k), dd(m), ds((size_t)m * k), dz(m);
    prompt_sets_kernel<<<m, 256, E * sizeof(int)>>>(dt.p, m, T, k, E, 0, dd.p, ds.p, dz.p);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    EMOE_CUDA(cudaDeviceSynchronize());
    dd.to_host(dominant);
    ds.to_host(sets);
    dz.to_host(sizes);
  });
}

int emoe_predict_host(emoe_predictor* P, int mode, const int32_t* sets, const int32_t* sizes, int layer,
                      double* scores, int32_t* experts, int32_t* n_experts) {
  return guard([&] {
    EMOE_REQUIRE(P, "predict: null predictor");
    validate_predict(P, mode, layer, sets, sizes);
    const int rows = mode == 0 ? P->m : 1;
    const int out_rows = mode == 1 ? P->m : rows;
    DevBuf<int32_t> dsets(sets, (size_t)rows * P->k), dsizes(sizes, rows);
    DevBuf<double> dsc((size_t)P->m * P->E);
    DevBuf<int32_t> dex((size_t)P->m * P->k), dn(P->m);
    EMOE_CUDA(cudaMemset(dex.p, 0xff, (size_t)P->m * P->k * sizeof(int32_t)));
    predict_kernel<<<1, 128>>>(make_predict_args(P, mode, layer, dsets.p, dsizes.p, dsc.p, dex.p, dn.p));
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    EMOE_CUDA(cudaDeviceSynchronize());
    std::vector<double> hs((size_t)P->m * P->E);
    std::vector<int32_t> he((size_t)P->m * P->k), hn(P->m);
    dsc.to_host(hs.data());
    dex.to_host(he.data());
    dn.to_host(hn.data());
    std::copy(hs.begin(), hs.begin() + (size_t)out_rows * P->E, scores);
    std::copy(he.begin(), he.begin() + (size_t)out_rows * P->k, experts);
    std::copy(hn.begin(), hn.begin() + out_rows, n_experts);
  });
}

int emoe_predicted_frequencies_host(emoe_predictor* P, int task, double* out) {
  return guard([&] {
    EMOE_REQUIRE(P && out, "predicted_frequencies: null argument");
    DevBuf<double> d((size_t)P->m * P->E);
    freq_kernel<<<1, 128>>>(P->task_counts, P->n_tasks, P->m, P->E, P->smoothing, task, d.p);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    EMOE_CUDA(cudaDeviceSynchronize());
    d.to_host(out);
  });
}

int emoe_expected_tokens_host(int m, int E, int n_tasks, const double* wo, const int32_t* sens, const uint8_t* has_sens,
                              int n_req, const int32_t* req_task, const int32_t* req_tokens,
                              const uint8_t* freq_present, const double* freqs, int task_aware, double* aggregate) {
  return guard([&] {
    validate_eq2(m, E, n_tasks, n_req, req_task);
    const size_t nt = std::max(1, n_tasks);
    DevBuf<double> dwo(nt), dfr(nt * m * E), dagg((size_t)m * E);
    DevBuf<int32_t> dsens(nt * m), drt(std::max(1, n_req)), drn(std::max(1, n_req));
    DevBuf<uint8_t> dhs(nt), dfp(nt);
    if (n_tasks) {
      EMOE_CUDA(cudaMemcpy(dwo.p, wo, n_tasks * sizeof(double), cudaMemcpyHostToDevice));
      EMOE_CUDA(cudaMemcpy(dsens.p, sens, (size_t)n_tasks * m * sizeof(int32_t), cudaMemcpyHostToDevice));
      EMOE_CUDA(cudaMemcpy(dhs.p, has_sens, n_tasks, cudaMemcpyHostToDevice));
      EMOE_CUDA(cudaMemcpy(dfp.p, freq_present, n_tasks, cudaMemcpyHostToDevice));
      EMOE_CUDA(cudaMemcpy(dfr.p, freqs, (size_t)n_tasks * m * E * sizeof(double), cudaMemcpyHostToDevice));
    }
    if (n_req) {
      EMOE_CUDA(cudaMemcpy(drt.p, req_task, n_req * sizeof(int32_t), cudaMemcpyHostToDevice));
      EMOE_CUDA(cudaMemcpy(drn.p, req_tokens, n_req * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    Eq2Args a{m, E, n_tasks, dwo.p, dsens.p, dhs.p, n_req, drt.p, drn.p, dfp.p, dfr.p, task_aware, dagg.p};
    eq2_kernel<<<1, 256>>>(a);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    EMOE_CUDA(cudaDeviceSynchronize());
    dagg.to_host(aggregate);
  });
}

static void run_plan(int m, int E, const double* aggregate, const uint8_t* resident, const int32_t* budgets,
                     double per_expert, int targets_given, int select_only, int32_t* targets, int32_t* target_sizes,
                     int32_t* ev, int32_t* nev, int32_t* ld, int32_t* nld, double* dur, double* de, int32_t* tl) {
  EMOE_REQUIRE(m >= 1 && E >= 1 && E <= MAXE, "plan: invalid shape");
  const size_t ME = (size_t)m * E;
  DevBuf<double> dagg(aggregate, ME), ddur(m), dde(1);
  DevBuf<uint8_t> dres(ME);
  if (resident)
    EMOE_CUDA(cudaMemcpy(dres.p, resident, ME, cudaMemcpyHostToDevice));
  else
    EMOE_CUDA(cudaMemset(dres.p, 0, ME));
  DevBuf<int32_t> dbud(budgets, m), dtg(ME), dts(m), dev(ME), dnev(m), dld(ME), dnld(m), dtl(1);
  if (targets_given) {
    EMOE_CUDA(cudaMemcpy(dtg.p, targets, ME * sizeof(int32_t), cudaMemcpyHostToDevice));
    EMOE_CUDA(cudaMemcpy(dts.p, target_sizes, m * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  PlanArgs a{m, E, dagg.p, dres.p, dbud.p, per_expert, dtg.p, dts.p, dev.p, dnev.p, dld.p, dnld.p, ddur.p, dde.p,
             dtl.p, targets_given, select_only};
  plan_kernel<<<1, 128>>>(a);
  EMOE_CUDA(cudaGetLastError());
    count_launch();
  EMOE_CUDA(cudaDeviceSynchronize());
  if (!targets_given) {
    if (targets) dtg.to_host(targets);
    if (target_sizes) dts.to_host(target_sizes);
  }
  if (!select_only) {
    if (ev) dev.to_host(ev);
    if (nev) dnev.to_host(nev);
    if (ld) dld.to_host(ld);
    if (nld) dnld.to_host(nld);
    if (dur) ddur.to_host(dur);
    if (de) dde.to_host(de);
    if (tl) dtl.to_host(tl);
  }
}

int emoe_select_experts_host(const double* aggregate, int m, int E, const int32_t* budgets, int32_t* out) {
  return guard([&] {
    validate_budgets(m, E, budgets);
    std::vector<int32_t> sizes(m);
    run_plan(m, E, aggregate, nullptr, budgets, 0.0, 0, 1, out, sizes.data(), nullptr, nullptr, nullptr, nullptr,
             nullptr, nullptr, nullptr);
  });
}

int emoe_loading_targets_host(const double* aggregate, int m, int E, const uint8_t* resident, const int32_t* budgets,
                              int32_t* out, int32_t* sizes) {
  return guard([&] {
    validate_budgets(m, E, budgets);
    std::vector<int32_t> ev((size_t)m * E), nev(m), ld((size_t)m * E), nld(m), tl(1);
    std::vector<double> dur(m), de(1);
    run_plan(m, E, aggregate, resident, budgets, 0.0, 0, 0, out, sizes, ev.data(), nev.data(), ld.data(), nld.data(),
             dur.data(), de.data(), tl.data());
  });
}

int emoe_plan_loading_host(const uint8_t* resident, const int32_t* budgets, int m, int E, const int32_t* target,
                           const int32_t* target_sizes, const double* aggregate, double per_expert, int32_t* ev,
                           int32_t* nev, int32_t* ld, int32_t* nld, double* dur, double* de, int32_t* tl) {
  return guard([&] {
    for (int l = 0; l < m; ++l) {
      if (target_sizes[l] > budgets[l]) throw ValidationError("plan_loading.target: exceeds layer budget");
      std::vector<char> seen(E, 0);
      for (int i = 0; i < target_sizes[l]; ++i) {
        const int e = target[l * E + i];
        if (e < 0 || e >= E) throw ValidationError("plan_loading.target: expert index out of range");
        if (seen[e]) throw ValidationError("plan_loading.target: duplicate expert index");
        seen[e] = 1;
      }
    }
    std::vector<int32_t> tg(target, target + (size_t)m * E), ts(target_sizes, target_sizes + m);
    run_plan(m, E, aggregate, resident, budgets, per_expert, 1, 0, tg.data(), ts.data(), ev, nev, ld, nld, dur, de,
             tl);
  });
}

int emoe_invocation_host(emoe_predictor* P, int mode, const int32_t* sets, const int32_t* sizes, int n_tasks,
                         const double* wo, const int32_t* sens, const uint8_t* has_sens, int n_req,
                         const int32_t* req_task, const int32_t* req_tokens, int task_aware, const uint8_t* resident,
                         const int32_t* budgets, double per_expert, double* aggregate, int32_t* evictions,
                         int32_t* n_evict, int32_t* loads, int32_t* n_load, double* delta_e) {
  return guard([&] {
    EMOE_REQUIRE(P, "invocation: null predictor");
    EMOE_REQUIRE(mode == 0 || mode == 1, "invocation: mode must be 0 (all layers) or 1 (chained)");
    EMOE_REQUIRE(n_tasks == P->n_tasks, "invocation: profile count must equal the predictor's task count");
    validate_predict(P, mode, 0, sets, sizes);
    validate_eq2(P->m, P->E, n_tasks, n_req, req_task);
    validate_budgets(P->m, P->E, budgets);
    const int m = P->m, E = P->E, k = P->k;
    const size_t ME = (size_t)m * E, nt = std::max(1, n_tasks);
    const int rows = mode == 0 ? m : 1;
    // arena layout: [uploaded inputs | downloaded outputs | device scratch]
    size_t off = 0;
    auto put = [&](size_t bytes) {
      const size_t o = off;
      off = (off + bytes + 255) / 256 * 256;
      return o;
    };
    const size_t o_sets = put((size_t)rows * k * 4), o_sizes = put((size_t)rows * 4), o_wo = put(nt * 8),
                 o_sens = put(nt * m * 4), o_hs = put(nt), o_fp = put(nt), o_rt = put(std::max(1, n_req) * 4),
                 o_rn = put(std::max(1, n_req) * 4), o_res = put(ME), o_bud = put((size_t)m * 4);
    const size_t in_bytes = off;
    const size_t o_agg = put(ME * 8), o_ev = put(ME * 4), o_nev = put((size_t)m * 4), o_ld = put(ME * 4),
                 o_nld = put((size_t)m * 4), o_de = put(8);
    const size_t out_end = off;
    const size_t o_ex = put((size_t)m * k * 4), o_n = put((size_t)m * 4), o_sc = put(ME * 8), o_fit = put(nt * ME * 8),
                 o_freq = put(nt * ME * 8), o_dur = put((size_t)m * 8), o_tg = put(ME * 4), o_ts = put((size_t)m * 4),
                 o_tl = put(4);
    P->arena_reserve(off);
    cudaStream_t s = P->inv_stream;
    EMOE_CUDA(cudaStreamSynchronize(s));  // the staging block is free (previous invocation done)
    uint8_t* h = P->arena_host;
    uint8_t* d = P->arena_dev;
    std::memcpy(h + o_sets, sets, (size_t)rows * k * 4);
    std::memcpy(h + o_sizes, sizes, (size_t)rows * 4);
    if (n_tasks) {
      std::memcpy(h + o_wo, wo, n_tasks * sizeof(double));
      std::memcpy(h + o_sens, sens, (size_t)n_tasks * m * sizeof(int32_t));
      std::memcpy(h + o_hs, has_sens, n_tasks);
      std::memset(h + o_fp, 1, n_tasks);
    }
    if (n_req) {
      std::memcpy(h + o_rt, req_task, n_req * sizeof(int32_t));
      std::memcpy(h + o_rn, req_tokens, n_req * sizeof(int32_t));
    }
    std::memcpy(h + o_res, resident, ME);
    std::memcpy(h + o_bud, budgets, (size_t)m * 4);
    auto i32 = [&](size_t o) { return reinterpret_cast<int32_t*>(d + o); };
    auto f64 = [&](size_t o) { return reinterpret_cast<double*>(d + o); };
    InvocationArgs a;
    a.pred = make_predict_args(P, mode, 0, i32(o_sets), i32(o_sizes), f64(o_sc), i32(o_ex), i32(o_n));
    a.task_counts = P->task_counts;
    a.n_tasks = n_tasks;
    a.fitted = f64(o_fit);
    a.freqs = f64(o_freq);
    a.eq2 = Eq2Args{m,         E,         n_tasks,       f64(o_wo),         i32(o_sens),
                    d + o_hs,  n_req,     i32(o_rt),     i32(o_rn),         d + o_fp,
                    f64(o_freq), task_aware, f64(o_agg)};
    a.plan = PlanArgs{m,          E,          f64(o_agg), d + o_res,  i32(o_bud), per_expert, i32(o_tg), i32(o_ts),
                      i32(o_ev),  i32(o_nev), i32(o_ld),  i32(o_nld), f64(o_dur), f64(o_de), i32(o_tl), 0,
                      0};
    if (P->hist_recorded) EMOE_CUDA(cudaStreamWaitEvent(s, P->hist_done, 0));
    EMOE_CUDA(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, s));
    const int blocks = mode == 0 ? m : 1;
    invocation_kernel<<<blocks, 128, 0, s>>>(a);
    EMOE_CUDA(cudaGetLastError());
    count_launch();
    if (blocks > 1) {
      plan_finalize_kernel<<<1, 32, 0, s>>>(a.plan);
      EMOE_CUDA(cudaGetLastError());
      count_launch();
    }
    EMOE_CUDA(cudaMemcpyAsync(h + o_agg, d + o_agg, out_end - o_agg, cudaMemcpyDeviceToHost, s));
    EMOE_CUDA(cudaStreamSynchronize(s));
    std::memcpy(aggregate, h + o_agg, ME * 8);
    std::memcpy(evictions, h + o_ev, ME * 4);
    std::memcpy(n_evict, h + o_nev, (size_t)m * 4);
    std::memcpy(loads, h + o_ld, ME * 4);
    std::memcpy(n_load, h + o_nld, (size_t)m * 4);
    std::memcpy(delta_e, h + o_de, 8);
  });
}

}  // extern "C"
