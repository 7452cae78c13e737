// C-ABI shim over the UNMODIFIED reference library (test infrastructure).
//
// Compiled by oracle/Makefile together with /root/reference/proj/core/src/*.cpp
// into oracle/_ref/libmoesim_ref.so.  Every entry point converts flat arrays
// into the reference's value types, calls the reference function named in its
// comment and flattens the result.  Nothing here re-implements reference
// logic: it is the "reference run here" that pins oracle/emoe_oracle.c, the
// golden fixtures under tests/golden/, and the CPU arm of bench.py
// (--impl reference).
//
// Return codes follow include/emoe.h: 0 ok, 2 ValidationError, 3 logic_error.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "moesim/engine.hpp"
#include "moesim/expert_store.hpp"
#include "moesim/predictor.hpp"
#include "moesim/report.hpp"
#include "moesim/workload.hpp"

using namespace moesim;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// flat trace [P][m][T][k] -> RoutingTrace
RoutingTrace make_trace(const int32_t* flat, int P, int m, int T, int k) {
  RoutingTrace t;
  t.num_layers = m;
  t.top_k = k;
  t.experts.assign(P, std::vector<std::vector<std::vector<int>>>(m, std::vector<std::vector<int>>(T, std::vector<int>(k))));
  for (int p = 0; p < P; ++p)
    for (int l = 0; l < m; ++l)
      for (int t2 = 0; t2 < T; ++t2)
        for (int r = 0; r < k; ++r)
          t.experts[p][l][t2][r] = flat[((static_cast<int64_t>(p) * m + l) * T + t2) * k + r];
  return t;
}

ModelShape make_shape(int m, int E, int k, uint64_t expert_bytes = 1, uint64_t base_bytes = 0) {
  ModelShape s;
  s.num_moe_layers = m;
  s.experts_per_layer = E;
  s.top_k = k;
  s.expert_bytes = expert_bytes;
  s.base_bytes = base_bytes;
  return s;
}

// resident bitmap [m][E] -> Placement with the given budgets (NULL = E)
Placement make_placement(const uint8_t* resident, const int32_t* budgets, int m, int E) {
  std::vector<int> b(m, E);
  if (budgets)
    for (int l = 0; l < m; ++l) b[l] = budgets[l];
  Placement p = Placement::empty(make_shape(m, E, 1), b);
  for (int l = 0; l < m; ++l)
    for (int e = 0; e < E; ++e)
      if (resident[l * E + e]) p.load(l, e);
  return p;
}

// flat model arrays -> TransitionModel.  task_counts is [n_tasks][m][E] with
// task names given in the same order.
TransitionModel make_model(int m, int E, int k, double smoothing, const double* layer_counts,
                           const double* prompt_counts, int n_tasks, const char* const* task_names,
                           const double* task_counts) {
  TransitionModel model;
  model.num_layers = m;
  model.num_experts = E;
  model.top_k = k;
  model.smoothing = smoothing;
  model.layer_counts.assign(m > 0 ? m - 1 : 0, Matrix(E, std::vector<double>(E, 0.0)));
  model.prompt_counts.assign(m, Matrix(E, std::vector<double>(E, 0.0)));
  for (int l = 0; l + 1 < m; ++l)
    for (int a = 0; a < E; ++a)
      for (int b = 0; b < E; ++b) model.layer_counts[l][a][b] = layer_counts[(l * E + a) * E + b];
  for (int l = 0; l < m; ++l)
    for (int a = 0; a < E; ++a)
      for (int b = 0; b < E; ++b) model.prompt_counts[l][a][b] = prompt_counts[(l * E + a) * E + b];
  for (int t = 0; t < n_tasks; ++t) {
    auto& rows = model.task_token_counts[task_names[t]];
    rows.assign(m, std::vector<double>(E, 0.0));
    for (int l = 0; l < m; ++l)
      for (int e = 0; e < E; ++e) rows[l][e] = task_counts[(static_cast<int64_t>(t) * m + l) * E + e];
  }
  return model;
}

void write_prediction(const Prediction& pred, int E, int k, double* scores, int32_t* experts,
                      int32_t* n_experts) {
  for (size_t l = 0; l < pred.layers.size(); ++l) {
    const auto& lp = pred.layers[l];
    for (int e = 0; e < E; ++e) scores[l * E + e] = lp.scores[e];
    n_experts[l] = static_cast<int32_t>(lp.experts.size());
    for (int r = 0; r < k; ++r)
      experts[l * k + r] = r < static_cast<int>(lp.experts.size()) ? lp.experts[r] : -1;
  }
}

std::vector<std::vector<int>> read_sets(const int32_t* sets, const int32_t* set_sizes, int m, int k) {
  std::vector<std::vector<int>> out(m);
  for (int l = 0; l < m; ++l)
    for (int r = 0; r < set_sizes[l]; ++r) out[l].push_back(sets[l * k + r]);
  return out;
}

std::vector<std::vector<double>> read_rows(const double* v, int m, int E) {
  std::vector<std::vector<double>> out(m, std::vector<double>(E));
  for (int l = 0; l < m; ++l)
    for (int e = 0; e < E; ++e) out[l][e] = v[l * E + e];
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// route_token (expert_store.cpp:206-220) per token; layer 0 of a 1-layer placement.
// n_scores == 0 passes the empty score vector.
int ref_route_tokens(const int32_t* choices, int64_t T, int k, const uint8_t* resident, int E,
                     const double* scores, int n_scores, int32_t* out_expert, int32_t* out_rank,
                     uint8_t* out_hit) {
  return guard([&] {
    Placement p = make_placement(resident, nullptr, 1, E);
    std::vector<double> sc(scores, scores + n_scores);
    std::vector<int> choice(k);
    for (int64_t t = 0; t < T; ++t) {
      for (int r = 0; r < k; ++r) choice[r] = choices[t * k + r];
      RouteResult res = route_token(choice, p, 0, sc);
      out_expert[t] = res.expert;
      out_rank[t] = res.rank;
      out_hit[t] = res.hit ? 1 : 0;
    }
  });
}

// Times route_token over T tokens held as the engine holds them (nested
// vectors, engine.cpp:538), best of `reps`; returns ns per token in *ns.
int ref_time_route_tokens(const int32_t* choices, int64_t T, int k, const uint8_t* resident, int E,
                          const double* scores, int n_scores, int reps, double* ns_per_token,
                          int64_t* hits) {
  return guard([&] {
    Placement p = make_placement(resident, nullptr, 1, E);
    std::vector<double> sc(scores, scores + n_scores);
    std::vector<std::vector<int>> toks(T, std::vector<int>(k));
    for (int64_t t = 0; t < T; ++t)
      for (int r = 0; r < k; ++r) toks[t][r] = choices[t * k + r];
    double best = 1e300;
    int64_t h = 0;
    for (int rep = 0; rep < reps; ++rep) {
      h = 0;
      auto t0 = std::chrono::steady_clock::now();
      for (int64_t t = 0; t < T; ++t) {
        RouteResult res = route_token(toks[t], p, 0, sc);
        h += res.hit ? 1 : 0;
      }
      auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double, std::nano>(t1 - t0).count());
    }
    *ns_per_token = best / static_cast<double>(T > 0 ? T : 1);
    *hits = h;
  });
}

// fit (predictor.cpp:137-185).  task_ids: per-prompt index into task_names or
// NULL (no per-task tallies).  Outputs are dense, tasks in std::map order,
// which is also the order of the sorted names the caller passes back.
int ref_fit(const int32_t* trace, int P, int m, int T, int k, const int32_t* task_ids,
            const char* const* task_names, double smoothing, int num_experts, int32_t* out_E,
            double* layer_counts, double* prompt_counts, double* task_counts, int32_t* out_n_tasks) {
  return guard([&] {
    RoutingTrace t = make_trace(trace, P, m, T, k);
    std::vector<std::string> ids;
    if (task_ids)
      for (int p = 0; p < P; ++p) ids.push_back(task_names[task_ids[p]]);
    TransitionModel model = fit(t, ids, smoothing, num_experts);
    const int E = model.num_experts;
    *out_E = E;
    for (int l = 0; l + 1 < m; ++l)
      for (int a = 0; a < E; ++a)
        for (int b = 0; b < E; ++b) layer_counts[(l * E + a) * E + b] = model.layer_counts[l][a][b];
    for (int l = 0; l < m; ++l)
      for (int a = 0; a < E; ++a)
        for (int b = 0; b < E; ++b) prompt_counts[(l * E + a) * E + b] = model.prompt_counts[l][a][b];
    int ti = 0;
    for (const auto& [name, rows] : model.task_token_counts) {
      for (int l = 0; l < m; ++l)
        for (int e = 0; e < E; ++e) task_counts[(static_cast<int64_t>(ti) * m + l) * E + e] = rows[l][e];
      ++ti;
    }
    *out_n_tasks = ti;
  });
}

int ref_time_fit(const int32_t* trace, int P, int m, int T, int k, int num_experts, int reps,
                 double* ns) {
  return guard([&] {
    RoutingTrace t = make_trace(trace, P, m, T, k);
    double best = 1e300;
    for (int rep = 0; rep < reps; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      TransitionModel model = fit(t, {}, 0.01, num_experts);
      auto t1 = std::chrono::steady_clock::now();
      if (model.num_experts < 1) throw std::runtime_error("fit");
      best = std::min(best, std::chrono::duration<double, std::nano>(t1 - t0).count());
    }
    *ns = best;
  });
}

// dominant_expert / prompt_expert_sets (workload.cpp:350-377)
int ref_prompt_expert_sets(const int32_t* trace, int P, int m, int T, int k, int prompt,
                           int32_t* dominant, int32_t* sets, int32_t* set_sizes) {
  return guard([&] {
    RoutingTrace t = make_trace(trace, P, m, T, k);
    for (int l = 0; l < m; ++l) dominant[l] = dominant_expert(t, prompt, l);
    auto s = prompt_expert_sets(t, prompt);
    for (int l = 0; l < m; ++l) {
      set_sizes[l] = static_cast<int32_t>(s[l].size());
      for (int r = 0; r < k; ++r) sets[l * k + r] = r < static_cast<int>(s[l].size()) ? s[l][r] : -1;
    }
  });
}

// predict_all_layers / predict_chained / predict_layerwise (predictor.cpp:187-220)
// mode 0 = all_layers (prev sets [m][k] + sizes), 1 = chained (prev sets row 0),
// 2 = layerwise (prev sets row 0, `layer`; writes only row 0 of the outputs)
int ref_predict(int m, int E, int k, double smoothing, const double* layer_counts,
                const double* prompt_counts, int mode, const int32_t* prev_sets,
                const int32_t* prev_sizes, int layer, double* scores, int32_t* experts,
                int32_t* n_experts) {
  return guard([&] {
    TransitionModel model = make_model(m, E, k, smoothing, layer_counts, prompt_counts, 0, nullptr, nullptr);
    auto sets = read_sets(prev_sets, prev_sizes, mode == 0 ? m : 1, k);
    if (mode == 0) {
      write_prediction(predict_all_layers(model, sets), E, k, scores, experts, n_experts);
    } else if (mode == 1) {
      write_prediction(predict_chained(model, sets[0]), E, k, scores, experts, n_experts);
    } else {
      Prediction p;
      p.layers.push_back(predict_layerwise(model, sets[0], layer));
      write_prediction(p, E, k, scores, experts, n_experts);
    }
  });
}

// predicted_frequencies (predictor.cpp:222-238)
int ref_predicted_frequencies(int m, int E, int n_tasks, const char* const* task_names,
                              const double* task_counts, double smoothing, const char* task,
                              double* out) {
  return guard([&] {
    std::vector<double> zeros(static_cast<size_t>(m) * E * E, 0.0);
    TransitionModel model = make_model(m, E, 1, smoothing, zeros.data(), zeros.data(), n_tasks,
                                       task_names, task_counts);
    auto f = predicted_frequencies(model, task);
    for (int l = 0; l < m; ++l)
      for (int e = 0; e < E; ++e) out[l * E + e] = f[l][e];
  });
}

// expected_tokens (expert_store.cpp:59-106).  Profiles: n_profiles task ids
// with wo() (expected_output_tokens) and sensitivity [n_profiles][m] (or a
// NULL row pointer via has_sens[i]==0 = empty vector).  Requests: task index +
// input tokens, running then incoming.  freqs: [n_freq][m][E] for the named
// tasks.  Outputs the per-layer aggregate [m][E].
int ref_expected_tokens(int m, int E, int n_profiles, const char* const* profile_ids,
                        const double* wo, const int32_t* sensitivity, const uint8_t* has_sens,
                        int n_running, const int32_t* running_task, const int32_t* running_tokens,
                        int n_incoming, const int32_t* incoming_task, const int32_t* incoming_tokens,
                        int n_freq, const char* const* freq_ids, const double* freqs, int task_aware,
                        double* aggregate) {
  return guard([&] {
    ModelShape shape = make_shape(m, E, 1);
    std::vector<TaskProfile> profiles(n_profiles);
    for (int i = 0; i < n_profiles; ++i) {
      profiles[i].task_id = profile_ids[i];
      profiles[i].expected_output_tokens = wo[i];
      profiles[i].output_tokens = {LengthDist::Family::constant, wo[i] > 0 ? wo[i] : 1.0, 0.0};
      if (has_sens[i]) profiles[i].sensitivity.assign(sensitivity + i * m, sensitivity + (i + 1) * m);
    }
    auto mk = [&](int n, const int32_t* task, const int32_t* toks) {
      std::vector<Request> out(n);
      for (int i = 0; i < n; ++i) {
        out[i].request_id = static_cast<uint64_t>(i);
        out[i].task_id = task[i] >= 0 ? profiles[task[i]].task_id : std::string("__unknown__");
        out[i].input_tokens = toks[i];
      }
      return out;
    };
    std::map<std::string, std::vector<std::vector<double>>> fm;
    for (int i = 0; i < n_freq; ++i)
      fm[freq_ids[i]] = read_rows(freqs + static_cast<int64_t>(i) * m * E, m, E);
    ExpectedTokens et = expected_tokens(shape, profiles, mk(n_running, running_task, running_tokens),
                                        mk(n_incoming, incoming_task, incoming_tokens), fm,
                                        task_aware != 0);
    for (int l = 0; l < m; ++l)
      for (int e = 0; e < E; ++e) aggregate[l * E + e] = et.aggregate[l][e];
  });
}

// select_experts (expert_store.cpp:123-138): out [m][E] (first budgets[l] valid)
int ref_select_experts(const double* aggregate, int m, int E, const int32_t* budgets, int32_t* out) {
  return guard([&] {
    auto sel = select_experts(read_rows(aggregate, m, E), make_shape(m, E, 1),
                              std::vector<int>(budgets, budgets + m));
    for (int l = 0; l < m; ++l)
      for (size_t i = 0; i < sel[l].size(); ++i) out[l * E + i] = sel[l][i];
  });
}

// loading_targets (expert_store.cpp:140-157): out [m][E] + sizes
int ref_loading_targets(const double* aggregate, int m, int E, const uint8_t* resident,
                        const int32_t* budgets, int32_t* out, int32_t* sizes) {
  return guard([&] {
    Placement cur = make_placement(resident, nullptr, m, E);
    auto tg = loading_targets(read_rows(aggregate, m, E), cur, std::vector<int>(budgets, budgets + m));
    for (int l = 0; l < m; ++l) {
      sizes[l] = static_cast<int32_t>(tg[l].size());
      for (size_t i = 0; i < tg[l].size(); ++i) out[l * E + i] = tg[l][i];
    }
  });
}

// plan_loading (expert_store.cpp:159-195).  Placement budgets come from
// `budgets`; cost = per_expert + expert_bytes / bw.  Outputs per layer:
// evictions [m][E] + n_evict, loads [m][E] + n_load, duration [m]; delta_e.
int ref_plan_loading(const uint8_t* resident, const int32_t* budgets, int m, int E,
                     const int32_t* target, const int32_t* target_sizes, const double* aggregate,
                     double per_expert, double hd_bandwidth, uint64_t expert_bytes,
                     int32_t* evictions, int32_t* n_evict, int32_t* loads, int32_t* n_load,
                     double* duration, double* delta_e, int32_t* total_loads) {
  return guard([&] {
    std::vector<int> b(budgets, budgets + m);
    ModelShape shape = make_shape(m, E, 1, expert_bytes, 0);
    Placement cur = Placement::empty(shape, b);
    for (int l = 0; l < m; ++l)
      for (int e = 0; e < E; ++e)
        if (resident[l * E + e]) cur.load(l, e);
    std::vector<std::vector<int>> tg(m);
    for (int l = 0; l < m; ++l) tg[l].assign(target + l * E, target + l * E + target_sizes[l]);
    CostModel cost;
    cost.per_expert_transfer = per_expert;
    cost.hd_bandwidth = hd_bandwidth;
    LoadingPlan plan = plan_loading(cur, tg, read_rows(aggregate, m, E), cost);
    for (int l = 0; l < m; ++l) {
      const auto& ops = plan.layers[l];
      n_evict[l] = static_cast<int32_t>(ops.evictions.size());
      n_load[l] = static_cast<int32_t>(ops.loads.size());
      for (size_t i = 0; i < ops.evictions.size(); ++i) evictions[l * E + i] = ops.evictions[i];
      for (size_t i = 0; i < ops.loads.size(); ++i) loads[l * E + i] = ops.loads[i];
      duration[l] = ops.duration;
    }
    *delta_e = plan.delta_e;
    *total_loads = plan.total_loads;
  });
}

// gen_routing_trace(shape, make_calibration(...)) (workload.cpp:242-286, :455)
int ref_gen_routing_trace(int m, int E, int k, double layer_lambda, double prompt_lambda,
                          int initial_expert, uint64_t seed, int P, int T, int32_t* out) {
  return guard([&] {
    ModelShape shape = make_shape(m, E, k, 1, 0);
    RoutingTrace t = gen_routing_trace(shape, make_calibration(shape, layer_lambda, prompt_lambda,
                                                               initial_expert, seed),
                                       P, T);
    for (int p = 0; p < P; ++p)
      for (int l = 0; l < m; ++l)
        for (int t2 = 0; t2 < T; ++t2)
          for (int r = 0; r < k; ++r)
            out[((static_cast<int64_t>(p) * m + l) * T + t2) * k + r] = t.experts[p][l][t2][r];
  });
}

// save_trace (report.cpp:260-267) / save_model (predictor.cpp:240-252) of a
// flat trace / fitted model, for byte-compatibility checks of the formats
int ref_save_trace(const int32_t* trace, int P, int m, int T, int k, const char* path) {
  return guard([&] { save_trace(make_trace(trace, P, m, T, k), path); });
}
int ref_fit_and_save_model(const int32_t* trace, int P, int m, int T, int k, const int32_t* task_ids,
                           const char* const* task_names, double smoothing, int num_experts, const char* path) {
  return guard([&] {
    RoutingTrace t = make_trace(trace, P, m, T, k);
    std::vector<std::string> ids;
    if (task_ids)
      for (int p = 0; p < P; ++p) ids.push_back(task_names[task_ids[p]]);
    save_model(fit(t, ids, smoothing, num_experts), path);
  });
}

// Rng (distributions.hpp:12-34): n uniform() / normal() draws from Rng(seed)
int ref_rng_uniform(uint64_t seed, int64_t n, double* out) {
  return guard([&] {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.uniform();
  });
}
int ref_rng_normal(uint64_t seed, int64_t n, double* out) {
  return guard([&] {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.normal();
  });
}

}  // extern "C"
