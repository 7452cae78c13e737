// Synthetic routing-trace generator: the reference's Markov generator
// (workload.cpp:242-286 with make_calibration, :455-470) restated so the
// benchmark can build the same inputs without the reference.  The stream is
// std::mt19937_64 with the reference's hand-written transforms
// (distributions.hpp:12-34), so a seed gives the reference's trace bit for bit
// (checked against the reference-generated golden traces in
// tests/test_oracle.py::test_product_trace_generator_matches_golden).
#include <cstdint>
#include <random>
#include <vector>

#include "capi_util.h"

namespace {

struct Rng {
  std::mt19937_64 gen;
  explicit Rng(uint64_t seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
};

// inverse-CDF draw; numerical slack falls back to the last positive entry
int sample_row(const std::vector<double>& row, Rng& rng) {
  const double u = rng.uniform();
  double acc = 0.0;
  for (size_t i = 0; i < row.size(); ++i) {
    acc += row[i];
    if (u < acc) return static_cast<int>(i);
  }
  for (int i = static_cast<int>(row.size()) - 1; i >= 0; --i)
    if (row[i] > 0.0) return i;
  return static_cast<int>(row.size()) - 1;
}

// rank 0 given, ranks 1..k-1 drawn without replacement from the row's
// remaining mass; ascending fill once the mass is exhausted
void sample_topk(const std::vector<double>& row, int top1, int k, Rng& rng, int32_t* out) {
  std::vector<double> rest(row);
  rest[top1] = 0.0;
  out[0] = top1;
  int n = 1;
  while (n < k) {
    double total = 0.0;
    for (double v : rest) total += v;
    if (total <= 1e-12) {
      for (int e = 0; n < k; ++e) {
        bool dup = false;
        for (int q = 0; q < n; ++q) dup |= (out[q] == e);
        if (!dup) out[n++] = e;
      }
      break;
    }
    const double u = rng.uniform() * total;
    double acc = 0.0;
    int chosen = -1;
    for (size_t e = 0; e < rest.size(); ++e) {
      acc += rest[e];
      if (u < acc) {
        chosen = static_cast<int>(e);
        break;
      }
    }
    if (chosen < 0)
      for (int e = static_cast<int>(rest.size()) - 1; e >= 0; --e)
        if (rest[e] > 0.0) {
          chosen = e;
          break;
        }
    out[n++] = chosen;
    rest[chosen] = 0.0;
  }
}

// lam * I + (1 - lam) * U  (workload.cpp mixed_matrix)
std::vector<std::vector<double>> mixed(int e, double lam) {
  std::vector<std::vector<double>> m(e, std::vector<double>(e, (1.0 - lam) / static_cast<double>(e)));
  for (int i = 0; i < e; ++i) m[i][i] += lam;
  return m;
}

}  // namespace

extern "C" int emoe_gen_routing_trace(int m, int E, int k, double layer_lambda, double prompt_lambda,
                                      int initial_expert, uint64_t seed, int P, int T, int32_t* out) {
  return emoe::guard([&] {
    EMOE_REQUIRE(m >= 1 && E >= 1 && k >= 1 && k <= E, "gen_routing_trace: invalid shape");
    EMOE_REQUIRE(layer_lambda >= 0.0 && layer_lambda <= 1.0, "calibration.layer_lambda: must be in [0, 1]");
    EMOE_REQUIRE(prompt_lambda >= 0.0 && prompt_lambda <= 1.0, "calibration.prompt_lambda: must be in [0, 1]");
    EMOE_REQUIRE(initial_expert >= 0 && initial_expert < E, "calibration.initial_expert: out of range");
    EMOE_REQUIRE(P >= 1, "gen_routing_trace: prompts must be >= 1");
    EMOE_REQUIRE(T >= 1, "gen_routing_trace: tokens_per_prompt must be >= 1");
    const auto layer_t = mixed(E, layer_lambda);   // every layer transition is the same mixed matrix
    const auto prompt_t = mixed(E, prompt_lambda);  // only prompt_transition[0] drives the generator
    Rng rng(seed);
    int prev_dom0 = initial_expert;
    std::vector<int> count(E);
    for (int p = 0; p < P; ++p) {
      const auto& seed_row = prompt_t[prev_dom0];
      const int s = sample_row(seed_row, rng);
      std::fill(count.begin(), count.end(), 0);
      for (int t = 0; t < T; ++t) {
        int cur = s;
        sample_topk(seed_row, cur, k, rng, out + ((static_cast<int64_t>(p) * m + 0) * T + t) * k);
        ++count[cur];
        for (int l = 1; l < m; ++l) {
          const auto& row = layer_t[cur];
          cur = sample_row(row, rng);
          sample_topk(row, cur, k, rng, out + ((static_cast<int64_t>(p) * m + l) * T + t) * k);
        }
      }
      int best = 0;
      for (int e = 1; e < E; ++e)
        if (count[e] > count[best]) best = e;
      prev_dom0 = best;
    }
  });
}
