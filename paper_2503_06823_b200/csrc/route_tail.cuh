// Per-token routing shared by the gate kernels (route.cu, gate_tc.cu): the
// reference restatement run by one thread per token on its logits row
//   top-k        descending logit, ascending index on ties
//   route_token  first resident gate choice; else the resident expert with the
//                highest layer score, smallest index on ties; empty scores ->
//                smallest resident (expert_store.cpp:206-220)
//   forced miss  no resident expert -> {choice0, -1, miss} (engine.cpp:533-537)
// plus the builder-defined k-slot served set and weights.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace emoe {
namespace routing {

constexpr int MAX_E = 128;

struct SharedRouteState {
  uint8_t resident[MAX_E];
  double scores[MAX_E];
  int counts[MAX_E];
  int n_res;
  int first_res;
  int fallback;  // route_token's fallback expert: token-independent, computed once per block
};

// Residency tables into shared memory; warp 0 derives the resident count, the
// first resident and the fallback expert (largest layer score among residents,
// smallest index on ties: the serial scan of engine.cpp's route_token).
__device__ inline void load_route_state(SharedRouteState& st, const RouteArgs& a) {
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) {
    st.resident[e] = a.resident[e];
    st.scores[e] = a.scores ? a.scores[e] : 0.0;
    st.counts[e] = 0;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x;
    int n = 0, first = -1, be = -1;
    double bs = 0.0;
    for (int e0 = 0; e0 < a.E; e0 += 32) {
      const int e = e0 + lane;
      const bool r = e < a.E && st.resident[e];
      const unsigned m = __ballot_sync(FULL, r);
      n += __popc(m);
      if (first < 0 && m) first = e0 + __ffs(m) - 1;
      if (r && (be < 0 || st.scores[e] > bs)) {
        bs = st.scores[e];
        be = e;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double os = __shfl_xor_sync(FULL, bs, off);
      const int oe = __shfl_xor_sync(FULL, be, off);
      if (oe >= 0 && (be < 0 || os > bs || (os == bs && oe < be))) {
        bs = os;
        be = oe;
      }
    }
    if (lane == 0) {
      st.n_res = n;
      st.first_res = first;
      st.fallback = a.scores ? be : first;
    }
  }
  __syncthreads();
}

// Residency remap + served set + weights for one token whose ranked gate
// choices are ti[0..k).  lg = logits row (null for choice input: the served
// slots then share the weight uniformly).
__device__ inline void route_tail(const int* ti, const float* lg, int64_t t, const RouteArgs& a, const RouteOut& o,
                           SharedRouteState& st) {
  const int E = a.E, k = a.k;
  int ex = -1, rk = -1, hit = 0;
  if (st.n_res == 0) {
    ex = ti[0];
    if (!a.forced_miss) atomicExch(a.error_flag, 3);
  } else {
    for (int r = 0; r < k; ++r)
      if (st.resident[ti[r]]) {
        ex = ti[r];
        rk = r;
        hit = r == 0;
        break;
      }
    if (rk < 0) ex = st.fallback;
  }
  if (o.route_expert) o.route_expert[t] = ex;
  if (o.route_rank) o.route_rank[t] = rk;
  if (o.route_hit) o.route_hit[t] = (uint8_t)hit;

  int si[8];
  int ns = 0;
  if (st.n_res > 0) {
    if (rk >= 0) {
      for (int r = 0; r < k; ++r)
        if (st.resident[ti[r]]) si[ns++] = ti[r];
    } else {
      si[ns++] = ex;
    }
  }
  float w[8];
  if (lg == nullptr) {
    for (int j = 0; j < ns; ++j) w[j] = 1.0f / ns;
  } else if (a.weight_mode == 0) {
    if (ns > 0) {
      const float mx = lg[si[0]];
      float den = 0.0f;
      for (int j = 0; j < ns; ++j) {
        w[j] = expf(lg[si[j]] - mx);
        den += w[j];
      }
      for (int j = 0; j < ns; ++j) w[j] = w[j] / den;
    }
  } else {
    const float mx = lg[ti[0]];
    float den = 0.0f;
    for (int e = 0; e < E; ++e) den += expf(lg[e] - mx);
    for (int j = 0; j < ns; ++j) w[j] = expf(lg[si[j]] - mx) / den;
  }
  if (o.served_idx)
    for (int j = 0; j < k; ++j) {
      o.served_idx[t * k + j] = j < ns ? si[j] : -1;
      o.served_w[t * k + j] = j < ns ? w[j] : 0.0f;
    }
  for (int j = 0; j < ns; ++j) atomicAdd(&st.counts[si[j]], 1);
}

// One token from its logits row: top-k (descending, ascending index on ties) then route_tail.
__device__ inline void route_one_token(const float* lg, int64_t t, const RouteArgs& a, const RouteOut& o,
                                SharedRouteState& st) {
  const int E = a.E, k = a.k;
  int ti[8];
  uint32_t used[MAX_E / 32] = {0, 0, 0, 0};
  {  // first choice: plain argmax (no exclusions)
    int best = 0;
    float bv = lg[0];
    for (int e = 1; e < E; ++e) {
      const float v = lg[e];
      if (v > bv) {
        best = e;
        bv = v;
      }
    }
    ti[0] = best;
    used[best >> 5] |= 1u << (best & 31);
    if (o.topk_idx) o.topk_idx[t * k] = best;
  }
  for (int r = 1; r < k; ++r) {
    int best = -1;
    float bv = 0.0f;
    for (int e = 0; e < E; ++e) {
      if (used[e >> 5] & (1u << (e & 31))) continue;
      float v = lg[e];
      if (best < 0 || v > bv) {
        best = e;
        bv = v;
      }
    }
    ti[r] = best;
    used[best >> 5] |= 1u << (best & 31);
    if (o.topk_idx) o.topk_idx[t * k + r] = best;
  }
  route_tail(ti, lg, t, a, o, st);
}

}  // namespace routing
}  // namespace emoe
