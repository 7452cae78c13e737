"""Host-side mirror of the reference ``moesim`` operator API for the hot path.

Same names, argument meaning and error behaviour as the reference C++ library
(/root/reference/proj/core/include/moesim/{expert_store,predictor,workload}.hpp);
every compute call goes through the C ABI in include/emoe.h into the sm_100a
kernels of lib/libemoe.so.  Errors map exactly as the ABI's return codes do:
``ValidationError`` (moesim::ValidationError), ``LogicError``
(std::logic_error), ``RuntimeError`` (CUDA).

Only ``Placement`` keeps host-side bookkeeping (as the reference does,
expert_store.cpp:11-57); the device copy of the residency table lives in
``MoELayer`` (layer.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from ._lib import lib


class ValidationError(ValueError):
    """moesim::ValidationError (types.hpp:11-14)."""


class LogicError(RuntimeError):
    """std::logic_error from the reference (expert_store.cpp:47-54, :213)."""


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.emoe_last_error().decode()
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise LogicError(msg)
    raise RuntimeError(msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _arr(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


# ---------------------------------------------------------------------------
# types (types.hpp, workload.hpp, cost_model.hpp)
# ---------------------------------------------------------------------------
@dataclass
class ModelShape:
    num_moe_layers: int = 0
    experts_per_layer: int = 0
    top_k: int = 0
    expert_bytes: int = 0
    base_bytes: int = 0

    def full_expert_bytes(self) -> int:
        return self.num_moe_layers * self.experts_per_layer * self.expert_bytes


@dataclass
class TaskProfile:
    """The fields of TaskProfile (workload.hpp:14-30) Eq. 2 reads."""
    task_id: str
    expected_output_tokens: float = 0.0  # W_o
    output_mean: float = 1.0             # output_tokens.mean() fallback
    sensitivity: List[int] = field(default_factory=list)

    def wo(self) -> float:
        return self.expected_output_tokens if self.expected_output_tokens > 0.0 else self.output_mean


@dataclass
class Request:
    task_id: str
    input_tokens: int
    request_id: int = 0


@dataclass
class CostModel:
    per_token_cost: float = 0.0
    per_expert_transfer: float = 0.0
    hd_bandwidth: float = 1.0
    predictor_invocation_cost: float = 0.0
    contention_factor: float = 1.0

    def expert_transfer_seconds(self, expert_bytes: int) -> float:
        return self.per_expert_transfer + float(expert_bytes) / self.hd_bandwidth


@dataclass
class RouteResult:
    expert: int = -1
    rank: int = -1
    hit: bool = False


# ---------------------------------------------------------------------------
# Placement (expert_store.hpp:15-43): host bookkeeping, exact byte accounting
# ---------------------------------------------------------------------------
class Placement:
    def __init__(self, shape: ModelShape, budget_per_layer: Sequence[int]):
        if shape.num_moe_layers < 1 or shape.experts_per_layer < 1:
            raise ValidationError("model: num_moe_layers and experts_per_layer must be >= 1")
        if len(budget_per_layer) != shape.num_moe_layers:
            raise ValidationError("placement.budget_per_layer: must have one entry per layer")
        for b in budget_per_layer:
            if b < 0 or b > shape.experts_per_layer:
                raise ValidationError("placement.budget_per_layer: entries must be in [0, experts_per_layer]")
        self._shape = shape
        self._budgets = [int(b) for b in budget_per_layer]
        self._resident = np.zeros((shape.num_moe_layers, shape.experts_per_layer), np.uint8)

    @staticmethod
    def full(shape: ModelShape) -> "Placement":
        p = Placement(shape, [shape.experts_per_layer] * shape.num_moe_layers)
        p._resident[:] = 1
        return p

    @staticmethod
    def empty(shape: ModelShape, budget_per_layer: Sequence[int]) -> "Placement":
        return Placement(shape, budget_per_layer)

    def resident(self, layer: int, expert: int) -> bool:
        return bool(self._resident[layer, expert])

    def residents(self, layer: int) -> List[int]:
        return [int(e) for e in np.flatnonzero(self._resident[layer])]

    def resident_count(self, layer: int) -> int:
        return int(self._resident[layer].sum())

    def budget(self, layer: int) -> int:
        return self._budgets[layer]

    def budgets(self) -> List[int]:
        return list(self._budgets)

    def shape(self) -> ModelShape:
        return self._shape

    def bitmap(self) -> np.ndarray:
        return self._resident.copy()

    def expert_bytes_used(self) -> int:
        return int(self._resident.sum()) * self._shape.expert_bytes

    def device_bytes_used(self) -> int:
        return self._shape.base_bytes + self.expert_bytes_used()

    def evict(self, layer: int, expert: int) -> None:
        if not self._resident[layer, expert]:
            raise LogicError("placement: evicting non-resident expert")
        self._resident[layer, expert] = 0

    def load(self, layer: int, expert: int) -> None:
        if self._resident[layer, expert]:
            raise LogicError("placement: loading resident expert")
        if self.resident_count(layer) >= self._budgets[layer]:
            raise LogicError("placement: layer budget exceeded")
        self._resident[layer, expert] = 1


# ---------------------------------------------------------------------------
# A2 route_token (expert_store.cpp:206-220), batched on the GPU
# ---------------------------------------------------------------------------
def route_tokens(choices: np.ndarray, resident: np.ndarray, scores: Optional[Sequence[float]] = None):
    """Batched route_token: choices [T, k] ranked gate choices, resident [E] 0/1."""
    choices = _arr(choices, np.int32)
    T, k = choices.shape
    resident = _arr(resident, np.uint8)
    E = resident.shape[0]
    sc = None if scores is None or len(scores) == 0 else _arr(scores, np.float64)
    ex = np.empty(T, np.int32)
    rk = np.empty(T, np.int32)
    hit = np.empty(T, np.uint8)
    check(lib.emoe_route_tokens_host(_p(choices), T, k, _p(resident), E, None if sc is None else _p(sc), _p(ex),
                                     _p(rk), _p(hit)))
    return ex, rk, hit


def route_token(gate_choice: Sequence[int], placement: Placement, layer: int,
                layer_scores: Sequence[float]) -> RouteResult:
    ex, rk, hit = route_tokens(np.asarray([gate_choice], np.int32), placement.bitmap()[layer], layer_scores)
    return RouteResult(int(ex[0]), int(rk[0]), bool(hit[0]))


# ---------------------------------------------------------------------------
# A6/A7 predictor (predictor.hpp)
# ---------------------------------------------------------------------------
@dataclass
class TransitionModel:
    num_layers: int
    num_experts: int
    top_k: int
    smoothing: float
    layer_counts: np.ndarray    # [m-1, E, E]
    prompt_counts: np.ndarray   # [m, E, E]
    task_ids: List[str]         # sorted (std::map order)
    task_counts: np.ndarray     # [n_tasks, m, E]

    def task_token_counts(self) -> Dict[str, np.ndarray]:
        return {t: self.task_counts[i] for i, t in enumerate(self.task_ids)}


@dataclass
class LayerPrediction:
    experts: List[int]
    scores: np.ndarray


class _Pred:
    """RAII wrapper of an emoe_predictor handle."""

    def __init__(self, m, E, k, n_tasks, smoothing):
        h = C.c_void_p()
        check(lib.emoe_predictor_create(m, E, k, n_tasks, smoothing, C.byref(h)))
        self.h = h

    @staticmethod
    def from_model(model: TransitionModel) -> "_Pred":
        p = _Pred(model.num_layers, model.num_experts, model.top_k, len(model.task_ids), model.smoothing)
        lc = _arr(model.layer_counts, np.float64)
        pc = _arr(model.prompt_counts, np.float64)
        tc = _arr(model.task_counts, np.float64)
        check(lib.emoe_predictor_set_counts_host(p.h, _p(lc) if lc.size else None, _p(pc), _p(tc) if tc.size else None))
        return p

    def __del__(self):
        if getattr(self, "h", None):
            lib.emoe_predictor_destroy(self.h)
            self.h = None


def fit(trace: np.ndarray, task_ids: Sequence[str] = (), smoothing: float = 0.01,
        num_experts: int = 0) -> TransitionModel:
    """fit (predictor.cpp:137-185) on the GPU.  trace: [P, m, T, k] int32."""
    import torch

    trace = _arr(trace, np.int32)
    if trace.ndim != 4 or trace.shape[0] == 0 or trace.shape[1] < 1:
        raise ValidationError("predictor.trace: empty")
    P, m, T, k = trace.shape
    if len(task_ids) and len(task_ids) != P:
        raise ValidationError("predictor.task_ids: size must match prompt count")
    E = num_experts if num_experts > 0 else int(trace.max()) + 1
    if E < 1:
        raise ValidationError("predictor.trace: no experts")
    if (trace < 0).any() or (trace >= E).any():
        raise ValidationError("predictor.trace: expert index out of range")
    names = sorted(set(task_ids))
    pred = _Pred(m, E, k, len(names), smoothing)
    dtrace = torch.from_numpy(trace).cuda()
    tid = None
    if len(task_ids):
        index = {n: i for i, n in enumerate(names)}
        tid = torch.tensor([index[t] for t in task_ids], dtype=torch.int32, device="cuda")
    check(lib.emoe_hist_update(pred.h, C.c_void_p(dtrace.data_ptr()), P, T,
                               None if tid is None else C.c_void_p(tid.data_ptr()), None))
    lc = np.zeros((max(m - 1, 0), E, E), np.float64)
    pc = np.zeros((m, E, E), np.float64)
    tc = np.zeros((len(names), m, E), np.float64)
    check(lib.emoe_predictor_counts_host(pred.h, _p(lc) if lc.size else None, _p(pc), _p(tc) if tc.size else None))
    return TransitionModel(m, E, k, smoothing, lc, pc, names, tc)


def _sets_array(sets: Sequence[Sequence[int]], k: int):
    arr = np.full((len(sets), k), -1, np.int32)
    sizes = np.zeros(len(sets), np.int32)
    for l, s in enumerate(sets):
        if len(s) > k:
            raise ValidationError("predictor: expert set larger than top_k")
        arr[l, : len(s)] = s
        sizes[l] = len(s)
    return arr, sizes


def _predict(model: TransitionModel, mode: int, sets, layer: int = 0):
    pred = _Pred.from_model(model)
    arr, sizes = _sets_array(sets, model.top_k)
    rows = model.num_layers if mode in (0, 1) else 1
    scores = np.zeros((rows, model.num_experts), np.float64)
    experts = np.full((rows, model.top_k), -1, np.int32)
    n = np.zeros(rows, np.int32)
    check(lib.emoe_predict_host(pred.h, mode, _p(arr), _p(sizes), layer, _p(scores), _p(experts), _p(n)))
    return [LayerPrediction([int(e) for e in experts[l, : n[l]]], scores[l]) for l in range(rows)]


def predict_layerwise(model: TransitionModel, prev_layer_experts: Sequence[int], layer: int) -> LayerPrediction:
    return _predict(model, 2, [list(prev_layer_experts)], layer)[0]


def predict_all_layers(model: TransitionModel, prev_prompt_experts: Sequence[Sequence[int]]) -> List[LayerPrediction]:
    if len(prev_prompt_experts) != model.num_layers:
        raise ValidationError("predictor.prev_prompt: layer count mismatch")
    return _predict(model, 0, prev_prompt_experts)


def predict_chained(model: TransitionModel, prev_prompt_layer0: Sequence[int]) -> List[LayerPrediction]:
    return _predict(model, 1, [list(prev_prompt_layer0)])


def predicted_frequencies(model: TransitionModel, task_id: str) -> np.ndarray:
    pred = _Pred.from_model(model)
    task = model.task_ids.index(task_id) if task_id in model.task_ids else -1
    out = np.zeros((model.num_layers, model.num_experts), np.float64)
    check(lib.emoe_predicted_frequencies_host(pred.h, task, _p(out)))
    return out


# ---------------------------------------------------------------------------
# A7/A8 expected_tokens, selection, planning (expert_store.hpp:45-99)
# ---------------------------------------------------------------------------
@dataclass
class ExpectedTokens:
    task_ids: List[str]
    values: np.ndarray      # [n_tasks_with_requests, m, E]
    aggregate: np.ndarray   # [m, E]


def _profile_arrays(profiles: Sequence[TaskProfile], m: int):
    by_id = {p.task_id: p for p in profiles}
    names = sorted(by_id)
    wo = np.array([by_id[n].wo() for n in names], np.float64)
    sens = np.zeros((max(len(names), 1), m), np.int32)
    has = np.zeros(max(len(names), 1), np.uint8)
    for i, n in enumerate(names):
        if by_id[n].sensitivity:
            has[i] = 1
            sens[i] = by_id[n].sensitivity
    return names, wo, sens, has


def _request_arrays(names, running, incoming):
    index = {n: i for i, n in enumerate(names)}
    reqs = list(running) + list(incoming)
    for r in reqs:
        if r.task_id not in index:
            raise ValidationError("expected_tokens.request: unknown task_id " + r.task_id)
    rt = np.array([index[r.task_id] for r in reqs] or [0], np.int32)
    rn = np.array([r.input_tokens for r in reqs] or [0], np.int32)
    return len(reqs), rt, rn


def expected_tokens(shape: ModelShape, profiles: Sequence[TaskProfile], running: Sequence[Request],
                    incoming: Sequence[Request], frequencies: Dict[str, np.ndarray],
                    task_aware: bool = True) -> ExpectedTokens:
    m, E = shape.num_moe_layers, shape.experts_per_layer
    names, wo, sens, has = _profile_arrays(profiles, m)
    n_req, rt, rn = _request_arrays(names, running, incoming)
    fp = np.array([1 if n in frequencies else 0 for n in names] or [0], np.uint8)
    fr = np.zeros((max(len(names), 1), m, E), np.float64)
    for i, n in enumerate(names):
        if n in frequencies:
            fr[i] = np.asarray(frequencies[n], np.float64)
    agg = np.zeros((m, E), np.float64)
    check(lib.emoe_expected_tokens_host(m, E, len(names), _p(wo) if len(names) else None, _p(sens), _p(has), n_req,
                                        _p(rt), _p(rn), _p(fp), _p(fr), int(task_aware), _p(agg)))
    # per-task grids (volume * f on sensitive layers), reported like the reference
    used = sorted({names[i] for i in rt[:n_req]})
    values = []
    for n in used:
        i = names.index(n)
        sel = rt[:n_req] == i
        volume = float(rn[:n_req][sel].astype(np.float64).sum()) + int(sel.sum()) * wo[i]
        f = fr[i] if fp[i] else np.full((m, E), 1.0 / E)
        g = volume * f
        if task_aware and has[i]:
            g = g * (sens[i][:, None] != 0)
        values.append(g)
    return ExpectedTokens(used, np.array(values).reshape(len(used), m, E), agg)


def select_experts(aggregate: np.ndarray, shape: ModelShape, budgets: Sequence[int]) -> List[List[int]]:
    aggregate = _arr(aggregate, np.float64)
    if aggregate.shape[0] != shape.num_moe_layers:
        raise ValidationError("select_experts.aggregate: must have one row per layer")
    if len(budgets) != aggregate.shape[0]:
        raise ValidationError("select_experts.budgets: must have one entry per layer")
    m, E = aggregate.shape
    b = _arr(budgets, np.int32)
    out = np.full((m, E), -1, np.int32)
    check(lib.emoe_select_experts_host(_p(aggregate), m, E, _p(b), _p(out)))
    return [[int(e) for e in out[l, : b[l]]] for l in range(m)]


def loading_targets(aggregate: np.ndarray, current: Placement, budgets: Sequence[int]) -> List[List[int]]:
    aggregate = _arr(aggregate, np.float64)
    m, E = aggregate.shape
    if m != current.shape().num_moe_layers:
        raise ValidationError("select_experts.aggregate: must have one row per layer")
    if len(budgets) != m:
        raise ValidationError("select_experts.budgets: must have one entry per layer")
    b = _arr(budgets, np.int32)
    out = np.full((m, E), -1, np.int32)
    sizes = np.zeros(m, np.int32)
    res = _arr(current.bitmap(), np.uint8)
    check(lib.emoe_loading_targets_host(_p(aggregate), m, E, _p(res), _p(b), _p(out), _p(sizes)))
    return [[int(e) for e in out[l, : sizes[l]]] for l in range(m)]


@dataclass
class LayerOps:
    layer: int
    evictions: List[int]
    loads: List[int]
    duration: float


@dataclass
class LoadingPlan:
    layers: List[LayerOps]
    delta_e: float
    total_loads: int

    def empty(self) -> bool:
        return self.total_loads == 0


def plan_loading(current: Placement, target: Sequence[Sequence[int]], aggregate: np.ndarray,
                 cost: CostModel) -> LoadingPlan:
    shape = current.shape()
    m, E = shape.num_moe_layers, shape.experts_per_layer
    if len(target) != m:
        raise ValidationError("plan_loading.target: must have one set per layer")
    agg = np.zeros((m, E), np.float64)
    aggregate = np.asarray(aggregate, np.float64)
    agg[: min(m, aggregate.shape[0])] = aggregate[:m]
    tg = np.full((m, E), -1, np.int32)
    ts = np.zeros(m, np.int32)
    for l, t in enumerate(target):
        if len(t) > E:
            raise ValidationError("plan_loading.target: exceeds layer budget")
        tg[l, : len(t)] = t
        ts[l] = len(t)
    b = _arr(current.budgets(), np.int32)
    ev = np.full((m, E), -1, np.int32)
    ld = np.full((m, E), -1, np.int32)
    ne = np.zeros(m, np.int32)
    nl = np.zeros(m, np.int32)
    dur = np.zeros(m, np.float64)
    de = np.zeros(1, np.float64)
    tl = np.zeros(1, np.int32)
    res = _arr(current.bitmap(), np.uint8)
    check(lib.emoe_plan_loading_host(_p(res), _p(b), m, E, _p(tg), _p(ts), _p(agg),
                                     cost.expert_transfer_seconds(shape.expert_bytes), _p(ev), _p(ne), _p(ld), _p(nl),
                                     _p(dur), _p(de), _p(tl)))
    layers = [LayerOps(l, [int(e) for e in ev[l, : ne[l]]], [int(e) for e in ld[l, : nl[l]]], float(dur[l]))
              for l in range(m)]
    return LoadingPlan(layers, float(de[0]), int(tl[0]))


def apply_plan_layer(placement: Placement, ops: LayerOps) -> None:
    for e in ops.evictions:
        placement.evict(ops.layer, e)
    for e in ops.loads:
        placement.load(ops.layer, e)


def apply_plan(placement: Placement, plan: LoadingPlan) -> None:
    for ops in plan.layers:
        apply_plan_layer(placement, ops)


# ---------------------------------------------------------------------------
# workload (workload.hpp:58-118)
# ---------------------------------------------------------------------------
def gen_routing_trace(shape: ModelShape, layer_lambda: float, prompt_lambda: float, initial_expert: int,
                      seed: int, prompts: int, tokens_per_prompt: int) -> np.ndarray:
    """gen_routing_trace(shape, make_calibration(shape, layer_lambda, prompt_lambda,
    initial_expert, seed), prompts, tokens) -> [P, m, T, k] int32."""
    out = np.empty((prompts, shape.num_moe_layers, tokens_per_prompt, shape.top_k), np.int32)
    check(lib.emoe_gen_routing_trace(shape.num_moe_layers, shape.experts_per_layer, shape.top_k, layer_lambda,
                                     prompt_lambda, initial_expert, seed, prompts, tokens_per_prompt, _p(out)))
    return out


def prompt_expert_sets(trace: np.ndarray, prompt: int):
    """(dominant_expert per layer, prompt_expert_sets) of one prompt (workload.cpp:350-377)."""
    import torch

    trace = _arr(trace, np.int32)
    P, m, T, k = trace.shape
    d = torch.from_numpy(trace).cuda()
    dom = np.zeros(m, np.int32)
    sets = np.full((m, k), -1, np.int32)
    sizes = np.zeros(m, np.int32)
    check(lib.emoe_prompt_expert_sets(C.c_void_p(d.data_ptr()), P, m, T, k, prompt, _p(dom), _p(sets), _p(sizes),
                                      None))
    return [int(v) for v in dom], [[int(e) for e in sets[l, : sizes[l]]] for l in range(m)]


def dominant_expert(trace: np.ndarray, prompt: int, layer: int) -> int:
    return prompt_expert_sets(trace, prompt)[0][layer]
