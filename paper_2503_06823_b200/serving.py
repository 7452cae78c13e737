"""The eMoE serving loop on the GPU: a stack of MoE layers under predicted
residency, periodic predictor invocations, task-aware skipping and expert
loads on a side stream overlapped with compute.

It restates the reference engine's predictor/load path with the real kernels
in place of the cost model (SURVEY.md §8a A7/A8, §8f "DES caller"):
  * invocation gating: the predictor fires when a prompt's arrival index is a
    multiple of the period p (engine.cpp:320-323);
  * invocation: predict from the previous prompt's per-layer expert sets,
    modulate by each task's fitted frequencies, Eq. 2 over the running and
    queued requests, loading_targets, plan_loading (engine.cpp:367-446) --
    one GPU call, emoe_invocation_host;
  * task-aware skip: when every request in the window belongs to a task that
    is insensitive on every layer, Eq. 2 is all zeros and loading_targets keeps
    the current residents (expert_store.cpp:140-157); the loop skips the
    invocation outright and counts it;
  * load schedule: per layer, evictions take effect at load start and loads at
    completion (engine.cpp:448-464); all layers share one copy stream, so
    layer l+1's copies start after layer l's (engine.cpp:431-440).  Compute
    never waits: each layer's forward polls its loads without blocking.
Routing follows the reference Markov trace (gate logits embedded from it,
the routing-driven mode of emoe_moe_forward).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Dict, List, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import moesim
from ._lib import lib
from .layer import MoELayer
from .moesim import _p, _sets_array, check


@dataclass
class TaskSpec:
    wo: float                 # expected output tokens (TaskProfile::wo)
    sensitivity: List[int]    # per layer, 1 = routing accuracy matters


@dataclass
class StreamConfig:
    m: int = 32
    E: int = 8
    k: int = 2
    L: int = 4
    d: int = 4096
    f: int = 14336
    activation: str = "swiglu"
    tokens_per_prompt: int = 8192
    period: int = 40
    mode: int = 0             # 0 = emoe_a (all layers), 1 = emoe_l (chained)
    task_aware: bool = True
    tasks: Dict[str, TaskSpec] = field(default_factory=dict)
    per_expert_seconds: float = 0.0


class MoEStack:
    """m MoE layers sharing pinned host experts, one copy stream, one predictor
    and (share_workspace) one activation workspace: the layers run one after
    another on one stream, so layer 0's routing/permutation/FFN buffers serve
    all of them (a Mixtral-shaped layer at 65,536 tokens needs ~6.5 GB)."""

    def __init__(self, cfg: StreamConfig, host_experts: Sequence, gate_weights: Sequence[torch.Tensor],
                 share_workspace: bool = True):
        self.cfg = cfg
        self.names = sorted(cfg.tasks)
        self.copy_stream = torch.cuda.Stream()
        self.layers: List[MoELayer] = []
        for l in range(cfg.m):
            layer = MoELayer(cfg.d, cfg.f, cfg.E, cfg.k, activation=cfg.activation, num_slots=cfg.L,
                             max_tokens=cfg.tokens_per_prompt)
            if share_workspace and self.layers:
                layer.share_workspace(self.layers[0])
            layer.set_gate(gate_weights[l])
            layer.set_copy_stream(self.copy_stream)
            for e, (w1, w3, w2) in enumerate(host_experts):
                layer.register_expert_pinned(e, w1, w3, w2)
            self.layers.append(layer)
        self.pred = moesim._Pred(cfg.m, cfg.E, cfg.k, len(self.names), 0.01)

    def close(self):
        for layer in reversed(self.layers):  # borrowers before the workspace owner
            layer.close()

    # -- predictor --------------------------------------------------------------
    def fit(self, trace_dev: torch.Tensor, task_ids: Sequence[str], group=None) -> None:
        """A6 over the training prompts (the engine fits once at setup, engine.cpp:249-258).
        With a process group of several ranks every rank tallies a shard and
        the tallies are merged (ep.fit_sharded): identical to one fit."""
        P, m, T, k = trace_dev.shape
        tid = torch.tensor([self.names.index(t) for t in task_ids], dtype=torch.int32, device=trace_dev.device)
        if group is not None and dist.get_world_size(group) > 1:
            from .ep import fit_sharded

            fit_sharded(self.pred.h, trace_dev, tid, group)
            return
        check(lib.emoe_hist_update(self.pred.h, C.c_void_p(trace_dev.data_ptr()), P, T, C.c_void_p(tid.data_ptr()),
                                   None))

    def invocation(self, prev_sets, requests: Sequence[tuple]):
        """engine invocation on the GPU -> per-layer (evictions, loads), aggregate, delta_e."""
        cfg = self.cfg
        m, E = cfg.m, cfg.E
        arr, sizes = _sets_array(prev_sets if cfg.mode == 0 else prev_sets[:1], cfg.k)
        wo = np.array([cfg.tasks[n].wo for n in self.names], np.float64)
        sens = np.array([cfg.tasks[n].sensitivity for n in self.names], np.int32).reshape(-1)
        has = np.ones(len(self.names), np.uint8)
        rt = np.array([self.names.index(t) for t, _ in requests], np.int32)
        rn = np.array([n for _, n in requests], np.int32)
        res = np.stack([layer.residency() for layer in self.layers]).astype(np.uint8)
        budgets = np.full(m, cfg.L, np.int32)
        agg = np.zeros((m, E))
        ev = np.full((m, E), -1, np.int32)
        ld = np.full((m, E), -1, np.int32)
        ne = np.zeros(m, np.int32)
        nl = np.zeros(m, np.int32)
        de = np.zeros(1)
        check(lib.emoe_invocation_host(self.pred.h, cfg.mode, _p(arr), _p(sizes), len(self.names), _p(wo), _p(sens),
                                       _p(has), len(rt), _p(rt), _p(rn), int(cfg.task_aware), _p(res), _p(budgets),
                                       cfg.per_expert_seconds, _p(agg), _p(ev), _p(ne), _p(ld), _p(nl), _p(de)))
        ops = [([int(e) for e in ev[l, : ne[l]]], [int(e) for e in ld[l, : nl[l]]]) for l in range(m)]
        return ops, agg, float(de[0])

    def set_scores(self, aggregate, stream=None) -> None:
        """The engine keeps the invocation's aggregate as every layer's route_token
        fallback scores (last_aggregate_, engine.cpp:424, :529-531); applied
        stream-ordered, so forwards already enqueued keep the previous scores."""
        self.scores = np.array(aggregate, np.float64)  # host copy (tests, reports)
        for l, layer in enumerate(self.layers):
            layer.set_scores(self.scores[l], stream)

    def apply(self, ops, stream=None) -> int:
        """Start the plan: per layer, evictions now, loads on the shared copy stream."""
        n = 0
        for layer, (evictions, loads) in zip(self.layers, ops):
            if evictions or loads:
                layer.begin_load(evictions, loads, stream)
                n += len(loads)
        return n

    def forward_prompt(self, x: torch.Tensor, logits: torch.Tensor, out: torch.Tensor, hits: torch.Tensor) -> None:
        """One prompt through every layer; routing-driven logits [m][T][E]."""
        for l, layer in enumerate(self.layers):
            layer.forward(x, logits=logits[l], out=out)
            hits[l] += layer.workspace()["route_hit"].sum()


def dynamic_targets(demand: np.ndarray, resident: np.ndarray, budget: int):
    """On-demand baseline for one layer (engine.cpp:469-497 dynamic_transfers):
    keep the `budget` experts with the largest demand (stable: ascending index on
    ties, experts without demand never kept); evict the other residents
    (ascending), load the kept non-residents (ascending).  -> (evictions, loads)"""
    ranked = sorted((e for e in range(len(demand)) if demand[e] > 0), key=lambda e: (-int(demand[e]), e))[:budget]
    needed = set(ranked)
    evictions = [int(e) for e in np.flatnonzero(resident) if e not in needed]
    loads = [e for e in sorted(needed) if not resident[e]]
    return evictions, loads


def run_stream(stack: MoEStack, trace: np.ndarray, trace_dev: torch.Tensor, prompt_tasks: Sequence[str],
               x: torch.Tensor, logits_of, first_prompt: int, n_prompts: int, residency: str = "predicted") -> dict:
    """Serve prompts first_prompt .. first_prompt+n_prompts-1 of the trace.
    logits_of(p) -> [m][T][E] fp32 device logits for prompt p.
    residency "predicted": the eMoE path above.  "dynamic": the reference's
    on-demand baseline -- no predictor; before each
    layer's forward the gate runs, the layer keeps the experts this prompt
    demands most and loads the missing ones synchronously on the critical path."""
    if residency not in ("predicted", "dynamic"):
        raise ValueError("residency must be 'predicted' or 'dynamic'")
    if residency == "dynamic":
        return _run_stream_dynamic(stack, x, logits_of, first_prompt, n_prompts)
    cfg = stack.cfg
    T = cfg.tokens_per_prompt
    sensitive = {n: any(cfg.tasks[n].sensitivity) for n in stack.names}
    out = torch.empty_like(x)
    hits = torch.zeros(cfg.m, dtype=torch.int64, device=x.device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = dict(invocations=0, skipped_invocations=0, planned_loads=0, invocation_host_ms=0.0, fired_at=[],
                 skipped_at=[], delta_e_planned_s=[])
    load_events = []
    torch.cuda.synchronize()
    ev0.record()
    for i in range(n_prompts):
        p = first_prompt + i
        if i % cfg.period == 0:  # predictor fires on this arrival (engine.cpp:320-323)
            window = list(range(p, min(p + cfg.period, first_prompt + n_prompts)))
            requests = [(prompt_tasks[q], T) for q in window]
            if cfg.task_aware and not any(sensitive[t] for t, _ in requests):
                # the reference would run the invocation and get an all-zero
                # aggregate (Eq. 2 is 0 on insensitive layers): residents kept
                # (loading_targets), and the fallback scores become zeros
                stack.set_scores(np.zeros((cfg.m, cfg.E)))
                stats["skipped_invocations"] += 1
                stats["skipped_at"].append(i)
            else:
                t0 = time.perf_counter()
                _, prev_sets = moesim_prompt_sets(trace_dev, p - 1)
                ops, agg, delta_e = stack.invocation(prev_sets, requests)
                stack.set_scores(agg)
                stats["delta_e_planned_s"].append(delta_e)  # plan_loading's estimate (expert_store.cpp:189-195)
                ls, le = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ls.record(stack.copy_stream)
                stats["planned_loads"] += stack.apply(ops)
                le.record(stack.copy_stream)
                load_events.append((ls, le))
                stats["invocation_host_ms"] += (time.perf_counter() - t0) * 1e3
                stats["invocations"] += 1
                stats["fired_at"].append(i)
        stack.forward_prompt(x, logits_of(p), out, hits)
    ev1.record()
    torch.cuda.synchronize()
    for layer in stack.layers:
        layer.poll_loads(blocking=True)
    ms = ev0.elapsed_time(ev1)
    load_ms = sum(a.elapsed_time(b) for a, b in load_events)
    # the measured copy time of each invocation's loads: the live delta_e the
    # engine's scheduler consumes (engine.cpp:333-334)
    stats["delta_e_measured_s"] = [a.elapsed_time(b) / 1e3 for a, b in load_events]
    expert_bytes = (3 if cfg.activation == "swiglu" else 2) * cfg.d * cfg.f * 2
    load_bytes = stats["planned_loads"] * expert_bytes
    stats.update(residency="predicted", ms=ms, tokens=n_prompts * T, tokens_per_s=n_prompts * T / (ms / 1e3),
                 hit_rate=float(hits.sum().item()) / (n_prompts * T * cfg.m), load_ms=load_ms, load_bytes=load_bytes,
                 load_gbs=load_bytes / max(load_ms, 1e-9) / 1e6,
                 load_overlap="compute never waits on loads: each layer polls its batch without blocking")
    return stats


def _run_stream_dynamic(stack: MoEStack, x: torch.Tensor, logits_of, first_prompt: int, n_prompts: int) -> dict:
    cfg = stack.cfg
    T = cfg.tokens_per_prompt
    out = torch.empty_like(x)
    hits = torch.zeros(cfg.m, dtype=torch.int64, device=x.device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    loads_total, load_ms = 0, 0.0
    torch.cuda.synchronize()
    ev0.record()
    for i in range(n_prompts):
        lg = logits_of(first_prompt + i)
        for l, layer in enumerate(stack.layers):
            layer.route(logits=lg[l])
            evictions, loads = dynamic_targets(layer.gate_demand(), layer.residency(), cfg.L)
            if evictions or loads:
                layer.begin_load(evictions, loads)
                layer.poll_loads(blocking=True)  # on the critical path (engine.cpp:498-501)
                loads_total += len(loads)
                load_ms += layer.last_load_stats()[1]
            layer.forward(x, logits=lg[l], out=out)
            hits[l] += layer.workspace()["route_hit"].sum()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    expert_bytes = (3 if cfg.activation == "swiglu" else 2) * cfg.d * cfg.f * 2
    load_bytes = loads_total * expert_bytes
    return dict(residency="dynamic", ms=ms, tokens=n_prompts * T, tokens_per_s=n_prompts * T / (ms / 1e3),
                hit_rate=float(hits.sum().item()) / (n_prompts * T * cfg.m), planned_loads=loads_total,
                load_ms=load_ms, load_bytes=load_bytes, load_gbs=load_bytes / max(load_ms, 1e-9) / 1e6,
                load_overlap="none: every layer waits for its on-demand loads before computing")


def profile_cost_model(stack: MoEStack, x: torch.Tensor, logits: torch.Tensor, sets, requests,
                       reps: int = 3) -> dict:
    """The reference CostModel (cost_model.hpp:10-21; scenario JSON "cost" object,
    scenario.cpp:252-260) measured on this GPU, i.e. the "profiled dE and c" the
    scheduler's Eq. 3 / Alg. 1 and the engine's iteration clock consume
    (engine.cpp:334, :545-546):
      per_token_cost        c = seconds per token through all m layers (no loads);
      hd_bandwidth          pinned host -> HBM expert copies on the copy stream;
      per_expert_transfer   fixed cost per expert copy beyond bytes / bandwidth;
      predictor_invocation_cost  one GPU invocation (predict .. plan_loading);
      contention_factor     compute slowdown while expert copies are in flight.
    logits: [m][T][E] routing-driven logits; sets/requests: an invocation's inputs.
    Leaves every layer's residency as it found it."""
    cfg = stack.cfg
    T = x.shape[0]
    out = torch.empty_like(x)
    hits = torch.zeros(cfg.m, dtype=torch.int64, device=x.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def stack_ms():
        stack.forward_prompt(x, logits, out, hits)  # warm
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            stack.forward_prompt(x, logits, out, hits)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    base_ms = stack_ms()
    # expert copies: swap one resident expert of layer 0 for a non-resident one and back
    layer = stack.layers[0]
    res = layer.residency()
    r_in, r_out = int(np.flatnonzero(res)[0]), int(np.flatnonzero(res == 0)[0])
    one = []
    for ev, ld in [([r_in], [r_out]), ([r_out], [r_in])] * reps:
        layer.begin_load(ev, ld)
        layer.poll_loads(blocking=True)
        one.append(layer.last_load_stats())
    # a batch of all L residents of layer 0 (swapped out and back) for the bandwidth
    resident = [int(e) for e in np.flatnonzero(res)]
    others = [int(e) for e in np.flatnonzero(res == 0)][: len(resident)]
    layer.begin_load(resident[: len(others)], others)
    layer.poll_loads(blocking=True)
    many = layer.last_load_stats()
    layer.begin_load(others, resident[: len(others)])
    layer.poll_loads(blocking=True)
    many_back = layer.last_load_stats()
    bw = (many[0] + many_back[0]) / ((many[1] + many_back[1]) / 1e3)
    one_s = float(np.median([ms for _, ms in one])) / 1e3
    setup = max(one_s - one[0][0] / bw, 1e-7)
    # contention: a few forwards of layer 1 alone, then the same while layer 0's
    # copies are in flight on the copy stream (the copies outlast them)
    contention = 1.0
    if cfg.m > 1:
        probe = stack.layers[1]
        n_fwd = 3
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def probe_ms(copying: bool):
            if copying:
                layer.begin_load(resident[: len(others)], others)
            e2.record()
            for _ in range(n_fwd):
                probe.forward(x, logits=logits[1], out=out)
            e3.record()
            torch.cuda.synchronize()
            if copying:
                layer.poll_loads(blocking=True)
                layer.begin_load(others, resident[: len(others)])
                layer.poll_loads(blocking=True)
            return e2.elapsed_time(e3)

        probe_ms(False)
        contention = max(1.0, probe_ms(True) / probe_ms(False))
    # one predictor invocation (host wall time, GPU kernels included)
    t0 = time.perf_counter()
    for _ in range(reps):
        stack.invocation(sets, requests)
    inv_s = (time.perf_counter() - t0) / reps
    return dict(per_token_cost=base_ms / 1e3 / T, per_expert_transfer=setup, hd_bandwidth=bw,
                predictor_invocation_cost=inv_s, contention_factor=contention)


def moesim_prompt_sets(trace_dev: torch.Tensor, prompt: int):
    """dominant experts and prompt_expert_sets of one prompt of a device trace."""
    P, m, T, k = trace_dev.shape
    dom = np.zeros(m, np.int32)
    sets = np.full((m, k), -1, np.int32)
    sizes = np.zeros(m, np.int32)
    check(lib.emoe_prompt_expert_sets(C.c_void_p(trace_dev.data_ptr()), P, m, T, k, prompt, _p(dom), _p(sets),
                                      _p(sizes), None))
    return dom.tolist(), [[int(e) for e in sets[l, : sizes[l]]] for l in range(m)]
