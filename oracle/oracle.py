"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two libraries, both built by oracle/Makefile:

* ``Port`` -> oracle/lib/libemoe_oracle.so, our plain-C restatement
  (oracle/emoe_oracle.c) of the reference algorithm.
* ``Ref``  -> oracle/_ref/libmoesim_ref.so, the UNMODIFIED reference sources
  (/root/reference/proj/core/src/*.cpp) plus a flat C shim (oracle/ref_capi.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "lib" / "libemoe_oracle.so"
REF_SO = HERE / "_ref" / "libmoesim_ref.so"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class ValidationError(ValueError):
    """Mirror of moesim::ValidationError (types.hpp:11-14): return code 2."""


class LogicError(RuntimeError):
    """Mirror of std::logic_error raised by the reference: return code 3."""


def _check(rc: int, err_fn) -> None:
    if rc == 0:
        return
    msg = err_fn().decode()
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise LogicError(msg)
    raise RuntimeError(msg)


def _a(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


def _names(names):
    arr = (C.c_char_p * max(1, len(names)))()
    for i, n in enumerate(names):
        arr[i] = n.encode()
    return arr


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


class Port:
    """Our C restatement (oracle/emoe_oracle.c)."""

    def __init__(self, path: Path = PORT_SO):
        if not Path(path).exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle port`")
        L = self.lib = C.CDLL(str(path))
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_get_threads.restype = C.c_int
        L.oracle_route_tokens.argtypes = [_i32p, C.c_int64, C.c_int, _u8p, C.c_int, C.c_void_p, C.c_int,
                                          _i32p, _i32p, _u8p]
        L.oracle_gate_route.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p,
                                        C.c_int, C.c_int, _i32p, _f32p, _i32p, _i32p, _u8p, _i32p, _f32p,
                                        _i32p]
        L.oracle_gate_logits_f32.argtypes = [_f32p, _f32p, C.c_int64, C.c_int, C.c_int, _f32p]
        L.oracle_permute.argtypes = [_i32p, C.c_int64, C.c_int, C.c_int, C.c_int, _i32p, _i64p, _i64p,
                                     _i32p, C.c_int64, C.POINTER(C.c_int64)]
        L.oracle_expert_ffn.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, _f32p, C.c_void_p, _f32p,
                                        C.c_int, C.c_int, _f32p, C.c_int]
        L.oracle_combine.argtypes = [_f32p, C.c_int, _i64p, _f32p, C.c_int64, C.c_int, C.c_int, _f32p]
        L.oracle_fit.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                 C.POINTER(C.c_int32), _f64p, _f64p, _f64p]
        L.oracle_dominant_expert.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.oracle_prompt_expert_sets.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                                _i32p]
        L.oracle_predict.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f64p, C.c_int, _i32p,
                                     _i32p, C.c_int, _f64p, _i32p, _i32p]
        L.oracle_predicted_frequencies.argtypes = [C.c_int, C.c_int, C.c_int, _f64p, C.c_double, C.c_int,
                                                   _f64p]
        L.oracle_expected_tokens.argtypes = [C.c_int, C.c_int, C.c_int, _f64p, _i32p, _u8p, C.c_int, _i32p,
                                             _i32p, _u8p, _f64p, C.c_int, _f64p]
        L.oracle_select_experts.argtypes = [_f64p, C.c_int, C.c_int, _i32p, _i32p]
        L.oracle_loading_targets.argtypes = [_f64p, C.c_int, C.c_int, _u8p, _i32p, _i32p, _i32p]
        L.oracle_plan_loading.argtypes = [_u8p, _i32p, C.c_int, C.c_int, _i32p, _i32p, _f64p, C.c_double,
                                          _i32p, _i32p, _i32p, _i32p, _f64p, C.POINTER(C.c_double),
                                          C.POINTER(C.c_int32)]
        L.oracle_invocation_aggregate.argtypes = [C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p, _i32p,
                                                  _u8p, C.c_int, _i32p, _i32p, C.c_int, _f64p]

    def _chk(self, rc):
        _check(rc, self.lib.oracle_last_error)

    def set_threads(self, n: int) -> None:
        self.lib.oracle_set_threads(int(n))

    def threads(self) -> int:
        return int(self.lib.oracle_get_threads())

    # ---- A2 ----
    def route_tokens(self, choices, resident, scores=None):
        choices = _a(choices, np.int32)
        T, k = choices.shape
        resident = _a(resident, np.uint8)
        E = resident.shape[0]
        sc = None if scores is None or len(scores) == 0 else _a(scores, np.float64)
        ex = np.empty(T, np.int32)
        rk = np.empty(T, np.int32)
        hit = np.empty(T, np.uint8)
        self._chk(self.lib.oracle_route_tokens(choices, T, k, resident, E,
                                               None if sc is None else sc.ctypes.data, 0 if sc is None else E,
                                               ex, rk, hit))
        return ex, rk, hit

    # ---- A1 + A2 ----
    def gate_route(self, logits, k, weight_mode, resident, scores=None, forced_miss=False):
        logits = _a(logits, np.float32)
        T, E = logits.shape
        resident = _a(resident, np.uint8)
        sc = None if scores is None or len(scores) == 0 else _a(scores, np.float64)
        out = dict(topk_idx=np.empty((T, k), np.int32), topk_logit=np.empty((T, k), np.float32),
                   route_expert=np.empty(T, np.int32), route_rank=np.empty(T, np.int32),
                   route_hit=np.empty(T, np.uint8), served_idx=np.empty((T, k), np.int32),
                   served_w=np.empty((T, k), np.float32), counts=np.empty(E, np.int32))
        self._chk(self.lib.oracle_gate_route(logits, T, E, k, weight_mode, resident,
                                             None if sc is None else sc.ctypes.data, 0 if sc is None else E,
                                             int(forced_miss), out["topk_idx"], out["topk_logit"],
                                             out["route_expert"], out["route_rank"], out["route_hit"],
                                             out["served_idx"], out["served_w"], out["counts"]))
        return out

    def gate_logits(self, x, wg):
        x = _a(x, np.float32)
        wg = _a(wg, np.float32)
        T, d = x.shape
        E = wg.shape[0]
        out = np.empty((T, E), np.float32)
        self.lib.oracle_gate_logits_f32(x, wg, T, d, E, out)
        return out

    # ---- A3 ----
    def permute(self, served_idx, E, pad):
        served_idx = _a(served_idx, np.int32)
        T, k = served_idx.shape
        cap = T * k + E * pad
        counts = np.empty(E, np.int32)
        offsets = np.empty(E + 1, np.int64)
        pos = np.empty((T, k), np.int64)
        src = np.empty(cap, np.int32)
        used = C.c_int64(0)
        self._chk(self.lib.oracle_permute(served_idx, T, k, E, pad, counts, offsets, pos, src, cap,
                                          C.byref(used)))
        return counts, offsets, pos, src[: used.value]

    # ---- A4 / A5 ----
    def expert_ffn(self, x, w1, w3, w2, act, round_bf16, threads=0):
        x = _a(x, np.float32)
        rows, d = x.shape
        f = w1.shape[0]
        w1 = _a(w1, np.float32)
        w2 = _a(w2, np.float32)
        w3c = None if w3 is None else _a(w3, np.float32)
        y = np.empty((rows, d), np.float32)
        self.lib.oracle_expert_ffn(x, rows, d, f, w1, None if w3c is None else w3c.ctypes.data, w2, act,
                                   int(round_bf16), y, threads)
        return y

    def combine(self, Y, pos, served_w, round_bf16):
        Y = _a(Y, np.float32)
        pos = _a(pos, np.int64)
        served_w = _a(served_w, np.float32)
        T, k = pos.shape
        d = Y.shape[1]
        y = np.empty((T, d), np.float32)
        self.lib.oracle_combine(Y, d, pos, served_w, T, k, int(round_bf16), y)
        return y

    # ---- A6 ----
    def fit(self, trace, task_ids=None, n_tasks=0, num_experts=0):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        E = num_experts if num_experts > 0 else int(trace.max()) + 1 if trace.size else 0
        Eo = C.c_int32(0)
        lc = np.zeros((max(m - 1, 0), max(E, 1), max(E, 1)), np.float64)
        pc = np.zeros((m, max(E, 1), max(E, 1)), np.float64)
        tc = np.zeros((max(n_tasks, 1), m, max(E, 1)), np.float64)
        tid = None if task_ids is None else _a(task_ids, np.int32)
        self._chk(self.lib.oracle_fit(trace, P, m, T, k, None if tid is None else tid.ctypes.data, n_tasks,
                                      num_experts, C.byref(Eo), lc, pc, tc))
        return dict(E=Eo.value, layer_counts=lc, prompt_counts=pc, task_counts=tc[:n_tasks])

    def dominant_expert(self, trace, prompt, layer):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        return int(self.lib.oracle_dominant_expert(trace, P, m, T, k, prompt, layer))

    def prompt_expert_sets(self, trace, prompt):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        sets = np.empty((m, k), np.int32)
        sizes = np.empty(m, np.int32)
        self._chk(self.lib.oracle_prompt_expert_sets(trace, P, m, T, k, prompt, sets, sizes))
        return sets, sizes

    # ---- A7 ----
    def predict(self, model, mode, prev_sets, prev_sizes, layer=0, k=None):
        m, E = model["prompt_counts"].shape[:2]
        k = k or model.get("k", prev_sets.shape[1])
        scores = np.zeros((m, E), np.float64)
        experts = np.full((m, k), -1, np.int32)
        n = np.zeros(m, np.int32)
        lc = model["layer_counts"] if model["layer_counts"].size else np.zeros((1, E, E))
        self._chk(self.lib.oracle_predict(m, E, k, model["smoothing"], _a(lc, np.float64),
                                          _a(model["prompt_counts"], np.float64), mode,
                                          _a(prev_sets, np.int32), _a(prev_sizes, np.int32), layer, scores,
                                          experts, n))
        return scores, experts, n

    def predicted_frequencies(self, task_counts, smoothing, task):
        n_tasks, m, E = task_counts.shape
        out = np.empty((m, E), np.float64)
        self._chk(self.lib.oracle_predicted_frequencies(m, E, n_tasks, _a(task_counts, np.float64), smoothing,
                                                        task, out))
        return out

    def expected_tokens(self, m, E, wo, sensitivity, has_sens, req_task, req_tokens, freq_present, freqs,
                        task_aware=True):
        n_tasks = len(wo)
        agg = np.empty((m, E), np.float64)
        self._chk(self.lib.oracle_expected_tokens(
            m, E, n_tasks, _a(wo, np.float64), _a(sensitivity, np.int32).reshape(-1), _a(has_sens, np.uint8),
            len(req_task), _a(req_task, np.int32), _a(req_tokens, np.int32), _a(freq_present, np.uint8),
            _a(freqs, np.float64).reshape(-1), int(task_aware), agg))
        return agg

    def select_experts(self, aggregate, budgets):
        aggregate = _a(aggregate, np.float64)
        m, E = aggregate.shape
        out = np.full((m, E), -1, np.int32)
        self._chk(self.lib.oracle_select_experts(aggregate, m, E, _a(budgets, np.int32), out))
        return [list(out[l, : budgets[l]]) for l in range(m)]

    def loading_targets(self, aggregate, resident, budgets):
        aggregate = _a(aggregate, np.float64)
        m, E = aggregate.shape
        out = np.full((m, E), -1, np.int32)
        sizes = np.empty(m, np.int32)
        self._chk(self.lib.oracle_loading_targets(aggregate, m, E, _a(resident, np.uint8).reshape(-1),
                                                  _a(budgets, np.int32), out, sizes))
        return [list(out[l, : sizes[l]]) for l in range(m)]

    def plan_loading(self, resident, budgets, targets, aggregate, per_expert_seconds):
        aggregate = _a(aggregate, np.float64)
        m, E = aggregate.shape
        tg = np.full((m, E), -1, np.int32)
        sizes = np.array([len(t) for t in targets], np.int32)
        for l, t in enumerate(targets):
            tg[l, : len(t)] = t
        ev = np.full((m, E), -1, np.int32)
        ld = np.full((m, E), -1, np.int32)
        ne = np.empty(m, np.int32)
        nl = np.empty(m, np.int32)
        dur = np.empty(m, np.float64)
        de = C.c_double(0)
        tl = C.c_int32(0)
        self._chk(self.lib.oracle_plan_loading(_a(resident, np.uint8).reshape(-1), _a(budgets, np.int32), m, E,
                                               tg, sizes, aggregate, per_expert_seconds, ev, ne, ld, nl, dur,
                                               C.byref(de), C.byref(tl)))
        return dict(evictions=[list(ev[l, : ne[l]]) for l in range(m)],
                    loads=[list(ld[l, : nl[l]]) for l in range(m)], duration=dur, delta_e=de.value,
                    total_loads=tl.value)

    def invocation_aggregate(self, pred_scores, fitted, wo, sensitivity, has_sens, req_task, req_tokens,
                             task_aware=True):
        pred_scores = _a(pred_scores, np.float64)
        m, E = pred_scores.shape
        agg = np.empty((m, E), np.float64)
        self._chk(self.lib.oracle_invocation_aggregate(
            m, E, len(wo), pred_scores, _a(fitted, np.float64).reshape(-1), _a(wo, np.float64),
            _a(sensitivity, np.int32).reshape(-1), _a(has_sens, np.uint8), len(req_task),
            _a(req_task, np.int32), _a(req_tokens, np.int32), int(task_aware), agg))
        return agg


class Ref:
    """The unmodified reference built here (oracle/_ref/libmoesim_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not Path(path).exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_route_tokens.argtypes = [_i32p, C.c_int64, C.c_int, _u8p, C.c_int, C.c_void_p, C.c_int, _i32p,
                                       _i32p, _u8p]
        L.ref_time_route_tokens.argtypes = [_i32p, C.c_int64, C.c_int, _u8p, C.c_int, C.c_void_p, C.c_int,
                                            C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.ref_fit.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_double,
                              C.c_int, C.POINTER(C.c_int32), _f64p, _f64p, _f64p, C.POINTER(C.c_int32)]
        L.ref_time_fit.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_double)]
        L.ref_prompt_expert_sets.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _i32p,
                                             _i32p]
        L.ref_predict.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f64p, C.c_int, _i32p, _i32p,
                                  C.c_int, _f64p, _i32p, _i32p]
        L.ref_predicted_frequencies.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, _f64p, C.c_double,
                                                C.c_char_p, _f64p]
        L.ref_expected_tokens.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, _f64p, _i32p, _u8p, C.c_int,
                                          _i32p, _i32p, C.c_int, _i32p, _i32p, C.c_int, C.c_void_p, _f64p,
                                          C.c_int, _f64p]
        L.ref_select_experts.argtypes = [_f64p, C.c_int, C.c_int, _i32p, _i32p]
        L.ref_loading_targets.argtypes = [_f64p, C.c_int, C.c_int, _u8p, _i32p, _i32p, _i32p]
        L.ref_plan_loading.argtypes = [_u8p, _i32p, C.c_int, C.c_int, _i32p, _i32p, _f64p, C.c_double,
                                       C.c_double, C.c_uint64, _i32p, _i32p, _i32p, _i32p, _f64p,
                                       C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.ref_gen_routing_trace.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                            C.c_uint64, C.c_int, C.c_int, _i32p]
        L.ref_save_trace.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p]
        L.ref_fit_and_save_model.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_double, C.c_int, C.c_char_p]
        L.ref_rng_uniform.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.ref_rng_normal.argtypes = [C.c_uint64, C.c_int64, _f64p]

    def _chk(self, rc):
        _check(rc, self.lib.ref_last_error)

    def route_tokens(self, choices, resident, scores=None):
        choices = _a(choices, np.int32)
        T, k = choices.shape
        resident = _a(resident, np.uint8)
        E = resident.shape[0]
        sc = None if scores is None or len(scores) == 0 else _a(scores, np.float64)
        ex = np.empty(T, np.int32)
        rk = np.empty(T, np.int32)
        hit = np.empty(T, np.uint8)
        self._chk(self.lib.ref_route_tokens(choices, T, k, resident, E, None if sc is None else sc.ctypes.data,
                                            0 if sc is None else E, ex, rk, hit))
        return ex, rk, hit

    def time_route_tokens(self, choices, resident, scores=None, reps=3):
        choices = _a(choices, np.int32)
        T, k = choices.shape
        resident = _a(resident, np.uint8)
        sc = None if scores is None or len(scores) == 0 else _a(scores, np.float64)
        ns = C.c_double(0)
        hits = C.c_int64(0)
        self._chk(self.lib.ref_time_route_tokens(choices, T, k, resident, resident.shape[0],
                                                 None if sc is None else sc.ctypes.data, 0 if sc is None else
                                                 resident.shape[0], reps, C.byref(ns), C.byref(hits)))
        return ns.value, hits.value

    def fit(self, trace, task_ids=None, task_names=(), smoothing=0.01, num_experts=0):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        E = num_experts if num_experts > 0 else (int(trace.max()) + 1 if trace.size else 1)
        lc = np.zeros((max(m - 1, 0), E, E), np.float64)
        pc = np.zeros((m, E, E), np.float64)
        tc = np.zeros((max(len(task_names), 1), m, E), np.float64)
        Eo = C.c_int32(0)
        nt = C.c_int32(0)
        names = _names(task_names)
        tid = None if task_ids is None else _a(task_ids, np.int32)
        self._chk(self.lib.ref_fit(trace, P, m, T, k, None if tid is None else tid.ctypes.data,
                                   C.cast(names, C.c_void_p), smoothing, num_experts, C.byref(Eo),
                                   lc if lc.size else np.zeros(1), pc, tc, C.byref(nt)))
        return dict(E=Eo.value, layer_counts=lc, prompt_counts=pc, task_counts=tc[: nt.value], smoothing=smoothing)

    def time_fit(self, trace, num_experts, reps=3):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        ns = C.c_double(0)
        self._chk(self.lib.ref_time_fit(trace, P, m, T, k, num_experts, reps, C.byref(ns)))
        return ns.value

    def prompt_expert_sets(self, trace, prompt):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        dom = np.empty(m, np.int32)
        sets = np.empty((m, k), np.int32)
        sizes = np.empty(m, np.int32)
        self._chk(self.lib.ref_prompt_expert_sets(trace, P, m, T, k, prompt, dom, sets, sizes))
        return dom, sets, sizes

    def predict(self, model, mode, prev_sets, prev_sizes, layer=0, k=None):
        m, E = model["prompt_counts"].shape[:2]
        k = k or prev_sets.shape[1]
        scores = np.zeros((m, E), np.float64)
        experts = np.full((m, k), -1, np.int32)
        n = np.zeros(m, np.int32)
        lc = model["layer_counts"] if model["layer_counts"].size else np.zeros((1, E, E))
        self._chk(self.lib.ref_predict(m, E, k, model["smoothing"], _a(lc, np.float64),
                                       _a(model["prompt_counts"], np.float64), mode, _a(prev_sets, np.int32),
                                       _a(prev_sizes, np.int32), layer, scores, experts, n))
        return scores, experts, n

    def predicted_frequencies(self, task_counts, task_names, smoothing, task):
        n_tasks, m, E = task_counts.shape
        out = np.empty((m, E), np.float64)
        names = _names(task_names)
        self._chk(self.lib.ref_predicted_frequencies(m, E, n_tasks, C.cast(names, C.c_void_p),
                                                     _a(task_counts, np.float64), smoothing, task.encode(), out))
        return out

    def expected_tokens(self, m, E, task_names, wo, sensitivity, has_sens, running, incoming, freq_names,
                        freqs, task_aware=True):
        """running / incoming: lists of (task index, input tokens)."""
        agg = np.empty((m, E), np.float64)
        rt = _a([r[0] for r in running] or [0], np.int32)
        rn = _a([r[1] for r in running] or [0], np.int32)
        it = _a([r[0] for r in incoming] or [0], np.int32)
        inn = _a([r[1] for r in incoming] or [0], np.int32)
        pn = _names(task_names)
        fn = _names(freq_names)
        fr = _a(freqs, np.float64).reshape(-1) if len(freq_names) else np.zeros(1)
        self._chk(self.lib.ref_expected_tokens(
            m, E, len(task_names), C.cast(pn, C.c_void_p), _a(wo, np.float64), _a(sensitivity, np.int32).reshape(-1),
            _a(has_sens, np.uint8), len(running), rt, rn, len(incoming), it, inn, len(freq_names),
            C.cast(fn, C.c_void_p), fr, int(task_aware), agg))
        return agg

    def select_experts(self, aggregate, budgets):
        aggregate = _a(aggregate, np.float64)
        m, E = aggregate.shape
        out = np.full((m, E), -1, np.int32)
        self._chk(self.lib.ref_select_experts(aggregate, m, E, _a(budgets, np.int32), out))
        return [list(out[l, : budgets[l]]) for l in range(m)]

    def loading_targets(self, aggregate, resident, budgets):
        aggregate = _a(aggregate, np.float64)
        m, E = aggregate.shape
        out = np.full((m, E), -1, np.int32)
        sizes = np.empty(m, np.int32)
        self._chk(self.lib.ref_loading_targets(aggregate, m, E, _a(resident, np.uint8).reshape(-1),
                                               _a(budgets, np.int32), out, sizes))
        return [list(out[l, : sizes[l]]) for l in range(m)]

    def plan_loading(self, resident, budgets, targets, aggregate, per_expert, hd_bandwidth, expert_bytes):
        aggregate = _a(aggregate, np.float64)
        m, E = aggregate.shape
        tg = np.full((m, E), -1, np.int32)
        sizes = np.array([len(t) for t in targets], np.int32)
        for l, t in enumerate(targets):
            tg[l, : len(t)] = t
        ev = np.full((m, E), -1, np.int32)
        ld = np.full((m, E), -1, np.int32)
        ne = np.empty(m, np.int32)
        nl = np.empty(m, np.int32)
        dur = np.empty(m, np.float64)
        de = C.c_double(0)
        tl = C.c_int32(0)
        self._chk(self.lib.ref_plan_loading(_a(resident, np.uint8).reshape(-1), _a(budgets, np.int32), m, E, tg,
                                            sizes, aggregate, per_expert, hd_bandwidth, expert_bytes, ev, ne, ld,
                                            nl, dur, C.byref(de), C.byref(tl)))
        return dict(evictions=[list(ev[l, : ne[l]]) for l in range(m)],
                    loads=[list(ld[l, : nl[l]]) for l in range(m)], duration=dur, delta_e=de.value,
                    total_loads=tl.value)

    def gen_routing_trace(self, m, E, k, layer_lambda, prompt_lambda, initial_expert, seed, P, T):
        out = np.empty((P, m, T, k), np.int32)
        self._chk(self.lib.ref_gen_routing_trace(m, E, k, layer_lambda, prompt_lambda, initial_expert, seed, P, T,
                                                 out))
        return out

    def save_trace(self, trace, path):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        self._chk(self.lib.ref_save_trace(trace, P, m, T, k, str(path).encode()))

    def fit_and_save_model(self, trace, task_ids, task_names, smoothing, num_experts, path):
        trace = _a(trace, np.int32)
        P, m, T, k = trace.shape
        names = _names(task_names)
        tid = None if task_ids is None else _a(task_ids, np.int32)
        self._chk(self.lib.ref_fit_and_save_model(trace, P, m, T, k, None if tid is None else tid.ctypes.data,
                                                  C.cast(names, C.c_void_p), smoothing, num_experts,
                                                  str(path).encode()))

    def rng_uniform(self, seed, n):
        out = np.empty(n, np.float64)
        self._chk(self.lib.ref_rng_uniform(seed, n, out))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n, np.float64)
        self._chk(self.lib.ref_rng_normal(seed, n, out))
        return out


def have_ref() -> bool:
    return REF_SO.exists()


def have_port() -> bool:
    return PORT_SO.exists()
