"""MoELayer: the predicted-residency MoE layer forward over the C ABI.

PyTorch is used only as plumbing here: device buffers, streams and pinned
host memory.  All compute runs in lib/libemoe.so (sm_100a kernels).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional, Sequence

import numpy as np
import torch

from ._lib import LayerConfig, Workspace, lib
from .moesim import check

_DT = {"bf16": (0, torch.bfloat16, 2), "fp32": (1, torch.float32, 4)}
_ACT = {"swiglu": 0, "relu": 1}
_WM = {"topk_softmax": 0, "full_softmax": 1}


def _stream_ptr(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class _CudaArray:
    """Zero-copy view of a raw device pointer for torch.as_tensor."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _view(ptr, shape, torch_dtype):
    if torch_dtype == torch.bfloat16:  # no bf16 typestr: view the bytes as int16 then reinterpret
        return torch.as_tensor(_CudaArray(ptr, shape, "<i2"), device="cuda").view(torch.bfloat16)
    ts = {torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8", torch.uint8: "|u1"}[torch_dtype]
    return torch.as_tensor(_CudaArray(ptr, shape, ts), device="cuda")


class MoELayer:
    def __init__(self, d_model: int, d_ff: int, num_experts: int, top_k: int, *, activation: str = "swiglu",
                 dtype: str = "bf16", weight_mode: str = "topk_softmax", num_slots: Optional[int] = None,
                 max_tokens: int = 65536, forced_miss: bool = False, gemm_cta_group: int = 0):
        self.d, self.f, self.E, self.k = d_model, d_ff, num_experts, top_k
        self.dtype_name = dtype
        self.code, self.torch_dtype, self.elem = _DT[dtype]
        self.activation = activation
        self.num_slots = num_slots or num_experts
        self.max_tokens = max_tokens
        cfg = LayerConfig(d_model, d_ff, num_experts, top_k, _ACT[activation], self.code, _WM[weight_mode],
                          self.num_slots, max_tokens, int(forced_miss), int(gemm_cta_group))
        h = C.c_void_p()
        check(lib.emoe_layer_create(C.byref(cfg), C.byref(h)))
        self.h = h
        w = Workspace()  # the layout constants are fixed at creation
        check(lib.emoe_layer_workspace(self.h, C.byref(w)))
        self.seg_pad = int(w.seg_pad)
        self.gemm_cta_group = int(w.gemm_cta_group)
        self.fp32_tensor_core = bool(w.fp32_tensor_core)

    def close(self):
        if getattr(self, "h", None):
            lib.emoe_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # -- weights ---------------------------------------------------------
    def _host(self, t: torch.Tensor, shape) -> torch.Tensor:
        t = t.detach().to("cpu", self.torch_dtype).contiguous()
        assert tuple(t.shape) == tuple(shape), (t.shape, shape)
        return t

    def set_gate(self, wg: torch.Tensor) -> None:
        wg = self._host(wg, (self.E, self.d))
        check(lib.emoe_layer_set_gate_host(self.h, C.c_void_p(wg.data_ptr())))

    def register_expert(self, e: int, w1: torch.Tensor, w3: Optional[torch.Tensor], w2: torch.Tensor) -> None:
        w1 = self._host(w1, (self.f, self.d))
        w2 = self._host(w2, (self.d, self.f))
        w3p = None
        if self.activation == "swiglu":
            w3 = self._host(w3, (self.f, self.d))
            w3p = C.c_void_p(w3.data_ptr())
        check(lib.emoe_layer_register_expert_host(self.h, e, C.c_void_p(w1.data_ptr()), w3p,
                                                  C.c_void_p(w2.data_ptr())))

    def register_expert_pinned(self, e: int, w1: torch.Tensor, w3: Optional[torch.Tensor], w2: torch.Tensor) -> None:
        """Use caller-owned pinned host tensors for expert e (no copy; kept alive here)."""
        for t in (w1, w2) + ((w3,) if w3 is not None else ()):
            assert t.device.type == "cpu" and t.is_pinned() and t.is_contiguous() and t.dtype == self.torch_dtype
        if not hasattr(self, "_pinned_refs"):
            self._pinned_refs = {}
        self._pinned_refs[e] = (w1, w3, w2)
        check(lib.emoe_layer_register_expert_pinned(self.h, e, C.c_void_p(w1.data_ptr()),
                                                    None if w3 is None else C.c_void_p(w3.data_ptr()),
                                                    C.c_void_p(w2.data_ptr())))

    def set_copy_stream(self, stream: Optional[torch.cuda.Stream]) -> None:
        """Share one copy stream across layers so loads run layer-sequentially (engine.cpp:431-440)."""
        self._copy_stream = stream
        check(lib.emoe_layer_set_copy_stream(self.h, None if stream is None else C.c_void_p(stream.cuda_stream)))

    def set_scores(self, scores: Optional[Sequence[float]], stream=None) -> None:
        """route_token fallback scores (the engine's last aggregate row of this
        layer, engine.cpp:424, :529-531); None = the empty score vector.
        Ordered on `stream` (default: the current stream) like a forward."""
        if scores is None or len(scores) == 0:
            check(lib.emoe_layer_set_scores(self.h, None, _stream_ptr(stream)))
            return
        s = np.ascontiguousarray(np.asarray(scores, np.float64))
        assert s.shape == (self.E,), f"scores must have {self.E} entries"
        check(lib.emoe_layer_set_scores(self.h, s.ctypes.data_as(C.c_void_p), _stream_ptr(stream)))

    def set_logits_mode(self, mode: str) -> None:
        """"replace": caller logits replace the gate (routing-driven parity mode,
        default); "add": the gate runs on x and the caller logits are added
        to its logits before top-k."""
        check(lib.emoe_layer_set_logits_mode(self.h, {"replace": 0, "add": 1}[mode]))

    def set_keep_logits(self, keep: bool) -> None:
        """Store the gate's fp32 logits in the workspace (default); False lets the
        fused tcgen05 gate (E >= 32) skip that store."""
        check(lib.emoe_layer_set_keep_logits(self.h, int(keep)))

    # -- residency (two-phase, engine.cpp:431-464) ------------------------
    def begin_load(self, evictions: Sequence[int], loads: Sequence[int], stream=None) -> None:
        ev = np.ascontiguousarray(np.asarray(list(evictions) or [0], np.int32))
        ld = np.ascontiguousarray(np.asarray(list(loads) or [0], np.int32))
        check(lib.emoe_layer_begin_load(self.h, ev.ctypes.data_as(C.c_void_p), len(evictions),
                                        ld.ctypes.data_as(C.c_void_p), len(loads), _stream_ptr(stream)))

    def poll_loads(self, blocking: bool = False, stream=None) -> bool:
        pending = C.c_int(0)
        check(lib.emoe_layer_poll_loads(self.h, int(blocking), _stream_ptr(stream), C.byref(pending)))
        return bool(pending.value)

    def residency(self) -> np.ndarray:
        out = np.zeros(self.E, np.uint8)
        check(lib.emoe_layer_residency(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def last_load_stats(self):
        b, ms = C.c_double(0), C.c_double(0)
        check(lib.emoe_layer_last_load_stats(self.h, C.byref(b), C.byref(ms)))
        return b.value, ms.value

    def load_initial(self, experts: Sequence[int]) -> None:
        """Make `experts` resident (blocking), evicting whatever else is resident."""
        cur = set(np.flatnonzero(self.residency()).tolist())
        want = set(int(e) for e in experts)
        self.begin_load(sorted(cur - want), sorted(want - cur))
        self.poll_loads(blocking=True)
        torch.cuda.synchronize()

    # -- forward -----------------------------------------------------------
    def forward(self, x: torch.Tensor, logits: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
        assert x.is_cuda and x.dtype == self.torch_dtype and x.is_contiguous() and x.shape[1] == self.d
        T = x.shape[0]
        if out is None:
            out = torch.empty_like(x)
        lp = None
        if logits is not None:
            assert logits.is_cuda and logits.dtype == torch.float32 and logits.shape == (T, self.E)
            lp = C.c_void_p(logits.contiguous().data_ptr())
        check(lib.emoe_moe_forward(self.h, C.c_void_p(x.data_ptr()), lp, C.c_void_p(out.data_ptr()), T,
                                   _stream_ptr(stream)))
        return out

    __call__ = forward

    def _check_host_pair(self, x_host: torch.Tensor, y_host: torch.Tensor) -> None:
        for name, t in (("x_host", x_host), ("y_host", y_host)):
            assert t.device.type == "cpu" and t.dtype == self.torch_dtype and t.is_contiguous(), \
                f"{name} must be a contiguous CPU {self.torch_dtype} tensor"
        assert x_host.dim() == 2 and x_host.shape[1] == self.d, f"x_host must be [T, {self.d}]"
        assert tuple(y_host.shape) == tuple(x_host.shape), "y_host must have x_host's shape"

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None) -> torch.Tensor:
        """End-to-end through host buffers: H2D of x, forward, D2H of y."""
        self._check_host_pair(x_host, y_host)
        check(lib.emoe_moe_forward_host(self.h, C.c_void_p(x_host.data_ptr()), C.c_void_p(y_host.data_ptr()),
                                        x_host.shape[0], _stream_ptr(stream)))
        return y_host

    def forward_host_async(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None) -> None:
        """Enqueue H2D + forward + D2H and return; call wait_host() before reading y_host.
        The queued copies hold raw pointers the torch allocator does not
        track, so every host pair is referenced here until wait_host()
        (deduplicated by address: a caller cycling through a few buffers adds
        nothing; more than 16 distinct pairs in flight waits first)."""
        self._check_host_pair(x_host, y_host)
        refs = self.__dict__.setdefault("_async_refs", {})
        key = (x_host.data_ptr(), y_host.data_ptr())
        if key not in refs and len(refs) >= 16:
            self.wait_host()
        check(lib.emoe_moe_forward_host_async(self.h, C.c_void_p(x_host.data_ptr()), C.c_void_p(y_host.data_ptr()),
                                              x_host.shape[0], _stream_ptr(stream)))
        refs[key] = (x_host, y_host)

    def wait_host(self) -> None:
        check(lib.emoe_layer_wait_host(self.h))
        self.__dict__.get("_async_refs", {}).clear()

    def route(self, x: Optional[torch.Tensor] = None, logits: Optional[torch.Tensor] = None, stream=None) -> None:
        T = x.shape[0] if x is not None else logits.shape[0]
        check(lib.emoe_route(self.h, C.c_void_p(x.data_ptr()) if x is not None else None,
                             C.c_void_p(logits.data_ptr()) if logits is not None else None, T, _stream_ptr(stream)))

    def gate_demand(self, stream=None) -> np.ndarray:
        """[E] int64: tokens of the last route/forward whose rank-0 gate choice is e
        (the on-demand baseline's demand map, engine.cpp:469-478)."""
        out = np.zeros(self.E, np.int64)
        check(lib.emoe_layer_gate_demand(self.h, out.ctypes.data_as(C.c_void_p), _stream_ptr(stream)))
        return out

    # -- stage entry points (expert parallelism) -----------------------------
    def set_route_residency(self, resident: Optional[Sequence[int]], stream=None) -> None:
        if resident is None:
            check(lib.emoe_layer_set_route_residency(self.h, None, _stream_ptr(stream)))
            return
        r = np.ascontiguousarray(np.asarray(resident, np.uint8))
        check(lib.emoe_layer_set_route_residency(self.h, r.ctypes.data_as(C.c_void_p), _stream_ptr(stream)))

    def route_permute(self, x: torch.Tensor, stream=None) -> None:
        check(lib.emoe_route_permute(self.h, C.c_void_p(x.data_ptr()), None, x.shape[0], _stream_ptr(stream)))

    def ffn_segments(self, x_rows: torch.Tensor, seg_offsets: torch.Tensor, seg_expert: torch.Tensor,
                     h_scratch: torch.Tensor, y_rows: torch.Tensor, stream=None) -> None:
        n = seg_expert.numel()
        check(lib.emoe_ffn_segments(self.h, C.c_void_p(x_rows.data_ptr()), x_rows.shape[0],
                                    C.c_void_p(seg_offsets.data_ptr()), C.c_void_p(seg_expert.data_ptr()), n,
                                    C.c_void_p(h_scratch.data_ptr()), C.c_void_p(y_rows.data_ptr()),
                                    _stream_ptr(stream)))

    def combine(self, y_rows: torch.Tensor, pos: torch.Tensor, served_w: torch.Tensor, out: torch.Tensor,
                stream=None) -> None:
        check(lib.emoe_combine(self.h, C.c_void_p(y_rows.data_ptr()), C.c_void_p(pos.data_ptr()),
                               C.c_void_p(served_w.data_ptr()), out.shape[0], C.c_void_p(out.data_ptr()),
                               _stream_ptr(stream)))

    def set_profiling(self, enable: bool = True) -> None:
        check(lib.emoe_layer_set_profiling(self.h, int(enable)))

    def stage_times(self) -> Dict[str, float]:
        """ms of the last forward's stages (needs set_profiling(True))."""
        ms = (C.c_float * 5)()
        check(lib.emoe_layer_stage_times(self.h, ms))
        return dict(zip(["route", "permute", "gemm1", "gemm2", "combine"], [float(v) for v in ms]))

    def stage_times_last(self) -> Dict[str, float]:
        """ms of the stages of the first profiled forward's events, not recycled:
        for a forward captured into a CUDA graph, read after each replay."""
        ms = (C.c_float * 5)()
        check(lib.emoe_layer_stage_times_last(self.h, ms))
        return dict(zip(["route", "permute", "gemm1", "gemm2", "combine"], [float(v) for v in ms]))

    def share_workspace(self, donor: "MoELayer") -> None:
        """Run on `donor`'s workspace (released here); see emoe_layer_share_workspace."""
        check(lib.emoe_layer_share_workspace(self.h, donor.h))
        self._ws_donor = donor  # keep the owner alive

    def workspace(self) -> Dict[str, torch.Tensor]:
        """Views of the last forward's intermediates (valid until the next call)."""
        w = Workspace()
        check(lib.emoe_layer_workspace(self.h, C.byref(w)))
        T, R, E, k = w.T, w.rows_cap, self.E, self.k
        self.seg_pad = int(w.seg_pad)
        self.gemm_cta_group = int(w.gemm_cta_group)
        self.fp32_tensor_core = bool(w.fp32_tensor_core)
        return {
            "logits": _view(w.logits, (T, E), torch.float32),
            "topk_idx": _view(w.topk_idx, (T, k), torch.int32),
            "route_expert": _view(w.route_expert, (T,), torch.int32),
            "route_rank": _view(w.route_rank, (T,), torch.int32),
            "route_hit": _view(w.route_hit, (T,), torch.uint8),
            "served_idx": _view(w.served_idx, (T, k), torch.int32),
            "served_w": _view(w.served_w, (T, k), torch.float32),
            "counts": _view(w.counts, (E,), torch.int32),
            "seg_offsets": _view(w.seg_offsets, (E + 1,), torch.int64),
            "pos": _view(w.pos, (T, k), torch.int32),
            "row_token": _view(w.row_token, (R,), torch.int32),
            "x_perm": _view(w.x_perm, (R, self.d), self.torch_dtype),
            "h": _view(w.h, (R, self.f), self.torch_dtype),
            "y_perm": _view(w.y_perm, (R, self.d), self.torch_dtype) if w.y_perm else None,
            "slot_of_expert": _view(w.slot_of_expert, (E,), torch.int32),
            "resident": _view(w.resident, (E,), torch.uint8),
        }
