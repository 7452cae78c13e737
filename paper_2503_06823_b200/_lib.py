"""Loads the in-tree CUDA library (lib/libemoe.so) and declares its C ABI.

There is no fallback: if the library is missing or was built for another
architecture, importing the package raises.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_2503_06823_b200/csrc -j``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# EMOE_LIB_PATH: an alternative build of the same library (compile-time A/B variants)
LIB_PATH = Path(os.environ.get("EMOE_LIB_PATH") or Path(__file__).resolve().parent / "lib" / "libemoe.so")

if not LIB_PATH.exists():
    raise ImportError(
        f"emoe CUDA library not built: {LIB_PATH} is missing (run `make -C paper_2503_06823_b200/csrc -j`)")

lib = C.CDLL(str(LIB_PATH))

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
dbl = C.c_double


class LayerConfig(C.Structure):
    _fields_ = [("d_model", C.c_int), ("d_ff", C.c_int), ("num_experts", C.c_int), ("top_k", C.c_int),
                ("activation", C.c_int), ("dtype", C.c_int), ("weight_mode", C.c_int), ("num_slots", C.c_int),
                ("max_tokens", i64), ("forced_miss", C.c_int), ("gemm_cta_group", C.c_int)]


class Workspace(C.Structure):
    _fields_ = [("T", i64), ("rows_cap", i64), ("seg_pad", i64), ("gemm_cta_group", i64), ("logits", vp), ("topk_idx", vp), ("route_expert", vp),
                ("route_rank", vp), ("route_hit", vp), ("served_idx", vp), ("served_w", vp), ("counts", vp),
                ("seg_offsets", vp), ("pos", vp), ("row_token", vp), ("x_perm", vp), ("h", vp), ("y_perm", vp),
                ("slot_of_expert", vp), ("resident", vp), ("fp32_tensor_core", i64)]


def _decl(name, *argtypes):
    fn = getattr(lib, name)
    fn.argtypes = list(argtypes)
    fn.restype = C.c_int
    return fn


lib.emoe_last_error.restype = C.c_char_p
lib.emoe_last_error.argtypes = []
_decl("emoe_version")
_decl("emoe_route_tokens_host", vp, i64, C.c_int, vp, C.c_int, vp, vp, vp, vp)
_decl("emoe_layer_create", C.POINTER(LayerConfig), C.POINTER(vp))
_decl("emoe_layer_destroy", vp)
_decl("emoe_layer_set_gate_host", vp, vp)
_decl("emoe_layer_register_expert_host", vp, C.c_int, vp, vp, vp)
_decl("emoe_layer_set_scores_host", vp, vp)
_decl("emoe_layer_set_scores", vp, vp, vp)
_decl("emoe_layer_set_logits_mode", vp, C.c_int)
_decl("emoe_layer_set_keep_logits", vp, C.c_int)
_decl("emoe_layer_register_expert_pinned", vp, C.c_int, vp, vp, vp)
_decl("emoe_layer_set_copy_stream", vp, vp)
_decl("emoe_layer_begin_load", vp, vp, C.c_int, vp, C.c_int, vp)
_decl("emoe_layer_poll_loads", vp, C.c_int, vp, C.POINTER(C.c_int))
_decl("emoe_layer_residency", vp, vp)
_decl("emoe_layer_last_load_stats", vp, C.POINTER(dbl), C.POINTER(dbl))
_decl("emoe_moe_forward", vp, vp, vp, vp, i64, vp)
_decl("emoe_moe_forward_host", vp, vp, vp, i64, vp)
_decl("emoe_moe_forward_host_async", vp, vp, vp, i64, vp)
_decl("emoe_layer_wait_host", vp)
_decl("emoe_route", vp, vp, vp, i64, vp)
_decl("emoe_layer_gate_demand", vp, vp, vp)
_decl("emoe_layer_workspace", vp, C.POINTER(Workspace))
_decl("emoe_layer_share_workspace", vp, vp)
_decl("emoe_route_permute", vp, vp, vp, i64, vp)
_decl("emoe_layer_set_route_residency", vp, vp, vp)
_decl("emoe_ffn_segments", vp, vp, i64, vp, vp, C.c_int, vp, vp, vp)
_decl("emoe_combine", vp, vp, vp, vp, i64, vp, vp)
_decl("emoe_ep_create", vp, C.c_int, C.c_int, vp, i64, vp, C.POINTER(vp))
_decl("emoe_ep_ipc_handle", vp, vp)
_decl("emoe_ep_open_peers", vp, vp)
_decl("emoe_ep_forward", vp, vp, vp, vp, i64, vp)
_decl("emoe_ep_status", vp, vp, C.POINTER(C.c_int), C.POINTER(i64))
_decl("emoe_ep_stats", vp, vp, vp)
_decl("emoe_ep_layout", vp, vp, vp, vp, vp, vp)
_decl("emoe_ep_set_profiling", vp, C.c_int)
_decl("emoe_ep_stage_times", vp, vp)
_decl("emoe_ep_destroy", vp)
_decl("emoe_epx_create", vp, C.c_int, C.c_int, vp, i64, C.POINTER(vp))
_decl("emoe_epx_cap_rows", vp, C.POINTER(i64))
_decl("emoe_epx_route", vp, vp, vp, i64, vp)
_decl("emoe_epx_dispatch", vp, vp, vp, i64, vp, vp)
_decl("emoe_epx_ffn", vp, vp, vp, vp)
_decl("emoe_epx_combine", vp, vp, vp, i64, vp)
_decl("emoe_epx_status", vp, vp, C.POINTER(C.c_int), C.POINTER(i64))
_decl("emoe_epx_destroy", vp)
IPC_HANDLE_BYTES = 64
_decl("emoe_layer_set_profiling", vp, C.c_int)
_decl("emoe_layer_stage_times", vp, vp)
_decl("emoe_layer_stage_times_last", vp, vp)
lib.emoe_kernel_launches.restype = C.c_longlong
lib.emoe_kernel_launches.argtypes = []
_decl("emoe_predictor_create", C.c_int, C.c_int, C.c_int, C.c_int, dbl, C.POINTER(vp))
_decl("emoe_predictor_destroy", vp)
_decl("emoe_predictor_reset", vp)
_decl("emoe_predictor_break_chain", vp)
_decl("emoe_hist_update", vp, vp, C.c_int, C.c_int, vp, vp)
_decl("emoe_hist_update_host", vp, vp, C.c_int, C.c_int, vp)
_decl("emoe_predictor_counts_host", vp, vp, vp, vp)
_decl("emoe_predictor_set_counts_host", vp, vp, vp, vp)
_decl("emoe_predictor_count_size", vp, C.POINTER(C.c_int64))
_decl("emoe_predictor_counts_dev", vp, vp, vp)
_decl("emoe_predictor_set_counts_dev", vp, vp, vp)
_decl("emoe_prompt_expert_sets", vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp)
_decl("emoe_prompt_expert_sets_host", vp, C.c_int, C.c_int, C.c_int, vp, vp, vp)
_decl("emoe_predict_host", vp, C.c_int, vp, vp, C.c_int, vp, vp, vp)
_decl("emoe_predicted_frequencies_host", vp, C.c_int, vp)
_decl("emoe_expected_tokens_host", C.c_int, C.c_int, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp, C.c_int, vp)
_decl("emoe_select_experts_host", vp, C.c_int, C.c_int, vp, vp)
_decl("emoe_loading_targets_host", vp, C.c_int, C.c_int, vp, vp, vp, vp)
_decl("emoe_plan_loading_host", vp, vp, C.c_int, C.c_int, vp, vp, vp, dbl, vp, vp, vp, vp, vp, vp, vp)
_decl("emoe_invocation_host", vp, C.c_int, vp, vp, C.c_int, vp, vp, vp, C.c_int, vp, vp, C.c_int, vp, vp, dbl, vp,
      vp, vp, vp, vp, vp)
_decl("emoe_gen_routing_trace", C.c_int, C.c_int, C.c_int, dbl, dbl, C.c_int, C.c_uint64, C.c_int, C.c_int, vp)

# every symbol include/emoe.h declares (checked by tests/test_boundary.py)
EXPORTED = [
    "emoe_last_error", "emoe_version", "emoe_route_tokens_host", "emoe_layer_create", "emoe_layer_destroy",
    "emoe_layer_set_gate_host", "emoe_layer_register_expert_host", "emoe_layer_register_expert_pinned",
    "emoe_layer_set_copy_stream", "emoe_layer_set_scores_host", "emoe_layer_set_scores", "emoe_layer_set_logits_mode", "emoe_layer_set_keep_logits",
    "emoe_layer_begin_load", "emoe_layer_poll_loads", "emoe_layer_residency", "emoe_layer_last_load_stats",
    "emoe_moe_forward", "emoe_moe_forward_host", "emoe_moe_forward_host_async", "emoe_layer_wait_host", "emoe_route", "emoe_layer_gate_demand", "emoe_route_permute", "emoe_layer_set_route_residency",
    "emoe_ffn_segments", "emoe_combine", "emoe_ep_create", "emoe_ep_ipc_handle", "emoe_ep_open_peers",
    "emoe_ep_forward", "emoe_ep_status", "emoe_ep_stats", "emoe_ep_layout", "emoe_ep_set_profiling",
    "emoe_ep_stage_times", "emoe_ep_destroy", "emoe_epx_create", "emoe_epx_cap_rows", "emoe_epx_route",
    "emoe_epx_dispatch", "emoe_epx_ffn", "emoe_epx_combine", "emoe_epx_status", "emoe_epx_destroy", "emoe_layer_workspace", "emoe_layer_share_workspace", "emoe_layer_set_profiling",
    "emoe_layer_stage_times", "emoe_layer_stage_times_last", "emoe_kernel_launches", "emoe_predictor_create",
    "emoe_predictor_destroy", "emoe_predictor_reset", "emoe_predictor_break_chain", "emoe_hist_update", "emoe_hist_update_host", "emoe_predictor_counts_host",
    "emoe_predictor_set_counts_host", "emoe_predictor_count_size", "emoe_predictor_counts_dev",
    "emoe_predictor_set_counts_dev", "emoe_prompt_expert_sets", "emoe_prompt_expert_sets_host", "emoe_predict_host",
    "emoe_predicted_frequencies_host", "emoe_expected_tokens_host", "emoe_select_experts_host",
    "emoe_loading_targets_host", "emoe_plan_loading_host", "emoe_invocation_host", "emoe_gen_routing_trace",
]
