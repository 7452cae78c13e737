"""B200-native predicted-residency MoE layer (eMoE, arXiv 2503.06823 hot path).

The compute lives in lib/libemoe.so (hand-written sm_100a CUDA behind the C
ABI in include/emoe.h); this package is the Python host mirror of the
reference ``moesim`` operator API plus the MoE layer handle.  Importing it
without the built library raises ImportError -- there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (fails loudly when the CUDA library is missing)
from .moesim import (CostModel, ExpectedTokens, LayerOps, LayerPrediction, LoadingPlan, LogicError, ModelShape,
                     Placement, Request, RouteResult, TaskProfile, TransitionModel, ValidationError, apply_plan,
                     apply_plan_layer, dominant_expert, expected_tokens, fit, gen_routing_trace, loading_targets,
                     plan_loading, predict_all_layers, predict_chained, predict_layerwise, predicted_frequencies,
                     prompt_expert_sets, route_token, route_tokens, select_experts)

__all__ = [
    "CostModel", "ExpectedTokens", "LayerOps", "LayerPrediction", "LoadingPlan", "LogicError", "ModelShape",
    "Placement", "Request", "RouteResult", "TaskProfile", "TransitionModel", "ValidationError", "apply_plan",
    "apply_plan_layer", "dominant_expert", "expected_tokens", "fit", "gen_routing_trace", "loading_targets",
    "plan_loading", "predict_all_layers", "predict_chained", "predict_layerwise", "predicted_frequencies",
    "prompt_expert_sets", "route_token", "route_tokens", "select_experts", "MoELayer",
]


def __getattr__(name):
    if name == "MoELayer":  # torch is only needed for the layer handle
        from .layer import MoELayer

        return MoELayer
    raise AttributeError(name)
