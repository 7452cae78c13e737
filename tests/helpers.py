"""Shared test helpers: synthetic layers, the oracle chain, tolerances.

Tolerances:
  integer outputs (routing indices, counts, offsets, permutation): bit-exact
  bf16 layer outputs: oracle mirrors the kernels' rounding points (H, Y, y
      rounded to bf16); norm-wise relative error <= 1e-3 and
      max|diff| / max|ref| <= 2^-7 (one bf16 ulp at the largest magnitude)
  fp32 layer outputs: norm-wise and max-abs/max|ref| relative error <= 1e-5
"""
from __future__ import annotations

import numpy as np
import torch

BF16_TOL = 1e-3
BF16_MAX_TOL = 2.0 ** -7
F32_TOL = 1e-5


def to_f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def make_weights(E, d, f, dtype, act, seed=1234):
    """x-independent weights: W_g ~ N(0,1/d), W1,W3 ~ N(0,1/d), W2 ~ N(0,1/f)."""
    g = torch.Generator().manual_seed(seed)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    wg = (torch.randn(E, d, generator=g) / d ** 0.5).to(td)
    experts = []
    for e in range(E):
        w1 = (torch.randn(f, d, generator=g) / d ** 0.5).to(td)
        w3 = (torch.randn(f, d, generator=g) / d ** 0.5).to(td) if act == "swiglu" else None
        w2 = (torch.randn(d, f, generator=g) / f ** 0.5).to(td)
        experts.append((w1, w3, w2))
    return wg, experts


def build_layer(E, d, f, k, dtype="bf16", act="swiglu", weight_mode="topk_softmax", slots=None, resident=None,
                max_tokens=4096, seed=1234, forced_miss=False, gemm_cta_group=0):
    from paper_2503_06823_b200 import MoELayer

    wg, experts = make_weights(E, d, f, dtype, act, seed)
    layer = MoELayer(d, f, E, k, activation=act, dtype=dtype, weight_mode=weight_mode, num_slots=slots or E,
                     max_tokens=max_tokens, forced_miss=forced_miss, gemm_cta_group=gemm_cta_group)
    layer.set_gate(wg)
    for e, (w1, w3, w2) in enumerate(experts):
        layer.register_expert(e, w1, w3, w2)
    if resident is None:
        resident = list(range(slots or E))
    layer.load_initial(resident)
    return layer, wg, experts


def rel_errors(got: np.ndarray, ref: np.ndarray):
    d = got.astype(np.float64) - ref.astype(np.float64)
    norm = float(np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-30))
    mx = float(np.abs(d).max() / max(np.abs(ref).max(), 1e-30)) if d.size else 0.0
    return norm, mx


def bf16_ulp(v: np.ndarray) -> np.ndarray:
    a = np.abs(v).astype(np.float64)
    e = np.floor(np.log2(np.maximum(a, 1e-38)))
    return np.exp2(e - 7)


def assert_bf16_close(got, ref, what=""):
    """bf16 outputs: norm-wise relative error <= 1e-3, and the largest element
    error within one bf16 ulp at the output's largest magnitude (2^-7 of
    max|ref|): a rounding flip of an intermediate (H or Y) can move an output by
    up to one ulp of that intermediate on top of the output's own rounding."""
    norm, mx = rel_errors(got, ref)
    assert norm <= BF16_TOL, f"{what}: norm-wise relative error {norm:.3e} > {BF16_TOL}"
    assert mx <= BF16_MAX_TOL, f"{what}: max-abs error {mx:.3e} of max|ref| > {BF16_MAX_TOL}"
    return norm, mx


def assert_f32_close(got, ref, what=""):
    norm, mx = rel_errors(got, ref)
    assert norm <= F32_TOL and mx <= F32_TOL, f"{what}: fp32 errors norm {norm:.3e} max {mx:.3e} > {F32_TOL}"
    return norm, mx


def trace_logits(choices: np.ndarray, E: int, seed: int = 99) -> np.ndarray:
    """Embed ranked gate choices as logits: logit[c_r] = 8 - r, others uniform in [-4, 4)
    (exact in bf16/fp32, tie-free, so top-k(logits) == choices)."""
    T, k = choices.shape
    rng = np.random.default_rng(seed)
    lg = rng.uniform(-4.0, 4.0, size=(T, E)).astype(np.float32)
    lg = np.round(lg * 64) / 64  # exactly representable
    for r in range(k):
        lg[np.arange(T), choices[:, r]] = 8.0 - r
    return lg.astype(np.float32)
