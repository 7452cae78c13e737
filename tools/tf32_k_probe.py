"""Config-1-shaped 3xTF32 GEMMs (E=8 top-2, 4 resident, T=512, f=3584, SwiGLU,
fp32) vs d_model: separates a per-tile fixed cost from the per-k-block cost
(the method that found the tile-decode stall of the bf16 short-K GEMM)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from helpers import build_layer, trace_logits  # noqa: E402

T, E, f = int(sys.argv[1]) if len(sys.argv) > 1 else 512, 8, 3584
resident = [1, 2, 3, 4]
rng = np.random.default_rng(0)
choices = np.stack([rng.choice(E, 2, replace=False) for _ in range(T)]).astype(np.int32)
for d in (512, 1024, 2048, 4096):
    layer, _, _ = build_layer(E, d, f, 2, "fp32", "swiglu", "topk_softmax", 4, resident, max_tokens=T)
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(1)).cuda()
    lg = torch.from_numpy(trace_logits(choices, E)).cuda()
    for _ in range(3):
        layer.forward(x, logits=lg)
    torch.cuda.synchronize()
    layer.set_profiling(True)
    for _ in range(10):
        layer.forward(x, logits=lg)
    torch.cuda.synchronize()
    st = layer.stage_times()
    S = int(layer.workspace()["counts"].sum().item())
    print(f"T={T} d={d:5d} S={S}  gemm1 {st['gemm1'] * 1e3:7.1f} us ({2 * S * d * 2 * f / st['gemm1'] / 1e9:6.1f} TF/s fp32)"
          f"  gemm2 {st['gemm2'] * 1e3:7.1f} us ({2 * S * f * d / st['gemm2'] / 1e9:6.1f} TF/s)", flush=True)
    layer.close()
