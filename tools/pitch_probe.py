"""Switch-shaped GEMM1 efficiency vs the row pitch (d_model): tests whether
the short-K GEMM1's operand loads suffer from the L2 slice mapping of
1536-B row strides.  Routing-driven (uniform over 26 resident of 128
experts), T = 65,536, f = 3072, ReLU, bf16; prints TFLOP/s of GEMM1 and
GEMM2 from the stage events."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from helpers import build_layer, trace_logits  # noqa: E402

T, E, f = 65536, 128, 3072
resident = sorted(np.random.default_rng(26).choice(E, 26, replace=False).tolist())
rng = np.random.default_rng(0)
choices = rng.choice(resident, size=(T, 1)).astype(np.int32)
for d in [int(v) for v in sys.argv[1:]] or [768, 832, 896, 1024]:
    layer, _, _ = build_layer(E, d, f, 1, "bf16", "relu", "full_softmax", 26, resident, max_tokens=T,
                              gemm_cta_group=2)
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(1)).to(torch.bfloat16).cuda()
    lg = torch.from_numpy(trace_logits(choices, E)).cuda()
    for _ in range(3):
        layer.forward(x, logits=lg)
    torch.cuda.synchronize()
    layer.set_profiling(True)
    for _ in range(10):
        layer.forward(x, logits=lg)
    torch.cuda.synchronize()
    st = layer.stage_times()
    flop = 2.0 * T * d * f
    print(f"d={d:5d} pitch={d * 2:5d} B  gemm1 {st['gemm1'] * 1e3:7.1f} us {flop / st['gemm1'] / 1e9:7.1f} TF/s   "
          f"gemm2 {st['gemm2'] * 1e3:7.1f} us {flop / st['gemm2'] / 1e9:7.1f} TF/s", flush=True)
    layer.close()
