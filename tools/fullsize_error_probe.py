"""Diagnostic: error budget of the bf16 FFN at the full Mixtral shape.

Compares, on sampled rows of each resident expert, the GPU rows with the
oracle computed with mirrored bf16 rounding (H, Y rounded) and without (fp32
H, fp64 accumulation): shows how much of the GPU-vs-mirrored difference is
rounding flips at K = 4096 / 14336 rather than GPU error."""
import os
os.environ.setdefault("EMOE_FUSED_COMBINE", "0")  # these probes read the per-row Y_perm

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import rel_errors, to_f32  # noqa: E402
from oracle.oracle import Port, bf16_round  # noqa: E402
from test_fullsize_gpu import full_layer  # noqa: E402


def main():
    port = Port()
    E, d, f, k = 8, 4096, 14336, 2
    resident = [0, 5, 6, 7]
    layer, wg, experts, x = full_layer(E, d, f, k, "swiglu", "topk_softmax", resident, 65536)
    layer.forward(x)
    torch.cuda.synchronize()
    ws = layer.workspace()
    counts = ws["counts"].cpu().numpy()
    offs = ws["seg_offsets"].cpu().numpy()
    src = ws["row_token"].cpu().numpy()
    rng = np.random.default_rng(1)
    for e in resident:
        rows = rng.choice(np.arange(offs[e], offs[e] + counts[e]), size=32, replace=False)
        w1, w3, w2 = (to_f32(w) for w in experts[e])
        xs = to_f32(x[torch.from_numpy(src[rows]).cuda()])
        mirrored = port.expert_ffn(xs, w1, w3, w2, 0, True)
        exact = port.expert_ffn(xs, w1, w3, w2, 0, False)
        gpu = to_f32(ws["y_perm"][torch.from_numpy(rows).cuda()])
        print(f"expert {e}: gpu~mirrored {rel_errors(gpu, mirrored)}  gpu~exact {rel_errors(gpu, exact)}  "
              f"mirrored~exact {rel_errors(mirrored, exact)}  bf16(exact)~exact {rel_errors(bf16_round(exact), exact)}")
    layer.close()


if __name__ == "__main__":
    main()
