"""Debug check of the grouped tcgen05 GEMMs against torch.matmul on the GPU.

python tools/gemm_check.py [T] [d] [f] [E] [k] [slots]
Prints per-expert max/norm relative errors of H (GEMM1 SwiGLU) and Y (GEMM2).
"""
import os
os.environ.setdefault("EMOE_FUSED_COMBINE", "0")  # these probes read the per-row Y_perm

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import build_layer  # noqa: E402


def main():
    a = [int(v) for v in sys.argv[1:]] + [0] * 7
    T, d, f, E, k, slots, cg = (a[0] or 2048, a[1] or 1024, a[2] or 2048, a[3] or 8, a[4] or 2, a[5] or 4, a[6])
    layer, wg, experts = build_layer(E, d, f, k, "bf16", "swiglu", "topk_softmax", slots, list(range(0, E, 2))[:slots],
                                     max_tokens=T, gemm_cta_group=cg)
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(5)).to(torch.bfloat16).cuda()
    y = layer.forward(x)
    torch.cuda.synchronize()
    ws = layer.workspace()
    off = ws["seg_offsets"].cpu().tolist()
    cnt = ws["counts"].cpu().tolist()
    print("cta_group", layer.gemm_cta_group, "counts", cnt, "offsets", off)
    ok = True
    for e in range(E):
        n = cnt[e]
        if n == 0:
            continue
        rows = slice(off[e], off[e] + n)
        xp = ws["x_perm"][rows].float()
        w1, w3, w2 = (w.cuda().float() for w in experts[e])
        g = xp @ w1.T
        u = xp @ w3.T
        h_ref = (g * torch.sigmoid(g) * u)
        h = ws["h"][rows].float()
        eh = ((h - h_ref).norm() / h_ref.norm()).item()
        mh = ((h - h_ref).abs().max() / h_ref.abs().max()).item()
        y_ref = h.to(torch.bfloat16).float() @ w2.T
        yp = ws["y_perm"][rows].float()
        ey = ((yp - y_ref).norm() / y_ref.norm()).item()
        my = ((yp - y_ref).abs().max() / y_ref.abs().max()).item()
        print(f"expert {e}: rows {n} H norm {eh:.2e} max {mh:.2e} | Y norm {ey:.2e} max {my:.2e}")
        ok &= eh < 1e-2 and ey < 1e-2
        if eh > 1e-2:
            bad = ((h - h_ref).abs() > 0.05 * h_ref.abs().max()).nonzero()
            print("  first bad H entries (row, col):", bad[:8].tolist())
    print("GEMM CHECK", "PASS" if ok else "FAIL")


if __name__ == "__main__":
    main()
