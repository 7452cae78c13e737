"""Probe: does tcgen05.mma.kind::tf32 read a raw fp32 operand as its
truncation to tf32?  Runs the config-1 shaped fp32 layer and prints the FFN
rows' error against the oracle (fp64).  Built normally the weight pools hold
hi = rn_tf32(W), lo = W - hi; built with -DEMOE_TF32_RAW_HI_PROBE they hold
hi = W (raw) and lo = W - trunc_tf32(W): the error stays ~1e-6 iff the tensor
core truncates raw operands (the premise of splitting operands in shared
memory instead of HBM)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
from helpers import rel_errors, to_f32  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from test_forward_gpu import run_case  # noqa: E402

port = Port()
c = run_case("config1_fp32_phi05", port)
ws = c["ws"]
seg = ws["seg_offsets"].cpu().numpy()
src = ws["row_token"].cpu().numpy()
yp = to_f32(ws["y_perm"])
x32 = to_f32(c["x"])
worst = (0.0, 0.0)
for e in range(c["E"]):
    rows = [r for r in range(int(seg[e]), int(seg[e + 1])) if src[r] >= 0][:16]
    if not rows:
        continue
    w1, w3, w2 = (to_f32(w) for w in c["experts"][e])
    ref = port.expert_ffn(x32[src[rows]], w1, w3, w2, 0, False)
    n, m = rel_errors(yp[rows], ref)
    worst = (max(worst[0], n), max(worst[1], m))
print(f"FFN rows vs oracle: norm {worst[0]:.3e} max {worst[1]:.3e}")
