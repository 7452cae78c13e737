"""Error of the 3xTF32 FFN against the oracle (fp64-accumulated restatement)
on the config-1 parity cases, for the accumulator chunk length in
EMOE_TF32_CHUNK: prints the worst norm-wise and max-element relative errors
of every fp32 check (tolerance 1e-5).  Run on a GPU:
    EMOE_TF32_CHUNK=8 python tools/tf32_chunk_error_probe.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import helpers  # noqa: E402

worst = {"norm": 0.0, "max": 0.0}
_orig = helpers.assert_f32_close


def _record(got, ref, what=""):
    norm, mx = helpers.rel_errors(got, ref)
    worst["norm"] = max(worst["norm"], norm)
    worst["max"] = max(worst["max"], mx)
    return norm, mx


helpers.assert_f32_close = _record
import test_forward_gpu as tf  # noqa: E402

tf.assert_f32_close = _record
from oracle.oracle import Port  # noqa: E402

port = Port()
for name in ("config1_fp32_phi05", "config1_fp32_phi1", "fp32_relu_top1", "fp32_many_tokens"):
    c = tf.run_case(name, port)
    tf.check_case(c, port)
    c["layer"].close()
print(f"EMOE_TF32_CHUNK={os.environ.get('EMOE_TF32_CHUNK', '4')}: worst fp32 error norm {worst['norm']:.3e} "
      f"max {worst['max']:.3e} (tolerance {helpers.F32_TOL})")
