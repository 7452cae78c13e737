"""Drop-in proof: the reference's own test suites (proj/tests/*.cpp, built
unchanged by `make -C oracle dropin`) pass when the reference's
expert_store.o / predictor.o are replaced by the emoe compat layer
(paper_2503_06823_b200/compat/moesim_compat.cpp), i.e. when route_token, fit,
predict_*, predicted_frequencies, expected_tokens, select_experts,
loading_targets and plan_loading run on the GPU through include/emoe.h --
and, through a workload.o whose two symbols are weakened at link time,
dominant_expert and prompt_expert_sets (workload.cpp:350-377) as well."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["dropin_test_expert_store", "dropin_test_predictor", "dropin_test_engine",
                                   "dropin_test_workload", "dropin_test_acceptance"])
def test_reference_suite_on_emoe(suite):
    exe = ROOT / "oracle" / "_ref" / suite
    if not exe.exists():
        pytest.skip("drop-in binaries not built (make -C oracle dropin, needs /root/reference at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
