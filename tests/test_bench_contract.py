"""bench.py keeps the driver's JSON contract: the reference arm on the host
cores (CPU, runs here) and the GPU arm on a B200 (a short synthetic run)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    from oracle.oracle import have_port, have_ref

    if not (have_port() and have_ref()):
        pytest.skip("oracle not built")
    d = run_bench("--impl", "reference", "--config", "synthetic", "--steps", "1", "--warmup", "3",
                  "--ref-budget-s", "4")
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= cb.keys() and cb["kind"] in ("port", "reference")
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("graph", ["on", "off"])
def test_gpu_arm_contract(graph):
    d = run_bench("--config", "synthetic", "--steps", "5", "--warmup", "3", "--e2e-steps", "4", "--graph", graph)
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] >= 5 * 8  # every step launches the routing, permutation, GEMM and combine kernels
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys() and 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert d["config"]["step_launch"].startswith("one CUDA graph" if graph == "on" else "eager")
