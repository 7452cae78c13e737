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
    assert d["config"]["tokens_per_step"] <= 512 and "of the 1x512 = 512 tokens" in cb["sample"]


def test_multi_gpu_default_is_expert_parallel():
    """bench.py --gpus N under torchrun measures the north star's EP split by
    default (the driver's SCALE run passes no --parallel)."""
    sys.path.insert(0, str(ROOT))
    import bench

    for argv in ([], ["--config", "stack"]):
        a = bench.build_parser().parse_args(argv)
        assert a.parallel == "ep" and a.ep_transport == "p2p"
        for n in (2, 4, 8):
            assert bench.parallelism_label(n, a.parallel, a.ep_transport) == f"ep{n}-p2p"
    assert bench.parallelism_label(1, "ep", "p2p") == "single"
    assert bench.parallelism_label(4, "replicas", "p2p") == "replicas4"


def test_reference_arm_is_independent_of_the_product():
    """--impl reference runs the reference's code and the oracle only: the
    product package is never imported and libemoe.so never mapped."""
    from oracle.oracle import have_port, have_ref

    if not (have_port() and have_ref()):
        pytest.skip("oracle not built")
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'synthetic', "
            "'--steps', '1', '--warmup', '3', '--ref-budget-s', '2']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT', any(m.startswith('paper_2503_06823_b200') for m in sys.modules), 'libemoe.so' in maps)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "PRODUCT False False" in out.stdout, out.stdout[-2000:]


@pytest.mark.gpu
def test_both_arms_same_inputs():
    """The reference arm and the GPU arm's cpu_baseline hash the same input
    bytes (x rows, W_g, resident experts) and agree on the resident set."""
    ref = run_bench("--impl", "reference", "--config", "synthetic", "--steps", "1", "--warmup", "3",
                    "--ref-budget-s", "4")
    gpu = run_bench("--config", "synthetic", "--steps", "3", "--warmup", "3", "--e2e-steps", "2")
    assert ref["config"]["input_digest"] == gpu["cpu_baseline"]["input_digest"]
    assert ref["config"]["resident_set"] == gpu["config"]["resident_set"]


@pytest.mark.gpu
@pytest.mark.parametrize("graph", ["on", "off"])
def test_gpu_arm_contract(graph):
    d = run_bench("--config", "synthetic", "--steps", "5", "--warmup", "3", "--e2e-steps", "4", "--graph", graph)
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    # every step launches at least: gate + routing (one kernel at this T), scan + permute (one kernel at
    # this T), GEMM1, GEMM2, combine and the A6 histogram update
    assert d["gpu_launches"] >= 5 * 6
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys() and 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert " of 512 tokens" in cb["sample"]  # the sample never exceeds the batch
    assert d["config"]["step_launch"].startswith("one CUDA graph" if graph == "on" else "eager")


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_gpu_arm_expert_parallel_path(transport):
    """The bench's expert-parallel path (a world-1 group on this one-GPU box):
    the EP forward runs in the timed steps, and for the peer-memory transport
    the line carries the EP stage times, exchange volume and placement (both
    transports: the NCCL one from events on the compute stream)."""
    d = run_bench("--config", "tiny", "--steps", "4", "--warmup", "3", "--e2e-steps", "3", "--ep-at-1",
                  "--ep-transport", transport, "--no-cpu-baseline")
    assert d["value"] > 0 and d["gpu_launches"] > 0
    if transport == "p2p":
        ep = d["ep"]
        assert set(ep["stages_ms"]) == {"route", "count_exchange", "dispatch", "dispatch_wait", "gemm1",
                                        "gemm2_return", "return_wait", "combine"}
        assert ep["rows_computed_per_rank"][0] > 0 and ep["placement"]
    else:
        ep = d["ep"]
        assert set(ep["stages_ms"]) == {"route", "count_exchange", "dispatch", "dispatch_a2a", "ffn", "return_a2a",
                                        "combine"}
        assert ep["stages_ms"]["ffn"] > 0 and ep["exchange"]["a2a_bytes_per_call"] > 0 and ep["placement"]


@pytest.mark.gpu
def test_p2p_failure_falls_back_to_nccl():
    """A peer-memory EP that cannot run (here: a 1-row receive buffer, so the
    first forward reports an overflow) makes every rank fall back to the NCCL
    transport with the same placement, and the line says why."""
    d = run_bench("--config", "tiny", "--steps", "2", "--warmup", "3", "--e2e-steps", "2", "--ep-at-1",
                  "--ep-transport", "p2p", "--ep-recv-cap", "1", "--no-cpu-baseline")
    assert d["value"] > 0 and d["ep"]["transport"].startswith("nccl")
    assert "status 2" in d["config"]["ep_p2p_fallback"]


@pytest.mark.gpu
def test_stack_expert_parallel_path():
    """--config stack on the EP path (world-1 group, 3 layers): every layer's
    EP handle on one shared region, the gate computed per layer."""
    d = run_bench("--config", "stack", "--stream-layers", "3", "--steps", "2", "--warmup", "3", "--ep-at-1")
    assert d["value"] > 0 and d["ep"]["layers"] == 3 and d["config"]["routing_follows_trace"]
