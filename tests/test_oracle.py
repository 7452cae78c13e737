"""Pins the CPU oracle (oracle/emoe_oracle.c) before it is trusted:
  * against the golden fixtures generated from the reference itself
    (tests/golden/reference_golden.json, tests/golden/make_golden.py);
  * against the reference build (oracle/_ref) on seeded random cases;
  * the reference's own unit suites pass under our doctest shim.
No GPU needed."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLD = json.loads((ROOT / "tests" / "golden" / "reference_golden.json").read_text())


def test_port_fit_and_predict_match_golden(port):
    for t, f in zip(GOLD["gen_routing_trace"], GOLD["fit"]):
        tr = np.array(t["trace"], np.int32)
        P, m, T, k = tr.shape
        E = f["E"]
        got = port.fit(tr, np.array([p % 2 for p in range(P)], np.int32), 2, E)
        assert got["E"] == E
        assert np.array_equal(got["layer_counts"], np.array(f["layer_counts"]).reshape(got["layer_counts"].shape))
        assert np.array_equal(got["prompt_counts"], np.array(f["prompt_counts"]))
        assert np.array_equal(got["task_counts"], np.array(f["task_counts"]))
        for p in range(P):
            assert port.dominant_expert(tr, p, 0) == f["dominant"][p][0]
            s, z = port.prompt_expert_sets(tr, p)
            assert np.array_equal(z, f["set_sizes"][p])
            for l in range(m):
                assert list(s[l, : z[l]]) == f["sets"][p][l][: z[l]]
        got["smoothing"] = 0.01
        s, z = port.prompt_expert_sets(tr, P - 1)
        for mode, want in f["predictions"].items():
            mode = int(mode)
            sc, ex, n = port.predict(got, mode, s if mode == 0 else s[:1], z if mode == 0 else z[:1], layer=1, k=k)
            rows = len(want["n"])
            assert np.array_equal(sc[:rows], np.array(want["scores"])), mode
            assert np.array_equal(ex[:rows], np.array(want["experts"])), mode
        for i, name in enumerate(["a", "b", "zz"]):
            got_f = port.predicted_frequencies(got["task_counts"], 0.01, i if i < 2 else -1)
            assert np.array_equal(got_f, np.array(f["frequencies"][name]))


def test_port_route_token_matches_golden(port):
    for r in GOLD["route_token"]:
        ch = np.array(r["choices"], np.int32)
        res = np.array(r["resident"], np.uint8)
        ex, rk, hit = port.route_tokens(ch, res, np.array(r["scores"]))
        assert ex.tolist() == r["expert"] and rk.tolist() == r["rank"] and hit.tolist() == r["hit"]
        ex, _, _ = port.route_tokens(ch, res, None)
        assert ex.tolist() == r["expert_noscores"]


def test_port_eq2_select_plan_match_golden(port):
    for c in GOLD["expected_tokens_plan"]:
        m, E = c["m"], c["E"]
        reqs = c["running"] + c["incoming"]
        fp = np.array([1, 0, 1], np.uint8)
        fr = np.zeros((3, m, E))
        fr[0], fr[2] = np.array(c["freqs"][0]), np.array(c["freqs"][1])
        agg = port.expected_tokens(m, E, c["wo"], np.array(c["sens"]), c["has"], [r[0] for r in reqs],
                                   [r[1] for r in reqs], fp, fr, True)
        assert np.array_equal(agg, np.array(c["aggregate"]))
        assert port.select_experts(agg, c["budgets"]) == c["select"]
        tg = port.loading_targets(agg, np.array(c["resident"], np.uint8), c["budgets"])
        assert tg == c["targets"]
        plan = port.plan_loading(np.array(c["resident"], np.uint8), np.full(m, E, np.int32), tg, agg,
                                 0.01 + 1000 / 1e9)
        assert plan["evictions"] == c["evictions"] and plan["loads"] == c["loads"]
        assert plan["duration"].tolist() == c["duration"] and plan["delta_e"] == c["delta_e"]


def test_product_trace_generator_matches_golden():
    """The product's host-side generator (libemoe, no GPU) is the reference's bit for bit."""
    import paper_2503_06823_b200 as emoe

    for t in GOLD["gen_routing_trace"]:
        m, E, k, ll, pl, ie, seed, P, T = t["args"]
        got = emoe.gen_routing_trace(emoe.ModelShape(m, E, k), ll, pl, ie, seed, P, T)
        assert np.array_equal(got, np.array(t["trace"], np.int32))


@pytest.mark.parametrize("seed", range(10))
def test_port_matches_reference_random(seed, port, ref):
    rng = np.random.default_rng(seed)
    m, E, k = int(rng.integers(1, 6)), int(rng.choice([2, 4, 8, 16, 64])), 0
    k = int(rng.integers(1, min(E, 4) + 1))
    P, T = int(rng.integers(2, 40)), int(rng.integers(1, 40))
    tr = ref.gen_routing_trace(m, E, k, float(rng.uniform()), float(rng.uniform()), int(rng.integers(E)), seed, P, T)
    names = ["x", "y", "z"]
    tids = rng.integers(0, 3, P).astype(np.int32)
    used = sorted({names[i] for i in tids})
    remap = np.array([used.index(names[i]) for i in tids], np.int32)
    r = ref.fit(tr, remap, used, 0.01, 0)
    p = port.fit(tr, remap, len(used), 0)
    assert r["E"] == p["E"]
    for key in ("layer_counts", "prompt_counts", "task_counts"):
        assert np.array_equal(r[key], p[key]), key
    # route_token
    ch = np.stack([rng.permutation(E)[:k] for _ in range(500)]).astype(np.int32)
    res = (rng.random(E) < 0.5).astype(np.uint8)
    res[int(rng.integers(E))] = 1
    sc = np.round(rng.random(E) * 3) / 3
    for a, b in zip(ref.route_tokens(ch, res, sc), port.route_tokens(ch, res, sc)):
        assert np.array_equal(a, b)


def test_port_reports_reference_errors(port):
    from oracle.oracle import LogicError, ValidationError

    with pytest.raises(LogicError):
        port.route_tokens(np.array([[1, 2]], np.int32), np.zeros(4, np.uint8))
    with pytest.raises(ValidationError):
        port.select_experts(np.zeros((1, 4)), [5])
    with pytest.raises(ValidationError):
        port.plan_loading(np.zeros((1, 4), np.uint8), [2], [[0, 1, 2]], np.zeros((1, 4)), 0.1)


@pytest.mark.parametrize("suite", ["test_predictor", "test_expert_store", "test_workload", "test_engine",
                                   "test_acceptance"])
def test_reference_suites_pass(suite):
    """The reference's own suites, built unchanged against the reference objects
    with our doctest shim (oracle/Makefile), pass here."""
    exe = ROOT / "oracle" / "_ref" / suite
    if not exe.exists():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
