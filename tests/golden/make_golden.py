"""Generate the golden fixtures from the reference itself (oracle/_ref built
from /root/reference by `make -C oracle ref`).  Run here, where the reference
exists; the JSON files are committed so the oracle can be pinned anywhere.

    python tests/golden/make_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle.oracle import Ref  # noqa: E402


def tolist(a):
    return np.asarray(a).tolist()


def main():
    R = Ref()
    out = {}
    # --- routing trace generator (workload.cpp:242-286)
    traces = []
    for i, (m, E, k, ll, pl, ie, seed, P, T) in enumerate(
            [(2, 8, 2, 0.6, 0.8, 0, 17, 6, 16), (1, 8, 2, 0.6, 0.8, 0, 17, 4, 64), (3, 16, 1, 0.5, 0.9, 3, 5, 5, 9)]):
        tr = R.gen_routing_trace(m, E, k, ll, pl, ie, seed, P, T)
        traces.append(dict(args=[m, E, k, ll, pl, ie, seed, P, T], trace=tolist(tr)))
    out["gen_routing_trace"] = traces

    # --- fit + dominant/sets + predictions on each trace
    fits = []
    for t in traces:
        tr = np.array(t["trace"], np.int32)
        P, m, T, k = tr.shape
        E = t["args"][1]
        names = ["a", "b"]
        tids = np.array([p % 2 for p in range(P)], np.int32)
        f = R.fit(tr, tids, names, 0.01, E)
        sets = [R.prompt_expert_sets(tr, p) for p in range(P)]
        s, z = sets[-1][1], sets[-1][2]
        preds = {}
        for mode in (0, 1):
            sc, ex, n = R.predict(f, mode, s if mode == 0 else s[:1], z if mode == 0 else z[:1], k=k)
            preds[str(mode)] = dict(scores=tolist(sc), experts=tolist(ex), n=tolist(n))
        if m > 1:
            sc, ex, n = R.predict(f, 2, s[:1], z[:1], layer=1, k=k)
            preds["2"] = dict(scores=tolist(sc), experts=tolist(ex), n=tolist(n))
        freqs = {nm: tolist(R.predicted_frequencies(f["task_counts"], names, 0.01, nm)) for nm in names + ["zz"]}
        fits.append(dict(E=E, layer_counts=tolist(f["layer_counts"]), prompt_counts=tolist(f["prompt_counts"]),
                         task_counts=tolist(f["task_counts"]),
                         dominant=[tolist(x[0]) for x in sets], sets=[tolist(x[1]) for x in sets],
                         set_sizes=[tolist(x[2]) for x in sets], predictions=preds, frequencies=freqs))
    out["fit"] = fits

    # --- route_token on seeded random inputs
    rng = np.random.default_rng(7)
    routes = []
    for E, k in [(8, 2), (8, 3), (128, 1), (16, 4)]:
        T = 64
        ch = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
        res = (rng.random(E) < 0.4).astype(np.uint8)
        res[0] = 1
        sc = np.round(rng.random(E) * 4) / 4
        ex, rk, hit = R.route_tokens(ch, res, sc)
        ex2, rk2, hit2 = R.route_tokens(ch, res, None)
        routes.append(dict(choices=tolist(ch), resident=tolist(res), scores=tolist(sc), expert=tolist(ex),
                           rank=tolist(rk), hit=tolist(hit), expert_noscores=tolist(ex2)))
    out["route_token"] = routes

    # --- Eq. 2 / select / targets / plan on seeded random instances
    eq = []
    for i in range(6):
        m, E = int(rng.integers(1, 5)), int(rng.integers(2, 33))
        names = ["t0", "t1", "t2"]
        wo = rng.uniform(1, 300, 3).round(1)
        sens = rng.integers(0, 2, (3, m)).astype(np.int32)
        has = np.array([1, 0, 1], np.uint8)
        running = [(int(rng.integers(3)), int(rng.integers(1, 500))) for _ in range(7)]
        incoming = [(int(rng.integers(3)), int(rng.integers(1, 500))) for _ in range(3)]
        freqs = rng.random((2, m, E))
        freqs /= freqs.sum(-1, keepdims=True)
        agg = R.expected_tokens(m, E, names, wo, sens, has, running, incoming, ["t0", "t2"], freqs, True)
        budgets = rng.integers(1, E + 1, m).astype(np.int32)
        resident = (rng.random((m, E)) < 0.5).astype(np.uint8)
        sel = R.select_experts(agg, budgets)
        tg = R.loading_targets(agg, resident, budgets)
        plan = R.plan_loading(resident, np.full(m, E, np.int32), tg, agg, 0.01, 1e9, 1000)
        eq.append(dict(m=m, E=E, names=names, wo=tolist(wo), sens=tolist(sens), has=tolist(has), running=running,
                       incoming=incoming, freq_names=["t0", "t2"], freqs=tolist(freqs), aggregate=tolist(agg),
                       budgets=tolist(budgets), resident=tolist(resident), select=[tolist(s) for s in sel],
                       targets=[tolist(s) for s in tg], evictions=[tolist(s) for s in plan["evictions"]],
                       loads=[tolist(s) for s in plan["loads"]], duration=tolist(plan["duration"]),
                       delta_e=plan["delta_e"], total_loads=plan["total_loads"]))
    out["expected_tokens_plan"] = eq
    out["rng"] = dict(seed=1234, uniform=tolist(R.rng_uniform(1234, 8)), normal=tolist(R.rng_normal(1234, 8)))
    (HERE / "reference_golden.json").write_text(json.dumps(out))
    print("wrote", HERE / "reference_golden.json")


if __name__ == "__main__":
    main()
