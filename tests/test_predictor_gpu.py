"""GPU parity of the predictor path (A2, A6, A7, A8) against the reference
itself (oracle/_ref) and the oracle port: bit-exact for every integer and fp64
output, on the reference's own frozen examples and on seeded random cases."""
import numpy as np
import pytest

import paper_2503_06823_b200 as emoe

pytestmark = pytest.mark.gpu


def shape(m, E, k, eb=1000, bb=5000):
    return emoe.ModelShape(m, E, k, eb, bb)


# ---------------- A2 route_token ----------------
def test_route_token_frozen_examples():
    """test_expert_store.cpp:299-329"""
    p = emoe.Placement.empty(shape(1, 8, 3), [3])
    for e in (2, 7, 4):
        p.load(0, e)
    r = emoe.route_token([2, 5, 6], p, 0, [])
    assert (r.expert, r.rank, r.hit) == (2, 0, True)
    r = emoe.route_token([5, 4, 6], p, 0, [])
    assert (r.expert, r.rank, r.hit) == (4, 1, False)
    r = emoe.route_token([5, 6, 0], p, 0, [0, 0, 0.1, 0, 0.2, 0.9, 0.8, 0.7])
    assert (r.expert, r.rank, r.hit) == (7, -1, False)
    assert emoe.route_token([5, 6, 0], p, 0, []).expert == 2
    with pytest.raises(emoe.LogicError):
        emoe.route_token([1, 2, 3], emoe.Placement.empty(shape(1, 8, 3), [3]), 0, [])


@pytest.mark.parametrize("seed", range(4))
def test_route_tokens_random_vs_reference(seed, ref):
    rng = np.random.default_rng(seed)
    E = int(rng.integers(2, 129))
    k = int(rng.integers(1, min(8, E) + 1))
    T = 5000
    choices = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    resident = (rng.random(E) < rng.uniform(0.1, 0.9)).astype(np.uint8)
    resident[rng.integers(E)] = 1
    scores = None if seed % 2 else np.round(rng.random(E) * 4) / 4  # ties exercised
    a = emoe.route_tokens(choices, resident, scores)
    b = ref.route_tokens(choices, resident, scores)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


# ---------------- A6 fit / dominant / sets ----------------
@pytest.mark.parametrize("case", [(3, 8, 2, 0.6, 0.8, 40, 64), (1, 8, 2, 0.6, 0.8, 30, 2048), (6, 128, 1, 0.5, 0.9, 20, 300),
                                  (4, 32, 4, 0.3, 0.4, 25, 17),
                                  # BASELINE sizes: config 2/3 history (200 prompts of 2048 tokens),
                                  # config 5 (32 layers, 8k-token prompts)
                                  (1, 8, 2, 0.6, 0.8, 200, 2048), (1, 128, 1, 0.6, 0.8, 200, 2048),
                                  (32, 8, 2, 0.6, 0.8, 40, 8192)])
def test_fit_matches_reference(case, ref):
    m, E, k, ll, pl, P, T = case
    tr = ref.gen_routing_trace(m, E, k, ll, pl, 0, 17, P, T)
    names = ["qa", "chat", "code"]
    tids = [names[p % 3] for p in range(P)]
    model = emoe.fit(tr, tids, 0.01, E)
    sorted_names = sorted(set(tids))
    r = ref.fit(tr, np.array([sorted_names.index(t) for t in tids], np.int32), sorted_names, 0.01, E)
    assert np.array_equal(model.layer_counts, r["layer_counts"])
    assert np.array_equal(model.prompt_counts, r["prompt_counts"])
    assert np.array_equal(model.task_counts, r["task_counts"])
    assert model.task_ids == sorted_names
    for p in (0, P // 2, P - 1):
        dom, sets = emoe.prompt_expert_sets(tr, p)
        rd, rs, rz = ref.prompt_expert_sets(tr, p)
        assert dom == list(rd)
        assert sets == [list(rs[l, : rz[l]]) for l in range(m)]


def test_fit_hand_trace():
    """test_predictor.cpp:106-150 (hand-counted tallies)"""
    t = np.array([
        [[[0, 1], [0, 2]], [[1, 2], [1, 3]], [[2, 3], [0, 1]]],
        [[[3, 0], [3, 2]], [[3, 1], [0, 2]], [[1, 0], [1, 2]]],
        [[[2, 1], [1, 0]], [[2, 0], [2, 3]], [[3, 0], [3, 1]]],
    ], np.int32)
    m = emoe.fit(t, ["a", "b", "a"])
    l0 = np.zeros((4, 4))
    l0[0, 1] = 2; l0[3, 3] = 1; l0[3, 0] = 1; l0[2, 2] = 1; l0[1, 2] = 1  # noqa: E702
    l1 = np.zeros((4, 4))
    l1[1, 2] = 1; l1[1, 0] = 1; l1[3, 1] = 1; l1[0, 1] = 1; l1[2, 3] = 2  # noqa: E702
    assert np.array_equal(m.layer_counts[0], l0) and np.array_equal(m.layer_counts[1], l1)
    p0 = np.zeros((4, 4)); p0[0, 3] = 1; p0[3, 1] = 1  # noqa: E702
    p1 = np.zeros((4, 4)); p1[1, 0] = 1; p1[0, 2] = 1  # noqa: E702
    p2 = np.zeros((4, 4)); p2[0, 1] = 1; p2[1, 3] = 1  # noqa: E702
    assert np.array_equal(m.prompt_counts, np.stack([p0, p1, p2]))
    assert np.array_equal(m.task_counts[0], [[3, 3, 2, 0], [1, 2, 3, 2], [2, 2, 1, 3]])
    assert np.array_equal(m.task_counts[1], [[1, 0, 1, 2], [1, 1, 1, 1], [1, 2, 1, 0]])


def test_fit_incremental_equals_concatenation(ref):
    """counts commute (test_predictor.cpp:284-296): two hist updates == one fit"""
    import ctypes as C

    import torch

    tr = ref.gen_routing_trace(3, 8, 2, 0.6, 0.7, 0, 11, 30, 20)
    full = emoe.fit(tr, [], 0.01, 8)
    pred = emoe.moesim._Pred(3, 8, 2, 0, 0.01)
    for part in (tr[:13], tr[13:]):
        d = torch.from_numpy(np.ascontiguousarray(part)).cuda()
        emoe.moesim.check(emoe._lib.lib.emoe_hist_update(pred.h, C.c_void_p(d.data_ptr()), part.shape[0], 20, None,
                                                         None))
        torch.cuda.synchronize()
    lc = np.zeros((2, 8, 8))
    pc = np.zeros((3, 8, 8))
    emoe.moesim.check(emoe._lib.lib.emoe_predictor_counts_host(pred.h, emoe.moesim._p(lc), emoe.moesim._p(pc), None))
    assert np.array_equal(lc, full.layer_counts) and np.array_equal(pc, full.prompt_counts)


# ---------------- A7 predict / frequencies ----------------
@pytest.mark.parametrize("seed", range(6))
def test_predict_matches_reference(seed, ref):
    rng = np.random.default_rng(100 + seed)
    m, E, k = int(rng.integers(2, 7)), int(rng.choice([4, 8, 32, 128])), int(rng.integers(1, 4))
    tr = ref.gen_routing_trace(m, E, k, float(rng.uniform(0.2, 0.9)), float(rng.uniform(0.2, 0.95)), 0, seed,
                               int(rng.integers(5, 60)), int(rng.integers(1, 50)))
    smoothing = [0.01, 1.0, 1e6, 0.0][seed % 4]
    model = emoe.fit(tr, [], smoothing, E)
    r = dict(layer_counts=model.layer_counts, prompt_counts=model.prompt_counts, smoothing=smoothing)
    _, sets = emoe.prompt_expert_sets(tr, tr.shape[0] - 1)
    a = emoe.predict_all_layers(model, sets)
    arr, sizes = emoe.moesim._sets_array(sets, k)
    rs, re_, rn = ref.predict(r, 0, arr, sizes, k=k)
    for l in range(m):
        assert a[l].experts == list(re_[l, : rn[l]])
        assert np.array_equal(a[l].scores, rs[l])
    c = emoe.predict_chained(model, sets[0])
    rs, re_, rn = ref.predict(r, 1, arr[:1], sizes[:1], k=k)
    for l in range(m):
        assert c[l].experts == list(re_[l, : rn[l]]) and np.array_equal(c[l].scores, rs[l])
    lw = emoe.predict_layerwise(model, sets[0], 1)
    rs, re_, rn = ref.predict(r, 2, arr[:1], sizes[:1], layer=1, k=k)
    assert lw.experts == list(re_[0, : rn[0]]) and np.array_equal(lw.scores, rs[0])


def test_predict_frozen_examples():
    """uniform ties (test_predictor.cpp:252-267), huge smoothing (:269-282)"""
    z = np.zeros
    model = emoe.TransitionModel(3, 6, 3, 0.01, z((2, 6, 6)), z((3, 6, 6)), [], z((0, 3, 6)))
    lp = emoe.predict_layerwise(model, [2], 1)
    assert lp.experts == [0, 1, 2]
    assert np.allclose(lp.scores, 1 / 6)
    for layer in emoe.predict_all_layers(model, [[4], [1], [5]]):
        assert layer.experts == [0, 1, 2]
    # rank_scores band: counts {1999, 2000} tie -> index order; {1990, 2000} -> score order
    pc = z((1, 4, 4))
    pc[0, 0, :2] = [1999, 2000]
    m1 = emoe.TransitionModel(1, 4, 2, 0.01, z((0, 4, 4)), pc, [], z((0, 1, 4)))
    assert emoe.predict_all_layers(m1, [[0]])[0].experts == [0, 1]
    pc[0, 0, :2] = [1990, 2000]
    assert emoe.predict_all_layers(m1, [[0]])[0].experts == [1, 0]
    with pytest.raises(emoe.ValidationError):
        emoe.predict_layerwise(model, [1], 0)
    with pytest.raises(emoe.ValidationError):
        emoe.predict_layerwise(model, [], 1)
    with pytest.raises(emoe.ValidationError):
        emoe.predict_layerwise(model, [7], 1)
    with pytest.raises(emoe.ValidationError):
        emoe.predict_all_layers(model, [[0], [1]])


def test_predicted_frequencies_match_reference(ref):
    tr = ref.gen_routing_trace(3, 8, 2, 0.5, 0.8, 1, 77, 24, 16)
    tids = [["low", "high", "mid"][p % 3] for p in range(24)]
    model = emoe.fit(tr, tids, 0.01, 8)
    for task in ["high", "low", "mid", "unseen"]:
        got = emoe.predicted_frequencies(model, task)
        want = ref.predicted_frequencies(model.task_counts, model.task_ids, 0.01, task)
        assert np.array_equal(got, want)


# ---------------- A7 Eq. 2, select, targets ----------------
def test_expected_tokens_frozen():
    """test_expert_store.cpp:79-132"""
    prof = [emoe.TaskProfile("qa", 200.0, 200.0, [1])]
    n = emoe.expected_tokens(shape(1, 4, 1), prof, [emoe.Request("qa", 100)], [emoe.Request("qa", 50)],
                             {"qa": np.full((1, 4), 0.25)})
    assert np.allclose(n.aggregate, 137.5) and n.task_ids == ["qa"]
    prof = [emoe.TaskProfile("a", 10.0, 10.0, [1]), emoe.TaskProfile("b", 20.0, 20.0, [1])]
    n = emoe.expected_tokens(shape(1, 2, 1), prof, [emoe.Request("a", 5), emoe.Request("b", 8)], [],
                             {"a": np.array([[1.0, 0.0]]), "b": np.array([[0.0, 1.0]])})
    assert n.aggregate[0].tolist() == [15.0, 28.0]
    with pytest.raises(emoe.ValidationError):
        emoe.expected_tokens(shape(1, 2, 1), prof, [emoe.Request("ghost", 5)], [], {})


@pytest.mark.parametrize("seed", range(8))
def test_expected_tokens_random_vs_reference(seed, ref):
    rng = np.random.default_rng(seed)
    m, E = int(rng.integers(1, 9)), int(rng.integers(2, 65))
    names = sorted({f"t{int(i)}" for i in rng.integers(0, 6, size=int(rng.integers(1, 5)))})
    wo = rng.uniform(1, 300, len(names)).round(1)
    sens = rng.integers(0, 2, (len(names), m)).astype(np.int32)
    has = rng.integers(0, 2, len(names)).astype(np.uint8)
    running = [(int(rng.integers(len(names))), int(rng.integers(1, 500))) for _ in range(int(rng.integers(0, 30)))]
    incoming = [(int(rng.integers(len(names))), int(rng.integers(1, 500))) for _ in range(int(rng.integers(1, 10)))]
    fnames = [n for n in names if rng.random() < 0.7]
    freqs = rng.random((len(fnames), m, E))
    freqs /= freqs.sum(-1, keepdims=True)
    for aware in (True, False):
        want = ref.expected_tokens(m, E, names, wo, sens, has, running, incoming, fnames, freqs, aware)
        profiles = [emoe.TaskProfile(n, float(wo[i]), 1.0, list(sens[i]) if has[i] else []) for i, n in enumerate(names)]
        got = emoe.expected_tokens(shape(m, E, 1), profiles, [emoe.Request(names[t], n) for t, n in running],
                                   [emoe.Request(names[t], n) for t, n in incoming],
                                   {n: freqs[i] for i, n in enumerate(fnames)}, aware)
        assert np.array_equal(got.aggregate, want)


@pytest.mark.parametrize("seed", range(8))
def test_select_targets_plan_random_vs_reference(seed, ref):
    rng = np.random.default_rng(1000 + seed)
    m, E = int(rng.integers(1, 6)), int(rng.integers(2, 129))
    agg = np.where(rng.random((m, E)) < 0.3, 0.0, np.round(rng.random((m, E)) * 50) / 2)  # ties
    agg[rng.random(m) < 0.3] = 0.0  # masked layers
    budgets = rng.integers(1, E + 1, m).astype(np.int32)
    sel = emoe.select_experts(agg, shape(m, E, 1), list(budgets))
    assert sel == [list(map(int, r)) for r in ref.select_experts(agg, budgets)]
    resident = (rng.random((m, E)) < 0.5).astype(np.uint8)
    cur = emoe.Placement.empty(shape(m, E, 1), [E] * m)
    for l in range(m):
        for e in np.flatnonzero(resident[l]):
            cur.load(l, int(e))
    tg = emoe.loading_targets(agg, cur, list(budgets))
    assert tg == [list(map(int, r)) for r in ref.loading_targets(agg, resident, budgets)]
    cost = emoe.CostModel(per_expert_transfer=0.01, hd_bandwidth=1e9)
    plan = emoe.plan_loading(cur, tg, agg, cost)
    want = ref.plan_loading(resident, np.full(m, E, np.int32), tg, agg, 0.01, 1e9, 1000)
    assert [o.evictions for o in plan.layers] == [list(map(int, r)) for r in want["evictions"]]
    assert [o.loads for o in plan.layers] == [list(map(int, r)) for r in want["loads"]]
    assert plan.delta_e == want["delta_e"] and plan.total_loads == want["total_loads"]
    assert [o.duration for o in plan.layers] == list(want["duration"])


def test_plan_loading_frozen():
    """test_expert_store.cpp:174-209 and :352-364"""
    s = shape(2, 6, 1)
    cur = emoe.Placement.empty(s, [4, 4])
    for e in (0, 1, 2):
        cur.load(0, e)
        cur.load(1, e)
    cost = emoe.CostModel(per_expert_transfer=0.1, hd_bandwidth=1e18)
    plan = emoe.plan_loading(cur, [[3, 4, 5], [0, 1, 3]], np.array([[0, 0, 0, 9, 8, 7], [5, 5, 5, 6, 0, 0]]), cost)
    assert abs(plan.delta_e - 0.4) < 1e-12 and plan.total_loads == 4
    assert plan.layers[0].evictions == [0, 1, 2] and plan.layers[0].loads == [3, 4, 5]
    assert plan.layers[1].evictions == [2] and plan.layers[1].loads == [3]
    assert emoe.plan_loading(cur, [[0, 1, 2], [0, 1, 2]], np.zeros((2, 6)), cost).empty()
    with pytest.raises(emoe.ValidationError):
        emoe.plan_loading(cur, [[0, 1, 2, 3, 4], [0]], np.zeros((2, 6)), cost)
    emoe.apply_plan(cur, plan)
    assert cur.residents(0) == [3, 4, 5] and cur.residents(1) == [0, 1, 3]
    assert emoe.select_experts(np.array([[10, 40, 40, 5]]), shape(1, 4, 1), [2]) == [[1, 2]]
    assert emoe.select_experts(np.zeros((1, 4)), shape(1, 4, 1), [2]) == [[0, 1]]
    with pytest.raises(emoe.ValidationError):
        emoe.select_experts(np.zeros((1, 4)), shape(1, 4, 1), [5])


# ---------------- full engine invocation ----------------
@pytest.mark.parametrize("mode", [0, 1])
def test_invocation_matches_oracle_chain(mode, ref, port):
    """engine.cpp:367-446 on the GPU vs the same chain through the reference
    pieces (predict + predicted_frequencies) and the oracle's engine restatement."""
    m, E, k = 4, 8, 2
    tr = ref.gen_routing_trace(m, E, k, 0.6, 0.8, 0, 17, 60, 32)
    names = ["cls", "conv"]
    tids = [names[p % 2] for p in range(50)]
    model = emoe.fit(tr[:50], tids, 0.01, E)
    _, sets = emoe.prompt_expert_sets(tr, 49)
    arr, sizes = emoe.moesim._sets_array(sets if mode == 0 else sets[:1], k)
    r = dict(layer_counts=model.layer_counts, prompt_counts=model.prompt_counts, smoothing=0.01)
    scores, _, _ = ref.predict(r, mode, arr, sizes, k=k)
    fitted = np.stack([ref.predicted_frequencies(model.task_counts, names, 0.01, n) for n in names])
    wo = np.array([32.0, 200.0])
    sens = np.array([[0, 0, 0, 0], [1, 1, 1, 1]], np.int32)
    has = np.array([1, 1], np.uint8)
    req_task = np.array([0, 1, 1, 0, 1], np.int32)
    req_tok = np.array([100, 2000, 300, 50, 800], np.int32)
    want_agg = port.invocation_aggregate(scores, fitted, wo, sens, has, req_task, req_tok, True)
    resident = np.zeros((m, E), np.uint8)
    resident[:, :4] = 1
    budgets = np.full(m, 4, np.int32)
    targets = ref.loading_targets(want_agg, resident, budgets)
    want_plan = ref.plan_loading(resident, np.full(m, E, np.int32), targets, want_agg, 0.5, 1e18, 1)

    pred = emoe.moesim._Pred.from_model(model)
    agg = np.zeros((m, E))
    ev = np.full((m, E), -1, np.int32)
    ld = np.full((m, E), -1, np.int32)
    ne = np.zeros(m, np.int32)
    nl = np.zeros(m, np.int32)
    de = np.zeros(1)
    p = emoe.moesim._p
    emoe.moesim.check(emoe._lib.lib.emoe_invocation_host(pred.h, mode, p(arr), p(sizes), 2, p(wo), p(sens), p(has), 5,
                                                         p(req_task), p(req_tok), 1, p(resident), p(budgets), 0.5,
                                                         p(agg), p(ev), p(ne), p(ld), p(nl), p(de)))
    assert np.array_equal(agg, want_agg)
    assert [list(ev[l, : ne[l]]) for l in range(m)] == [list(x) for x in want_plan["evictions"]]
    assert [list(ld[l, : nl[l]]) for l in range(m)] == [list(x) for x in want_plan["loads"]]
    assert de[0] == want_plan["delta_e"]


def test_gpu_predictor_matches_golden():
    """GPU fit / sets / predictions / frequencies vs the reference's golden fixtures."""
    import json
    from pathlib import Path

    gold = json.loads((Path(__file__).parent / "golden" / "reference_golden.json").read_text())
    for t, f in zip(gold["gen_routing_trace"], gold["fit"]):
        tr = np.array(t["trace"], np.int32)
        P, m, T, k = tr.shape
        model = emoe.fit(tr, ["a" if p % 2 == 0 else "b" for p in range(P)], 0.01, f["E"])
        assert np.array_equal(model.layer_counts.reshape(-1), np.array(f["layer_counts"]).reshape(-1))
        assert np.array_equal(model.prompt_counts, np.array(f["prompt_counts"]))
        assert np.array_equal(model.task_counts, np.array(f["task_counts"]))
        for p in range(P):
            dom, sets = emoe.prompt_expert_sets(tr, p)
            assert dom == f["dominant"][p]
            assert sets == [f["sets"][p][l][: f["set_sizes"][p][l]] for l in range(m)]
        _, sets = emoe.prompt_expert_sets(tr, P - 1)
        a = emoe.predict_all_layers(model, sets)
        want = f["predictions"]["0"]
        for l in range(m):
            assert a[l].experts == want["experts"][l][: want["n"][l]]
            assert np.array_equal(a[l].scores, np.array(want["scores"][l]))
        for name in ["a", "b", "zz"]:
            assert np.array_equal(emoe.predicted_frequencies(model, name), np.array(f["frequencies"][name]))
    for r in gold["route_token"]:
        ex, rk, hit = emoe.route_tokens(np.array(r["choices"]), np.array(r["resident"]), np.array(r["scores"]))
        assert ex.tolist() == r["expert"] and rk.tolist() == r["rank"] and hit.tolist() == r["hit"]
