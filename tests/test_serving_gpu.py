"""The serving loop on the GPU (predictor every p prompts, task-aware skip,
layer-sequential side-stream loads) against the oracle's restatement of the
engine's invocation chain (engine.cpp:320-323, 367-464)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_stream_invocations_and_residency_match_oracle(port, ref):
    from helpers import trace_logits
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig, TaskSpec, run_stream

    m, E, k, L, d, f, T, p = 4, 8, 2, 4, 256, 512, 256, 4
    tasks = {"cls": TaskSpec(8.0, [0] * m), "conv": TaskSpec(32.0, [1] * m)}
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=T, period=p, mode=0, tasks=tasks)
    P_train, P_serve = 30, 16
    trace = ref.gen_routing_trace(m, E, k, 0.6, 0.8, 0, 17, P_train + P_serve, T)
    train_tasks = ["conv" if q % 3 else "cls" for q in range(P_train)]
    serve_tasks = ["conv", "cls", "conv", "conv", "cls", "cls", "cls", "cls",
                   "cls", "conv", "cls", "cls", "conv", "conv", "conv", "cls"]
    prompt_tasks = train_tasks + serve_tasks
    g = torch.Generator().manual_seed(3)
    host = [tuple((torch.randn(*s, generator=g) / s[1] ** 0.5).to(torch.bfloat16).pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    gates = [(torch.randn(E, d, generator=g) / d ** 0.5).to(torch.bfloat16) for _ in range(m)]
    stack = MoEStack(cfg, host, gates)
    trace_dev = torch.from_numpy(trace).cuda()
    stack.fit(trace_dev[:P_train].contiguous(), train_tasks)
    for layer in stack.layers:
        layer.load_initial(range(L))
    logits = {q: torch.from_numpy(np.stack([trace_logits(trace[q, l], E, seed=q * 31 + l) for l in range(m)])).cuda()
              for q in range(P_train, P_train + P_serve)}
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    st = run_stream(stack, trace, trace_dev, prompt_tasks, x, lambda q: logits[q], P_train, P_serve)
    assert st["fired_at"] == [0, 8, 12] and st["skipped_at"] == [4], st

    # oracle replay of the engine's invocation chain
    names = sorted(tasks)
    model = port.fit(trace[:P_train], np.array([names.index(t) for t in train_tasks], np.int32), len(names), E)
    model["smoothing"] = 0.01
    fitted = np.stack([port.predicted_frequencies(model["task_counts"], 0.01, i) for i in range(len(names))])
    resident = np.zeros((m, E), np.uint8)
    resident[:, :L] = 1
    wo = np.array([tasks[n].wo for n in names])
    sens = np.array([tasks[n].sensitivity for n in names], np.int32)
    for i in st["fired_at"]:
        q = P_train + i
        sets, sizes = port.prompt_expert_sets(trace, q - 1)
        scores, _, _ = port.predict(model, 0, sets, sizes, k=k)
        window = list(range(q, min(q + p, P_train + P_serve)))
        agg = port.invocation_aggregate(scores, fitted, wo, sens, np.ones(2, np.uint8),
                                        [names.index(prompt_tasks[w]) for w in window], [T] * len(window), True)
        targets = port.loading_targets(agg, resident, [L] * m)
        resident = np.zeros((m, E), np.uint8)
        for l in range(m):
            resident[l, targets[l]] = 1
    got = np.stack([layer.residency() for layer in stack.layers])
    assert np.array_equal(got, resident)
    assert st["planned_loads"] > 0 and 0.0 < st["hit_rate"] <= 1.0
    # route_token's fallback (no gate choice resident) takes the resident expert
    # with the highest score of the last invocation's aggregate
    # (engine.cpp:424, :529-532): every layer's routing of the last prompt
    # against the reference route_token with those scores, fallback tokens included
    q = P_train + P_serve - 1
    n_fallback = 0
    for l, layer in enumerate(stack.layers):
        layer.forward(x, logits=logits[q][l])
        ws = layer.workspace()
        ex, rk, hit = ref.route_tokens(trace[q, l], resident[l], scores=agg[l])
        assert np.array_equal(ws["route_expert"].cpu().numpy(), ex), f"layer {l}: route_token expert"
        assert np.array_equal(ws["route_rank"].cpu().numpy(), rk), f"layer {l}: route_token rank"
        n_fallback += int((rk == -1).sum())
    assert n_fallback > 0, "no fallback token in the check"
    stack.close()


def _engine_dynamic_replay(trace, first, n, m, E, L, resident):
    """engine.cpp:469-497 dynamic_transfers, restated for prompt batches: per layer,
    demand = tokens per rank-0 choice; keep the top-L by demand (map order breaks
    ties); evict the rest; load the missing.  Returns residency and load count."""
    loads = 0
    hits = 0
    for q in range(first, first + n):
        for l in range(m):
            demand = np.bincount(trace[q, l, :, 0], minlength=E)
            ranked = sorted([e for e in range(E) if demand[e] > 0], key=lambda e: (-demand[e], e))[:L]
            loads += sum(1 for e in ranked if not resident[l, e])
            resident[l] = 0
            resident[l, ranked] = 1
            hits += int(resident[l, trace[q, l, :, 0]].sum())
    return resident, loads, hits


def test_dynamic_residency_matches_engine_replay(ref):
    from helpers import trace_logits
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig, TaskSpec, run_stream

    m, E, k, L, d, f, T = 3, 8, 2, 3, 256, 512, 512
    tasks = {"conv": TaskSpec(32.0, [1] * m)}
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=T, period=4, mode=0, tasks=tasks)
    P = 6
    trace = ref.gen_routing_trace(m, E, k, 0.3, 0.3, 0, 23, P, T)
    g = torch.Generator().manual_seed(5)
    host = [tuple((torch.randn(*s, generator=g) / s[1] ** 0.5).to(torch.bfloat16).pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    gates = [torch.zeros(E, d, dtype=torch.bfloat16) for _ in range(m)]
    stack = MoEStack(cfg, host, gates)
    for layer in stack.layers:
        layer.load_initial(range(L))
    logits = {q: torch.from_numpy(np.stack([trace_logits(trace[q, l], E, seed=q * 7 + l) for l in range(m)])).cuda()
              for q in range(P)}
    # the demand map read back from the GPU route is the rank-0 histogram of the trace
    stack.layers[0].route(logits=logits[0][0])
    assert np.array_equal(stack.layers[0].gate_demand(), np.bincount(trace[0, 0, :, 0], minlength=E))
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    st = run_stream(stack, trace, None, ["conv"] * P, x, lambda q: logits[q], 0, P, residency="dynamic")
    resident = np.zeros((m, E), np.uint8)
    resident[:, :L] = 1
    want, loads, hits = _engine_dynamic_replay(trace, 0, P, m, E, L, resident)
    got = np.stack([layer.residency() for layer in stack.layers])
    assert np.array_equal(got, want)
    assert st["planned_loads"] == loads
    assert st["hit_rate"] == pytest.approx(hits / (P * T * m), abs=0)
    stack.close()


def test_profile_cost_model_is_a_valid_reference_cost(ref):
    """The measured CostModel satisfies CostModel::validate (types.cpp:7-14) and
    leaves the stack's residency untouched."""
    from helpers import trace_logits
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig, TaskSpec, profile_cost_model

    m, E, k, L, d, f, T = 3, 8, 2, 4, 256, 512, 512
    tasks = {"conv": TaskSpec(32.0, [1] * m)}
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=T, period=4, mode=0, tasks=tasks)
    trace = ref.gen_routing_trace(m, E, k, 0.6, 0.8, 0, 17, 12, T)
    g = torch.Generator().manual_seed(9)
    host = [tuple((torch.randn(*s, generator=g) / s[1] ** 0.5).to(torch.bfloat16).pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    stack = MoEStack(cfg, host, [torch.zeros(E, d, dtype=torch.bfloat16) for _ in range(m)])
    trace_dev = torch.from_numpy(trace).cuda()
    stack.fit(trace_dev[:10].contiguous(), ["conv"] * 10)
    for layer in stack.layers:
        layer.load_initial(range(L))
    before = np.stack([layer.residency() for layer in stack.layers])
    lg = torch.from_numpy(np.stack([trace_logits(trace[11, l], E, seed=l) for l in range(m)])).cuda()
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    cost = profile_cost_model(stack, x, lg, [[0, 1]] * m, [("conv", T)] * 4, reps=2)
    assert cost["per_token_cost"] > 0 and cost["per_expert_transfer"] > 0 and cost["hd_bandwidth"] > 1e9
    assert cost["predictor_invocation_cost"] > 0 and cost["contention_factor"] >= 1.0
    assert np.array_equal(np.stack([layer.residency() for layer in stack.layers]), before)
    stack.close()


def test_stack_shared_workspace_bit_identical():
    """A stack whose layers share one workspace (the default) computes the
    same outputs, layer by layer, as one with a workspace per layer; a layer
    chain (y of layer l feeds layer l+1) exercises the reuse."""
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig

    m, E, k, L, d, f, T = 3, 8, 2, 4, 256, 512, 700
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=1024, period=4, mode=0, tasks={})
    g = torch.Generator().manual_seed(9)
    host = [tuple((torch.randn(*s, generator=g) / s[1] ** 0.5).to(torch.bfloat16).pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    gates = [(torch.randn(E, d, generator=g) / d ** 0.5).to(torch.bfloat16) for _ in range(m)]
    x = torch.randn(T, d, generator=g).to(torch.bfloat16).cuda()
    outs = []
    for share in (True, False):
        stack = MoEStack(cfg, host, gates, share_workspace=share)
        for l, layer in enumerate(stack.layers):
            layer.load_initial([(l + j) % E for j in range(L)])
        h, ys = x, []
        for layer in stack.layers:
            h = layer.forward(h)
            ys.append(h.clone())
        torch.cuda.synchronize()
        outs.append(ys)
        stack.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
