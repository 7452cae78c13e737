"""Output parity for configs 4 and 5 at their full layer shape (Mixtral:
d = 4096, f = 14336, E = 8, top-2), on sampled tokens against the CPU oracle.

  * config 4: two chained layers of a stack on one shared workspace, T =
    65,536 tokens; layer 1's input is layer 0's output.  Layer 1's routing of
    every token bit-exact given its GPU logits, its permutation bit-exact,
    and sampled tokens of its output within the bf16 tolerance of the oracle
    chain (gate weights, expert weights and residency of that layer).
  * config 5: the serving loop (predictor invocations, task-aware skip,
    side-stream expert loads) over 8k-token prompts; afterwards every
    layer's forward of the last prompt on sampled tokens against the oracle
    with the weights the side stream loaded into the slots.
The 32-layer stack and the 80-prompt stream differ from these only in the
number of layers / prompts: each layer is the same code on the same shared
workspace.
"""
import numpy as np
import pytest
import torch

from helpers import assert_bf16_close, to_f32, trace_logits

pytestmark = pytest.mark.gpu

E, K, D, F = 8, 2, 4096, 14336


def host_experts(seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [tuple((torch.randn(*s, generator=g, device="cuda") / s[1] ** 0.5).to(torch.bfloat16).cpu().pin_memory()
                  for s in ((F, D), (F, D), (D, F))) for _ in range(E)]


def check_layer_tokens(port, layer, x_in, y_out, wg, host, n_tok, seed, what, logits_bias=None, scores=None):
    """Routing / permutation of every token bit-exact and n_tok sampled output
    tokens within tolerance, for one forward of `layer` (x_in -> y_out)."""
    from oracle.oracle import bf16_round

    T = x_in.shape[0]
    ws = layer.workspace()
    res = layer.residency()
    lg = to_f32(ws["logits"])
    rng = np.random.default_rng(seed)
    sample = rng.choice(T, 128, replace=False)
    ref_lg = port.gate_logits(to_f32(x_in[torch.from_numpy(sample).cuda()]), to_f32(wg))
    if logits_bias is not None:
        ref_lg = ref_lg + to_f32(logits_bias[torch.from_numpy(sample).cuda()])
    assert np.abs(lg[sample] - ref_lg).max() / np.abs(ref_lg).max() < 1e-4, f"{what}: gate logits"
    o = port.gate_route(lg, K, 0, res, scores)
    served = ws["served_idx"].cpu().numpy()
    assert np.array_equal(served, o["served_idx"]), f"{what}: routing"
    counts, offsets, pos, src = port.permute(served, E, layer.seg_pad)
    assert np.array_equal(ws["pos"].cpu().numpy().astype(np.int64), pos), f"{what}: permutation"
    toks = rng.choice(T, n_tok, replace=False)
    xs = to_f32(x_in[torch.from_numpy(toks).cuda()])
    yref = np.zeros((n_tok, D), np.float32)
    for e in np.unique(served[toks][served[toks] >= 0]):
        w1, w3, w2 = (to_f32(w) for w in host[int(e)])
        sel = [(i, j) for i, t in enumerate(toks) for j in range(K) if served[t, j] == e]
        ye = port.expert_ffn(xs[[i for i, _ in sel]], w1, w3, w2, 0, True)
        for r, (i, j) in enumerate(sel):
            yref[i] += np.float32(o["served_w"][toks[i], j]) * ye[r]
    return assert_bf16_close(to_f32(y_out[torch.from_numpy(toks).cuda()]), bf16_round(yref), what)


def test_config4_stack_layer_full_shape(port):
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig

    T = 65536
    host = host_experts(1234)
    g = torch.Generator(device="cuda").manual_seed(99)
    gates = [(torch.randn(E, D, generator=g, device="cuda") / D ** 0.5).to(torch.bfloat16) for _ in range(2)]
    cfg = StreamConfig(m=2, E=E, k=K, L=4, d=D, f=F, tokens_per_prompt=T, period=40, mode=0, tasks={})
    stack = MoEStack(cfg, host, gates)
    stack.layers[0].load_initial([0, 5, 6, 7])
    stack.layers[1].load_initial([1, 2, 4, 6])
    x = torch.randn(T, D, generator=g, device="cuda").to(torch.bfloat16)
    h0 = stack.layers[0].forward(x)
    h1 = stack.layers[1].forward(h0)  # shares layer 0's workspace
    torch.cuda.synchronize()
    norm, mx = check_layer_tokens(port, stack.layers[1], h0, h1, gates[1], host, 16, 7, "stack layer 1")
    print(f"\nconfig 4 stack layer 1 (T={T}): sampled tokens norm {norm:.2e} max {mx:.2e}")
    stack.close()


def test_config5_stream_full_shape(port, ref):
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig, TaskSpec, run_stream

    m, T, p = 2, 8192, 2
    tasks = {"cls": TaskSpec(16.0, [0] * m), "conv": TaskSpec(256.0, [1] * m)}
    cfg = StreamConfig(m=m, E=E, k=K, L=4, d=D, f=F, tokens_per_prompt=T, period=p, mode=0, tasks=tasks)
    P_train, P_serve = 12, 6
    trace = ref.gen_routing_trace(m, E, K, 0.6, 0.8, 0, 17, P_train + P_serve, T)
    prompt_tasks = ["conv" if q % 3 else "cls" for q in range(P_train + P_serve)]
    host = host_experts(4321)
    g = torch.Generator(device="cuda").manual_seed(5)
    gates = [(torch.randn(E, D, generator=g, device="cuda") / D ** 0.5).to(torch.bfloat16) for _ in range(m)]
    stack = MoEStack(cfg, host, gates)
    for layer in stack.layers:
        layer.load_initial(range(4))
        layer.set_logits_mode("add")  # the gate runs; the trace is a dominant bias
    trace_dev = torch.from_numpy(trace).cuda()
    stack.fit(trace_dev[:P_train].contiguous(), prompt_tasks[:P_train])
    logits = {q: torch.from_numpy(np.stack([trace_logits(trace[q, l], E, seed=q * 31 + l) * 16
                                            for l in range(m)])).cuda() for q in range(P_train, P_train + P_serve)}
    x = torch.randn(T, D, generator=g, device="cuda").to(torch.bfloat16)
    st = run_stream(stack, trace, trace_dev, prompt_tasks, x, lambda q: logits[q], P_train, P_serve)
    assert st["invocations"] >= 1 and st["planned_loads"] >= 1, st
    for layer in stack.layers:
        layer.poll_loads(blocking=True)
    q = P_train + P_serve - 1
    h = x
    for l, layer in enumerate(stack.layers):
        y = layer.forward(h, logits=logits[q][l])
        torch.cuda.synchronize()
        scores = getattr(stack, "scores", None)  # the last invocation's aggregate: route_token's fallback
        norm, mx = check_layer_tokens(port, layer, h, y, gates[l], host, 12, 11 + l, f"stream layer {l}",
                                      logits_bias=logits[q][l], scores=None if scores is None else scores[l])
        print(f"\nconfig 5 stream layer {l} (T={T}, resident {np.flatnonzero(layer.residency()).tolist()}): "
              f"sampled tokens norm {norm:.2e} max {mx:.2e}")
        h = y.clone()
    stack.close()
