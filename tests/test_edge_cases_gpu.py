"""Edge cases of the forward against the oracle: ragged and tiny token counts,
every token on one expert, k = E, a single expert, a single resident expert
(everything falls back), many experts."""
import numpy as np
import pytest
import torch

from helpers import assert_bf16_close, build_layer, to_f32, trace_logits

pytestmark = pytest.mark.gpu


def check(layer, x, experts, port, logits=None, scores=None, wm=0, act=0):
    y = layer.forward(x.cuda(), logits=None if logits is None else torch.from_numpy(logits).cuda())
    torch.cuda.synchronize()
    ws = layer.workspace()
    T = x.shape[0]
    E, k = layer.E, layer.k
    lg = to_f32(ws["logits"])
    o = port.gate_route(lg, k, wm, layer.residency(), scores)
    served = ws["served_idx"].cpu().numpy()
    assert np.array_equal(served, o["served_idx"])
    assert np.array_equal(ws["route_expert"].cpu().numpy(), o["route_expert"])
    counts, offsets, pos, src = port.permute(served, E, layer.seg_pad)
    assert np.array_equal(ws["counts"].cpu().numpy(), counts)
    assert np.array_equal(ws["pos"].cpu().numpy().astype(np.int64), pos)
    x32 = to_f32(x)
    yref = np.zeros((T, x.shape[1]), np.float32)
    for e in range(E):
        rows = np.flatnonzero((served == e).any(axis=1))
        if rows.size == 0:
            continue
        w1, w3, w2 = (None if w is None else to_f32(w) for w in experts[e])
        ye = port.expert_ffn(x32[rows], w1, w3, w2, act, True)
        for i, t in enumerate(rows):
            j = int(np.flatnonzero(served[t] == e)[0])
            yref[t] += np.float32(o["served_w"][t, j]) * ye[i]
    from oracle.oracle import bf16_round

    assert_bf16_close(to_f32(y), bf16_round(yref), "edge forward")


@pytest.mark.parametrize("T", [1, 127, 129, 255])
def test_ragged_token_counts(T, port):
    layer, _, experts = build_layer(8, 256, 512, 2, slots=4, resident=[0, 1, 4, 6], max_tokens=512)
    x = torch.randn(T, 256, generator=torch.Generator().manual_seed(T)).to(torch.bfloat16)
    check(layer, x, experts, port)
    layer.close()


def test_all_tokens_one_expert(port):
    layer, _, experts = build_layer(8, 256, 512, 2, slots=4, resident=[1, 2, 3, 5], max_tokens=3000)
    T = 3000
    choices = np.tile(np.array([[3, 6]], np.int32), (T, 1))  # rank 0 resident, rank 1 not
    x = torch.randn(T, 256, generator=torch.Generator().manual_seed(1)).to(torch.bfloat16)
    check(layer, x, experts, port, logits=trace_logits(choices, 8))
    assert layer.workspace()["counts"].cpu().tolist() == [0, 0, 0, T, 0, 0, 0, 0]
    layer.close()


def test_k_equals_E_and_single_expert(port):
    layer, _, experts = build_layer(4, 256, 256, 4, slots=4, max_tokens=600)  # k = E = 4
    x = torch.randn(600, 256, generator=torch.Generator().manual_seed(2)).to(torch.bfloat16)
    check(layer, x, experts, port)
    layer.close()
    layer, _, experts = build_layer(1, 256, 256, 1, slots=1, max_tokens=300)  # E = k = 1
    x = torch.randn(300, 256, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16)
    check(layer, x, experts, port)
    layer.close()


def test_single_resident_everything_falls_back(port):
    layer, _, experts = build_layer(8, 256, 512, 2, slots=1, resident=[5], max_tokens=1000)
    scores = np.linspace(1, 0, 8)
    layer.set_scores(scores)
    x = torch.randn(1000, 256, generator=torch.Generator().manual_seed(4)).to(torch.bfloat16)
    check(layer, x, experts, port, scores=scores)
    ws = layer.workspace()
    assert (ws["route_expert"] == 5).all()
    layer.close()


def test_many_experts_switch_shape(port):
    E = 128
    res = list(range(0, 128, 5))  # 26 resident, like Switch-base-128 at phi = 0.2
    layer, _, experts = build_layer(E, 256, 512, 1, act="relu", weight_mode="full_softmax", slots=len(res),
                                    resident=res, max_tokens=5000)
    x = torch.randn(5000, 256, generator=torch.Generator().manual_seed(5)).to(torch.bfloat16)
    check(layer, x, experts, port, wm=1, act=1)
    layer.close()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_stage_api_equals_forward(dtype, port):
    """The expert-parallel stage entry points (emoe_route_permute ->
    emoe_ffn_segments on caller rows -> emoe_combine) reproduce the fused
    forward bit for bit -- for fp32 this runs the 3xTF32 GEMMs on caller
    rows through their own split scratch."""
    import torch

    E, d, f, k, T = 8, 256, 512, 2, 900
    layer, _, _ = build_layer(E, d, f, k, dtype, "swiglu", "topk_softmax", 4, [1, 2, 5, 6], max_tokens=1024)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(21)).to(td).cuda()
    y_ref = layer.forward(x).clone()
    layer.route_permute(x)
    ws = layer.workspace()
    seg = ws["seg_offsets"].clone()
    R = int(seg[-1].item())
    rows = ws["x_perm"][:R].clone()
    h = torch.empty(R, f, dtype=td, device="cuda")
    y_rows = torch.empty(R, d, dtype=td, device="cuda")
    layer.ffn_segments(rows, seg, torch.arange(E, dtype=torch.int32, device="cuda"), h, y_rows)
    y = torch.empty_like(x)
    layer.combine(y_rows, ws["pos"], ws["served_w"], y)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    layer.close()


def _near_tie_logits(T, E, seed):
    """Rows built to stress top-k tie-breaking (ascending index on equal
    logits): all equal, a tie at the top, a tie straddling the k-th place,
    neighbours one ulp apart, quantised values with many ties, +0 / -0."""
    rng = np.random.default_rng(seed)
    L = np.empty((T, E), np.float32)
    for t in range(T):
        kind = t % 6
        if kind == 0:
            L[t] = np.float32(rng.normal())
        elif kind == 1:
            L[t] = rng.normal(size=E).astype(np.float32) - 4
            a, b = rng.choice(E, 2, replace=False)
            L[t, a] = L[t, b] = np.float32(2.5)
        elif kind == 2:
            L[t] = np.float32(-1)
            top = rng.choice(E, 3, replace=False)
            L[t, top[0]] = 3
            L[t, top[1:]] = 1  # two equal candidates for the next place
        elif kind == 3:
            base = np.float32(rng.normal())
            L[t] = base
            for j, e in enumerate(rng.permutation(E)[:4]):  # 1-ulp ladder above the rest
                v = base
                for _ in range(j + 1):
                    v = np.nextafter(v, np.float32(np.inf), dtype=np.float32)
                L[t, e] = v
        elif kind == 4:
            L[t] = (np.round(rng.normal(size=E) * 2) / 2).astype(np.float32)
        else:
            L[t] = np.where(rng.random(E) < 0.5, np.float32(0.0), np.float32(-0.0))
    return L


@pytest.mark.parametrize("E,k,wm", [(8, 2, 0), (8, 1, 1), (32, 2, 0)])
def test_near_tie_logits_given(E, k, wm, port):
    """Routing-driven logits with exact ties and one-ulp gaps: top-k and the
    served set bit-exact against the oracle, weights to the expf tolerance."""
    T = 600
    res = list(range(0, E, 2))
    layer, _, experts = build_layer(E, 256, 256, k, act="swiglu" if k > 1 else "relu",
                                    weight_mode="topk_softmax" if wm == 0 else "full_softmax", slots=len(res),
                                    resident=res, max_tokens=T)
    L = _near_tie_logits(T, E, 17 + E + k)
    x = torch.randn(T, 256, generator=torch.Generator().manual_seed(6)).to(torch.bfloat16)
    layer.forward(x.cuda(), logits=torch.from_numpy(L).cuda())
    torch.cuda.synchronize()
    ws = layer.workspace()
    o = port.gate_route(L, k, wm, layer.residency(), None)
    assert np.array_equal(ws["topk_idx"].cpu().numpy(), o["topk_idx"])
    assert np.array_equal(ws["served_idx"].cpu().numpy(), o["served_idx"])
    # weights: device expf vs the C library's (a few ulp), as in test_forward_gpu
    np.testing.assert_allclose(ws["served_w"].cpu().numpy(), o["served_w"], rtol=2e-6, atol=1e-7)
    layer.close()


def test_near_tie_logits_fused_tc_gate(port):
    """The fused tcgen05 gate + route (E = 128, top-1, full-softmax weights):
    x = 0 makes the gate's logits exactly 0, so in logits-bias mode the
    routed logits are exactly the near-tie bias rows -- routing bit-exact
    against the oracle on them, weights to the expf tolerance."""
    E, T = 128, 1536
    res = list(range(0, 128, 5))
    layer, _, _ = build_layer(E, 256, 512, 1, act="relu", weight_mode="full_softmax", slots=len(res), resident=res,
                              max_tokens=T)
    layer.set_logits_mode("add")
    L = _near_tie_logits(T, E, 99)
    x = torch.zeros(T, 256, dtype=torch.bfloat16)
    layer.forward(x.cuda(), logits=torch.from_numpy(L).cuda())
    torch.cuda.synchronize()
    ws = layer.workspace()
    o = port.gate_route(L + np.float32(0.0), 1, 1, layer.residency(), None)
    assert np.array_equal(ws["topk_idx"].cpu().numpy(), o["topk_idx"])
    assert np.array_equal(ws["served_idx"].cpu().numpy(), o["served_idx"])
    # weights: device expf vs the C library's (a few ulp), as in test_forward_gpu
    np.testing.assert_allclose(ws["served_w"].cpu().numpy(), o["served_w"], rtol=2e-6, atol=1e-7)
    layer.close()
