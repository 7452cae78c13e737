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
