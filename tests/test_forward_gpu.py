"""GPU parity of the MoE layer forward (A1-A5) against the CPU oracle.

Each stage is checked on the same inputs:
  A1 gate logits (fp32 accumulate) vs oracle_gate_logits_f32   (tolerance)
  A1+A2 top-k / route_token / served set given the GPU logits   (bit-exact)
  A3 counts / padded offsets / positions / row sources          (bit-exact)
     permuted rows == source rows                               (bit-exact)
  A4 expert FFN rows vs oracle_expert_ffn (mirrored rounding)   (tolerance)
  A5 combine vs oracle_combine of the GPU expert outputs        (tolerance)
  end to end: sampled tokens vs the full oracle chain           (tolerance)
"""
import numpy as np
import pytest
import torch

from helpers import (assert_bf16_close, assert_f32_close, build_layer, to_f32, trace_logits)

CASES = {
    # name: E, d, f, k, dtype, act, weight_mode, slots, resident, T, gemm_cta_group (0 = auto)
    "mixtral_small": (8, 512, 1024, 2, "bf16", "swiglu", "topk_softmax", 4, [1, 3, 4, 6], 1000, 0),
    "mixtral_small_cta1": (8, 512, 1024, 2, "bf16", "swiglu", "topk_softmax", 4, [1, 3, 4, 6], 1000, 1),
    "mixtral_full_resident": (8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 8, None, 640, 0),
    "switch_small": (32, 256, 512, 1, "bf16", "relu", "full_softmax", 8, [0, 2, 5, 7, 11, 19, 23, 31], 777, 0),
    "switch_small_cta2": (32, 256, 512, 1, "bf16", "relu", "full_softmax", 8, [0, 2, 5, 7, 11, 19, 23, 31], 777,
                          2),
    # K > 2048 in both GEMMs: the 4-epilogue-warp kernels (shorter K uses 8)
    "mixtral_longk": (8, 2304, 2304, 2, "bf16", "swiglu", "topk_softmax", 4, [0, 3, 4, 7], 600, 0),
    "mixtral_longk_cta2": (8, 2304, 2304, 2, "bf16", "swiglu", "topk_softmax", 4, [0, 3, 4, 7], 600, 2),
    "config1_fp32_phi05": (8, 1024, 3584, 2, "fp32", "swiglu", "topk_softmax", 4, [0, 2, 5, 7], 512, 0),
    "config1_fp32_phi1": (8, 1024, 3584, 2, "fp32", "swiglu", "topk_softmax", 8, None, 512, 0),
    "fp32_relu_top1": (16, 256, 512, 1, "fp32", "relu", "full_softmax", 8, [0, 2, 5, 7, 9, 11, 13, 15], 500, 0),
    # T >= 74 route blocks: the fused fp32 gate+route kernel (smaller T computes logits first)
    "fp32_many_tokens": (8, 256, 512, 2, "fp32", "swiglu", "topk_softmax", 4, [0, 2, 5, 7], 9600, 0),
}


def run_case(name, port, use_trace_logits=False, scores=None, logits_mode="replace"):
    E, d, f, k, dtype, act, wm, slots, resident, T, cg = CASES[name]
    layer, wg, experts = build_layer(E, d, f, k, dtype, act, wm, slots, resident, max_tokens=max(T, 128),
                                     gemm_cta_group=cg)
    layer.set_logits_mode(logits_mode)
    if scores is not None:
        layer.set_scores(scores)
    g = torch.Generator().manual_seed(7)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.randn(T, d, generator=g).to(td)
    xd = x.cuda()
    logits_in = None
    if use_trace_logits:
        crng = np.random.default_rng(3)
        choices = np.stack([crng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
        logits_in = torch.from_numpy(trace_logits(choices, E)).cuda()
        if logits_mode == "add":  # a bias that dominates the gate's own logits (~N(0, 1))
            logits_in = logits_in * 16
    y = layer.forward(xd, logits=logits_in)
    torch.cuda.synchronize()
    ws = {key: (None if v is None else v.clone()) for key, v in layer.workspace().items()}
    res = layer.residency()
    return dict(layer=layer, wg=wg, experts=experts, x=x, y=y, ws=ws, resident=res, T=T, E=E, d=d, f=f, k=k,
                dtype=dtype, act=act, wm=wm, logits_in=logits_in, logits_mode=logits_mode)


def check_case(c, port, scores=None):
    T, E, k, d, f = c["T"], c["E"], c["k"], c["d"], c["f"]
    ws = c["ws"]
    x32 = to_f32(c["x"])
    lg = to_f32(ws["logits"])
    # A1 logits
    if c["logits_in"] is None or c.get("logits_mode") == "add":
        ref_lg = port.gate_logits(x32, to_f32(c["wg"]))
        if c["logits_in"] is not None:  # logits-bias mode: the gate's logits + the caller's
            ref_lg = (ref_lg + to_f32(c["logits_in"])).astype(np.float32)
        err = np.abs(lg - ref_lg).max() / max(np.abs(ref_lg).max(), 1e-30)
        assert err < 1e-4, f"gate logits rel err {err:.3e}"
    else:
        assert np.array_equal(lg, to_f32(c["logits_in"]))
    # A1 + A2 on the GPU logits: bit-exact
    o = port.gate_route(lg, k, 0 if c["wm"] == "topk_softmax" else 1, c["resident"], scores)
    assert np.array_equal(to_f32(ws["topk_idx"]).astype(np.int32), o["topk_idx"])
    assert np.array_equal(ws["route_expert"].cpu().numpy(), o["route_expert"])
    assert np.array_equal(ws["route_rank"].cpu().numpy(), o["route_rank"])
    assert np.array_equal(ws["route_hit"].cpu().numpy(), o["route_hit"])
    served = ws["served_idx"].cpu().numpy()
    assert np.array_equal(served, o["served_idx"])
    np.testing.assert_allclose(ws["served_w"].cpu().numpy(), o["served_w"], rtol=2e-6, atol=1e-7)
    # A3 permutation: bit-exact
    counts, offsets, pos, src = port.permute(served, E, c["layer"].seg_pad)
    assert np.array_equal(ws["counts"].cpu().numpy(), counts)
    assert np.array_equal(ws["seg_offsets"].cpu().numpy(), offsets)
    assert np.array_equal(ws["pos"].cpu().numpy().astype(np.int64), pos)
    R = int(offsets[-1])
    assert np.array_equal(ws["row_token"][:R].cpu().numpy(), src)
    valid = np.flatnonzero(src >= 0)
    xp = ws["x_perm"][:R].cpu()
    assert torch.equal(xp[valid], c["x"][src[valid]]), "permuted rows differ from their source rows"
    # A4 expert FFN on sampled rows of every active expert (mirrored rounding)
    rng = np.random.default_rng(0)
    bf = c["dtype"] == "bf16"
    # fused combine (bf16, k <= 2): GEMM2's epilogue wrote y directly, so the
    # sampled rows are checked through their tokens in the end-to-end check
    fused = ws["y_perm"] is None
    yp = None if fused else to_f32(ws["y_perm"][:R])
    fused_toks = []
    for e in range(E):
        rows = np.arange(offsets[e], offsets[e] + counts[e])
        if rows.size == 0:
            continue
        pick = rng.choice(rows, size=min(12, rows.size), replace=False)
        if fused:
            fused_toks.extend(src[pick].tolist())
            continue
        w1, w3, w2 = (None if w is None else to_f32(w) for w in c["experts"][e])
        ref = port.expert_ffn(x32[src[pick]], w1, w3, w2, 0 if c["act"] == "swiglu" else 1, bf)
        (assert_bf16_close if bf else assert_f32_close)(yp[pick], ref, f"expert {e} FFN rows")
    # A5 combine of the GPU expert outputs
    if not fused:
        yc = port.combine(yp, pos, ws["served_w"].cpu().numpy(), bf)
        (assert_bf16_close if bf else assert_f32_close)(to_f32(c["y"]), yc, "combine")
    # end to end on sampled tokens: oracle FFN for each served slot + oracle combine
    toks = np.unique(np.concatenate([rng.choice(T, size=min(16, T), replace=False),
                                     np.asarray(fused_toks, np.int64)]).astype(np.int64))
    yref = np.zeros((toks.size, d), np.float32)
    for i, t in enumerate(toks):
        acc = np.zeros(d, np.float32)
        for j in range(k):
            e = served[t, j]
            if e < 0:
                continue
            w1, w3, w2 = (None if w is None else to_f32(w) for w in c["experts"][e])
            ye = port.expert_ffn(x32[t:t + 1], w1, w3, w2, 0 if c["act"] == "swiglu" else 1, bf)[0]
            acc += np.float32(o["served_w"][t, j]) * ye
        yref[i] = acc
    if bf:
        from oracle.oracle import bf16_round

        yref = bf16_round(yref)
        assert_bf16_close(to_f32(c["y"])[toks], yref, "end-to-end tokens")
    else:
        assert_f32_close(to_f32(c["y"])[toks], yref, "end-to-end tokens")


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_forward_parity(name, port):
    c = run_case(name, port)
    check_case(c, port)
    c["layer"].close()


@pytest.mark.gpu
def test_forward_trace_logits_and_fallback_scores(port):
    """Routing-driven mode (trace embedded as logits) with fallback scores set."""
    scores = np.linspace(0.1, 0.8, 8)[::-1].copy()
    c = run_case("mixtral_small", port, use_trace_logits=True, scores=scores)
    check_case(c, port, scores=scores)
    assert (c["ws"]["route_rank"].cpu().numpy() == -1).any(), "case should exercise the fallback path"
    c["layer"].close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mixtral_small", "switch_small", "config1_fp32_phi05", "fp32_relu_top1",
                                  "fp32_many_tokens"])
def test_forward_logits_bias_mode(name, port):
    """EMOE_LOGITS_ADD: the gate runs on x (every gate kernel: mma.sync E < 32,
    tcgen05 GEMM + route E >= 32, fp32 fused and logits-first) and the caller's
    logits are added before top-k; the trace bias dominates, so routing follows
    it while the gate's arithmetic is real."""
    c = run_case(name, port, use_trace_logits=True, logits_mode="add")
    check_case(c, port)
    E, k = c["E"], c["k"]
    choices = np.argsort(-to_f32(c["logits_in"]), axis=1, kind="stable")[:, :k]
    assert np.array_equal(c["ws"]["topk_idx"].cpu().numpy(), choices), "the bias should decide the routing"
    c["layer"].close()


@pytest.mark.gpu
def test_forward_deterministic(port):
    c1 = run_case("mixtral_small", port)
    y1 = c1["y"].clone()
    c1["layer"].close()
    c2 = run_case("mixtral_small", port)
    assert torch.equal(y1, c2["y"]), "forward is not bit-reproducible"
    c2["layer"].close()


@pytest.mark.gpu
def test_forward_host_pipelined_equals_device_forward():
    """The host-buffer API (chunked H2D / forward / D2H overlap) is bit-identical
    to one device forward over all tokens, and chunk boundaries do not leak."""
    from helpers import build_layer

    T = 20000  # 3 chunks of 8192
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 4, [0, 3, 5, 6], max_tokens=T)
    x = torch.randn(T, 256, generator=torch.Generator().manual_seed(21)).to(torch.bfloat16)
    y_dev = layer.forward(x.cuda()).cpu()
    y_host = torch.empty_like(x).pin_memory()
    layer.forward_host(x.pin_memory(), y_host)
    assert torch.equal(y_dev, y_host)
    layer.close()


@pytest.mark.gpu
def test_forced_miss_and_no_resident_error():
    """No resident expert: forced-miss layers serve nothing (y = 0, engine.cpp:533-537);
    otherwise the forward raises the reference's logic_error."""
    from paper_2503_06823_b200 import LogicError, MoELayer

    from helpers import make_weights

    wg, experts = make_weights(8, 256, 512, "bf16", "swiglu")
    for forced in (True, False):
        layer = MoELayer(256, 512, 8, 2, num_slots=4, max_tokens=256, forced_miss=forced)
        layer.set_gate(wg)
        x = torch.randn(256, 256).to(torch.bfloat16).cuda()
        if forced:
            y = layer.forward(x)
            torch.cuda.synchronize()
            assert torch.count_nonzero(y) == 0
            ws = layer.workspace()
            assert (ws["route_rank"] == -1).all() and (ws["served_idx"] == -1).all()
            assert torch.equal(ws["route_expert"], ws["topk_idx"][:, 0])
        else:
            with pytest.raises(LogicError):
                layer.forward(x)
        layer.close()


@pytest.mark.gpu
def test_two_phase_residency_and_loads():
    """Evictions apply at load start, loads at completion (engine.cpp:448-464);
    double loads / evictions / budget overflow raise like Placement (expert_store.cpp:46-57)."""
    from paper_2503_06823_b200 import LogicError

    from helpers import build_layer

    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 4, [0, 1, 2, 3], max_tokens=512)
    assert layer.residency().tolist() == [1, 1, 1, 1, 0, 0, 0, 0]
    with pytest.raises(LogicError):
        layer.begin_load([], [0])          # already resident
    with pytest.raises(LogicError):
        layer.begin_load([5], [])          # not resident
    with pytest.raises(LogicError):
        layer.begin_load([], [4])          # budget 4 exceeded
    layer.begin_load([1, 2], [6, 7])
    res = layer.residency()
    assert res[1] == 0 and res[2] == 0     # evictions visible immediately
    layer.poll_loads(blocking=True)
    assert layer.residency().tolist() == [1, 0, 0, 1, 0, 0, 1, 1]
    b, ms = layer.last_load_stats()
    assert b == 2 * 3 * 256 * 512 * 2 and ms > 0
    x = torch.randn(300, 256).to(torch.bfloat16).cuda()
    layer.forward(x)
    torch.cuda.synchronize()
    served = layer.workspace()["served_idx"].cpu().numpy()
    assert set(np.unique(served[served >= 0]).tolist()) <= {0, 3, 6, 7}
    layer.close()


@pytest.mark.gpu
def test_forward_host_async_pipelined_calls():
    """Back-to-back async host calls (alternating staging sets) give each call
    the same bits as a device forward of its own input."""
    from helpers import build_layer

    T = 9000
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 4, [1, 2, 5, 6], max_tokens=T)
    xs = [torch.randn(T, 256, generator=torch.Generator().manual_seed(40 + i)).to(torch.bfloat16).pin_memory()
          for i in range(3)]
    ys = [torch.empty_like(x).pin_memory() for x in xs]
    for x, y in zip(xs, ys):
        layer.forward_host_async(x, y)
    layer.wait_host()
    for x, y in zip(xs, ys):
        assert torch.equal(layer.forward(x.cuda()).cpu(), y)
    layer.close()


_FUSED_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import build_layer
E, d, f, cg, T = {args!r}
layer, _, _ = build_layer(E, d, f, 1, "bf16", "relu", "full_softmax", 8, [0, 2, 5, 7, 11, 19, 23, 31][:8],
                          max_tokens=T, gemm_cta_group=cg)
x = torch.randn(T, d, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
y = layer.forward(x)
torch.save(dict(y=y.cpu(), fused=layer.workspace()["y_perm"] is None), {out!r})
"""


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(32, 256, 512, 1, 777), (32, 256, 512, 2, 777), (32, 768, 1024, 2, 3001)])
def test_top1_fused_combine_bit_identical(args, tmp_path):
    """Top-1 layers: GEMM2's epilogue scattering w_t * Y_row into y (default)
    is bit-identical to GEMM2 + the separate combine (EMOE_FUSED_COMBINE=0)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    outs = []
    for flag in ("1", "0"):
        out = tmp_path / f"y{flag}.pt"
        code = _FUSED_SCRIPT.format(root=str(root), tests=str(root / "tests"), args=args, out=str(out))
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, EMOE_FUSED_COMBINE=flag),
                       timeout=300)
        outs.append(torch.load(out))
    assert outs[0]["fused"] and not outs[1]["fused"]
    assert torch.equal(outs[0]["y"], outs[1]["y"])


_FUSED2_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import build_layer
d, f, cg, T, resident = {args!r}
layer, _, _ = build_layer(8, d, f, 2, "bf16", "swiglu", "topk_softmax", len(resident), resident,
                          max_tokens=T, gemm_cta_group=cg)
ys = []
for i, n in enumerate((T, T // 3 + 5, T)):  # repeated forwards: the arrival counters re-zero themselves
    x = torch.randn(n, d, generator=torch.Generator().manual_seed(7 + i)).to(torch.bfloat16).cuda()
    ys.append(layer.forward(x).cpu())
torch.save(dict(ys=ys, fused=layer.workspace()["y_perm"] is None), {out!r})
"""


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(256, 512, 1, 777, [0, 2, 5, 7]), (256, 512, 2, 1500, [1, 6]),
                                  (768, 1024, 1, 3001, [0, 1, 2, 3, 4, 5, 6, 7]), (512, 768, 2, 2048, [3])])
def test_top2_fused_combine_bit_identical(args, tmp_path):
    """Top-2 layers: GEMM2's epilogue combining a token's two rows (the
    second to arrive reads the first's published row; EMOE_FUSED_COMBINE=2,
    opt-in) is bit-identical to GEMM2 + the separate combine
    (EMOE_FUSED_COMBINE=0), with single- and double-served tokens and across
    repeated forwards."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    outs = []
    for flag in ("2", "0"):
        out = tmp_path / f"y{flag}.pt"
        code = _FUSED2_SCRIPT.format(root=str(root), tests=str(root / "tests"), args=args, out=str(out))
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, EMOE_FUSED_COMBINE=flag),
                       timeout=300)
        outs.append(torch.load(out))
    assert outs[0]["fused"] and not outs[1]["fused"]
    for a, b in zip(outs[0]["ys"], outs[1]["ys"]):
        assert torch.equal(a, b)


_RASTER_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import build_layer
layer, _, _ = build_layer(8, 768, 2048, 2, "bf16", "swiglu", "topk_softmax", 4, [1, 3, 4, 6], max_tokens=3000,
                          gemm_cta_group={cg})
x = torch.randn(2999, 768, generator=torch.Generator().manual_seed(5)).to(torch.bfloat16).cuda()
torch.save(layer.forward(x).cpu(), {out!r})
"""


@pytest.mark.gpu
@pytest.mark.parametrize("cg", [1, 2])
def test_column_panel_raster_bit_identical(cg, tmp_path):
    """The tile order (row panels vs column panels with their L2 policies,
    the long-K GEMM2 default) never changes a tile's arithmetic: outputs are
    bit-identical across rasters."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    outs = []
    for env in ({"EMOE_GEMM1_NPANEL": "0", "EMOE_GEMM2_NPANEL": "0"},
                {"EMOE_GEMM1_NPANEL": "5", "EMOE_GEMM2_NPANEL": "1"}):
        out = tmp_path / f"y{len(outs)}.pt"
        code = _RASTER_SCRIPT.format(root=str(root), tests=str(root / "tests"), cg=cg, out=str(out))
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, **env), timeout=300)
        outs.append(torch.load(out))
    assert torch.equal(outs[0], outs[1])


_GATE_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import build_layer, to_f32
E, d, k, T, keep = {args!r}
res = list(range(0, E, 3))[: max(1, E // 5)]
layer, _, _ = build_layer(E, d, 512, k, "bf16", "relu" if k == 1 else "swiglu",
                          "full_softmax" if k == 1 else "topk_softmax", len(res), res, max_tokens=T)
layer.set_keep_logits(keep)
layer.set_scores([float((e * 37) % 11) for e in range(E)])
x = torch.randn(T, d, generator=torch.Generator().manual_seed(5)).to(torch.bfloat16).cuda()
y = layer.forward(x)
ws = layer.workspace()
out = {{key: ws[key].cpu() for key in ("topk_idx", "route_expert", "route_rank", "route_hit", "served_idx",
                                       "served_w", "pos", "counts")}}
out["y"] = y.cpu()
out["logits"] = ws["logits"].cpu() if keep else None
torch.save(out, {out_path!r})
"""


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(128, 768, 1, 65536), (128, 768, 1, 1000), (64, 512, 2, 3000), (32, 256, 1, 777),
                                  (96, 512, 2, 2500), (128, 1024, 1, 3000), (64, 2048, 2, 1300)])
def test_fused_gate_route_bit_identical(args, tmp_path):
    """E >= 32: the fused tcgen05 gate + route -- the CTA-pair form with the
    gate resident in shared memory (default where it fits) and the streaming
    form (EMOE_GATE_TC=stream), logits stored or not -- gives bit-identical
    routing, weights, permutation and outputs to the split path (dense gate
    GEMM -> logits -> route_from_logits_kernel, EMOE_GATE_ROUTE=split), and
    all store the same logits."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    E, d, k, T = args
    runs = {}
    for name, env, form, keep in (("split", "split", "", True), ("fused", "fused", "", True),
                                  ("fused_nolog", "fused", "", False), ("stream", "fused", "stream", True)):
        out = tmp_path / f"{name}.pt"
        code = _GATE_SCRIPT.format(root=str(root), tests=str(root / "tests"), args=(E, d, k, T, keep),
                                   out_path=str(out))
        subprocess.run([sys.executable, "-c", code], check=True,
                       env=dict(os.environ, EMOE_GATE_ROUTE=env, EMOE_GATE_TC=form), timeout=300)
        runs[name] = torch.load(out)
    assert torch.equal(runs["split"]["logits"], runs["fused"]["logits"])
    assert torch.equal(runs["split"]["logits"], runs["stream"]["logits"])
    for name in ("fused", "fused_nolog", "stream"):
        for key, v in runs["split"].items():
            if key != "logits":
                assert torch.equal(v, runs[name][key]), f"{name}: {key} differs from the split path"
    assert (runs["split"]["route_rank"] == -1).any(), "the case should exercise the fallback"


_BULK_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import build_layer
E, d, f, k, T, res, act = {args!r}
layer, _, _ = build_layer(E, d, f, k, "bf16", act, "topk_softmax" if k > 1 else "full_softmax", len(res), res,
                          max_tokens=T)
x = torch.randn(T, d, generator=torch.Generator().manual_seed(9)).to(torch.bfloat16).cuda()
y = layer.forward(x)
ws = layer.workspace()
R = int(ws["seg_offsets"][-1].item())
rt = ws["row_token"][:R].cpu()
xp = ws["x_perm"][:R].cpu()
torch.save(dict(y=y.cpu(), pos=ws["pos"].cpu(), row_token=rt, x_perm=xp[rt >= 0]), {out!r})
"""


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(8, 1024, 1024, 2, 40000, [0, 2, 5, 7], "swiglu"),
                                  (8, 4096, 1024, 2, 40000, [1, 3, 4, 6], "swiglu"),
                                  (32, 768, 1024, 1, 50000, [0, 3, 9, 17, 21, 30], "relu"),
                                  (8, 512, 512, 2, 38000, [3], "swiglu")])
def test_bulk_copy_permute_combine_bit_identical(args, tmp_path):
    """Large batches of long rows move them with cp.async.bulk
    (permute_bulk_kernel): positions, row sources, permuted rows and outputs
    bit-identical to the LDG/STG kernel (EMOE_BULK_COPY=0)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    outs = []
    for flag in ("1", "0"):
        out = tmp_path / f"b{flag}.pt"
        code = _BULK_SCRIPT.format(root=str(root), tests=str(root / "tests"), args=args, out=str(out))
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, EMOE_BULK_COPY=flag),
                       timeout=300)
        outs.append(torch.load(out))
    for key in outs[0]:
        assert torch.equal(outs[0][key], outs[1][key]), f"{key} differs between the bulk and LDG/STG paths"


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(8, 1024, 1024, 2, 5000, [0, 2, 5, 7], "swiglu"),
                                  (32, 768, 1024, 1, 6000, [0, 3, 9, 17, 21, 30], "relu"),
                                  (8, 2304, 2304, 2, 3000, [1, 3, 4, 6], "swiglu"),
                                  (8, 512, 512, 2, 777, [3], "swiglu")])
def test_gemm_weight_multicast_bit_identical(args, tmp_path):
    """EMOE_GEMM_MC=2 (1-CTA MMAs, each weight tile multicast over a 2-CTA
    cluster on adjacent row blocks, segments padded to 256 rows): positions
    change with the padding, but every token's output is bit-identical."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    outs = []
    for flag in ("2", "1"):
        out = tmp_path / f"mc{flag}.pt"
        code = _BULK_SCRIPT.replace("max_tokens=T)", "max_tokens=T, gemm_cta_group=1)").format(
            root=str(root), tests=str(root / "tests"), args=args, out=str(out))
        env = dict(os.environ, EMOE_GEMM_MC=flag)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
        outs.append(torch.load(out))
    assert torch.equal(outs[0]["y"], outs[1]["y"]), "outputs differ with the weight multicast"
    assert torch.equal(outs[0]["x_perm"], outs[1]["x_perm"])  # the same rows, in the same order


@pytest.mark.gpu
def test_tf32_both_cta_groups_parity():
    """3xTF32 in both forms: the fp32 parity cases with each
    EMOE_TF32_CG (CTA-pair 256 x 128 tiles with segments padded to 256 rows,
    or single-CTA 128 x 128 tiles) -- every fp32 stage within the 1e-5
    tolerance of the oracle, permutation bit-exact for that padding."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    here = Path(__file__).resolve()
    for cg in ("1", "2"):
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                            str(here), "-k", "test_forward_parity and fp32"], cwd=str(here.parent.parent),
                           env=dict(os.environ, EMOE_TF32_CG=cg), capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and " passed" in r.stdout, f"EMOE_TF32_CG={cg}\n" + r.stdout[-3000:] + r.stderr[-2000:]


_SCAN_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import build_layer
E, d, f, k, T, res, act, dtype = {args!r}
layer, _, _ = build_layer(E, d, f, k, dtype, act, "topk_softmax" if k > 1 else "full_softmax", len(res), res,
                          max_tokens=T)
td = torch.bfloat16 if dtype == "bf16" else torch.float32
x = torch.randn(T, d, generator=torch.Generator().manual_seed(5)).to(td).cuda()
y = layer.forward(x)
ws = layer.workspace()
R = int(ws["seg_offsets"][-1].item())
torch.save(dict(y=y.cpu(), pos=ws["pos"].cpu(), counts=ws["counts"].cpu(), offs=ws["seg_offsets"].cpu(),
                row_token=ws["row_token"][:R].cpu()), {out!r})
"""


@pytest.mark.gpu
@pytest.mark.parametrize("args", [(8, 256, 512, 2, 4096, [0, 2, 5, 7], "swiglu", "bf16"),
                                  (128, 256, 512, 1, 3000, list(range(0, 128, 5)), "relu", "bf16"),
                                  (8, 256, 512, 2, 700, [1, 2, 3, 4], "swiglu", "fp32"),
                                  (32, 512, 512, 3, 1, [4, 9], "swiglu", "bf16")])
def test_small_batch_scan_fold_bit_identical(args, tmp_path):
    """Up to 32 token blocks the K3a scan runs inside the permute kernel
    (EMOE_SMALL_SCAN=1, default): counts, padded offsets, positions, row
    sources and outputs bit-identical to scan_kernel + permute (=0)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    outs = []
    for flag in ("1", "0"):
        out = tmp_path / f"s{flag}.pt"
        code = _SCAN_SCRIPT.format(root=str(root), tests=str(root / "tests"), args=args, out=str(out))
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, EMOE_SMALL_SCAN=flag),
                       timeout=300)
        outs.append(torch.load(out))
    for key in outs[0]:
        assert torch.equal(outs[0][key], outs[1][key]), f"{key} differs between the folded and separate scan"
