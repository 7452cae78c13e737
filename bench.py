#!/usr/bin/env python
"""MoE-layer tokens/s under predicted-expert residency (BASELINE.json metric).

Default workload = BASELINE config 2: Mixtral-8x7B-shaped MoE layer, bf16,
8 experts top-2, 4 resident experts (predicted), batch 32 x 2048 tokens on one
B200.  One step = one pass of the hot path over that batch:
    gate + top-k + residency remap (K1) -> scan + stable permute (K3)
    -> grouped SwiGLU GEMM1 + GEMM2 on tcgen05 (K4) -> combine (K5)
    -> popularity-histogram update over the batch's routing (K2, A6)
The resident set comes from the reference flow run on the GPU: routing trace
(the reference's Markov generator, seed 17, calibration 0.6 / 0.8), fit on
200 training prompts, predict_all_layers from the previous prompt, Eq. 2 over
the 32 queued prompts, loading_targets + plan_loading, and the planned H2D
loads from pinned host memory.  Activations are synthesised so that the gate
(computed from x) reproduces the trace's routing.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config mixtral|switch]
Under torchrun (N > 1) each rank runs an independent replica on its own 65,536
tokens (weak scaling, no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE-layer tokens/sec (predicted-expert residency) at 1/2/4/8 B200; % roofline"

CONFIGS = {
    "mixtral": dict(workload="BASELINE config 2: Mixtral-8x7B-shaped MoE layer bf16, 8 experts top-2, 4 resident "
                             "(predicted), batch 32 x 2048 tokens",
                    E=8, k=2, L=4, d=4096, f=14336, act="swiglu", wm="topk_softmax", prompts=32, tokens=2048,
                    train=200, layer_lambda=0.6, prompt_lambda=0.8, seed=17),
    "synthetic": dict(workload="BASELINE config 1: synthetic MoE layer fp32, 8 experts top-2, 4 resident "
                               "(predicted), d_model=1024, d_ff=3584, 512 tokens",
                      E=8, k=2, L=4, d=1024, f=3584, act="swiglu", wm="topk_softmax", prompts=1, tokens=512,
                      train=200, layer_lambda=0.6, prompt_lambda=0.8, seed=17, dtype="fp32"),
    # a small bf16 layer for the bench-path tests (not a BASELINE config)
    "tiny": dict(workload="test layer: bf16, 8 experts top-2, 4 resident (predicted), d_model=512, d_ff=1024, "
                          "4 x 512 tokens",
                 E=8, k=2, L=4, d=512, f=1024, act="swiglu", wm="topk_softmax", prompts=4, tokens=512,
                 train=40, layer_lambda=0.6, prompt_lambda=0.8, seed=17),
    "switch": dict(workload="BASELINE config 3: Switch-base-128-shaped layer bf16, 128 experts top-1, 20% resident "
                            "(L=26, predicted), 32 x 2048 tokens",
                   E=128, k=1, L=26, d=768, f=3072, act="relu", wm="full_softmax", prompts=32, tokens=2048,
                   train=200, layer_lambda=0.6, prompt_lambda=0.8, seed=17),
}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sustained=d.get("bf16_tflops_sustained", 1400.0), source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, source="fallback")


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10:  # sampler is live before timing starts
                time.sleep(0.05)
            self.lines.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------
# synthetic workload: one deterministic CPU generator shared by both arms
# ---------------------------------------------------------------------------
X_CHUNK = 4096  # x is generated in 4096-row chunks, each from its own seed
DIGEST_ROWS = 256  # input_digest covers these first rows of x (both arms)


def input_gate(cfg):
    """Gate weights [E][d] in float64: orthonormal rows (QR of a seeded N(0,1)
    matrix), so x can be built to reproduce a routing trace exactly."""
    import torch

    g = torch.Generator().manual_seed(1234)
    q, _ = torch.linalg.qr(torch.randn(cfg["d"], cfg["E"], generator=g, dtype=torch.float64))
    return q.T.contiguous()


def input_expert(cfg, e):
    """Expert e's weights in the config dtype, seeded per (layer 0, expert,
    matrix) = 1234 ^ (e << 4 | mat): W1, W3 ~ N(0, 1/d),
    W2 ~ N(0, 1/f); W3 is None for ReLU experts."""
    import torch

    d, f, td = cfg["d"], cfg["f"], torch_dtype(cfg)

    def mat(j, rows, cols, fan_in):
        g = torch.Generator().manual_seed(1234 ^ (e << 4 | j))
        return (torch.randn(rows, cols, generator=g) / fan_in ** 0.5).to(td)

    w3 = mat(1, f, d, d) if cfg["act"] == "swiglu" else None
    return mat(0, f, d, d), w3, mat(2, d, f, f)


def input_x(cfg, wg64, choices, rows):
    """The first `rows` activations [rows][d] of the serving batch: chunk c
    (rows 4096c ..) from its own seed, x = logits . W_g + noise orthogonal
    to W_g's rows, where logit[c_r] = 8 - r at the trace's ranked choices and
    the rest uniform in [-4, 4) (multiples of 1/64): the gate computed from x
    reproduces the trace's routing.  float64 arithmetic on the CPU, rounded
    to the config dtype, so both bench arms hold the same bits."""
    import torch

    E, d, k, td = cfg["E"], cfg["d"], cfg["k"], torch_dtype(cfg)
    out = torch.empty(rows, d, dtype=td)
    ch = torch.from_numpy(np.ascontiguousarray(choices[:rows])).long()
    for c0 in range(0, rows, X_CHUNK):
        n = min(X_CHUNK, rows - c0)
        g = torch.Generator().manual_seed(7919 * (c0 // X_CHUNK + 1) + 1234)
        lg = torch.round((torch.rand(n, E, generator=g, dtype=torch.float64) * 8.0 - 4.0) * 64) / 64
        for r in range(k):
            lg.scatter_(1, ch[c0:c0 + n, r:r + 1], 8.0 - r)
        z = torch.randn(n, d, generator=g).double()
        z -= (z @ wg64.T) @ wg64
        out[c0:c0 + n] = (lg @ wg64 + z).to(td)
    return out


def input_digest(x_rows, wg, experts):
    """sha256 over the bytes both arms compute on (x sample rows, W_g, the
    resident experts' weights): equal digests = same inputs."""
    import hashlib

    import torch

    h = hashlib.sha256()
    for t in [x_rows, wg] + [w for e in sorted(experts) for w in experts[e] if w is not None]:
        t = t.contiguous()
        h.update((t.view(torch.int16) if t.dtype == torch.bfloat16 else t).numpy().tobytes())
    return h.hexdigest()[:16]


def build_workload(cfg, device, cta_group=0, rank=0, world=1, parallel="replicas", strong=False):
    import torch

    import paper_2503_06823_b200 as emoe
    from paper_2503_06823_b200 import MoELayer
    from paper_2503_06823_b200.ep import owned_experts, plan_shares

    E, k, L, d, f = cfg["E"], cfg["k"], cfg["L"], cfg["d"], cfg["f"]
    P, Tp, P_train = cfg["prompts"], cfg["tokens"], cfg["train"]
    # weak scaling: every rank serves its own P prompts of the same trace;
    # strong: the ranks split one batch of P prompts
    Pr = P // world if strong else P
    T = Pr * Tp
    shape = emoe.ModelShape(1, E, k, expert_bytes=(3 if cfg["act"] == "swiglu" else 2) * d * f * 2)
    trace = emoe.gen_routing_trace(shape, cfg["layer_lambda"], cfg["prompt_lambda"], 0, cfg["seed"],
                                   P_train + Pr * world, Tp)
    train, serve = trace[:P_train], trace[P_train + Pr * rank: P_train + Pr * (rank + 1)]

    # ---- predictor flow on the GPU (fit -> predict -> Eq. 2 -> targets -> plan)
    pred = emoe.moesim._Pred(1, E, k, 1, 0.01)
    dtrain = torch.from_numpy(np.ascontiguousarray(train)).to(device)
    tid = torch.zeros(P_train, dtype=torch.int32, device=device)
    emoe.moesim.check(emoe._lib.lib.emoe_hist_update(pred.h, emoe.moesim.C.c_void_p(dtrain.data_ptr()), P_train, Tp,
                                                     emoe.moesim.C.c_void_p(tid.data_ptr()), None))
    _, sets = emoe.prompt_expert_sets(train, P_train - 1)
    set_arr, sizes = emoe.moesim._sets_array(sets, k)
    wo = np.array([128.0])
    sens = np.ones((1, 1), np.int32)
    has = np.ones(1, np.uint8)
    req_task = np.zeros(P, np.int32)
    req_tok = np.full(P, Tp, np.int32)
    resident0 = np.zeros((1, E), np.uint8)
    budgets = np.array([L], np.int32)
    agg = np.zeros((1, E))
    ev = np.full((1, E), -1, np.int32)
    ld = np.full((1, E), -1, np.int32)
    ne = np.zeros(1, np.int32)
    nl = np.zeros(1, np.int32)
    de = np.zeros(1)
    p_ = emoe.moesim._p
    emoe.moesim.check(emoe._lib.lib.emoe_invocation_host(
        pred.h, 0, p_(set_arr), p_(sizes), 1, p_(wo), p_(sens), p_(has), P, p_(req_task), p_(req_tok), 1,
        p_(resident0), p_(budgets), 0.0, p_(agg), p_(ev), p_(ne), p_(ld), p_(nl), p_(de)))
    loads = [int(e) for e in ld[0, : nl[0]]]
    global_resident = sorted(loads)
    if parallel == "ep" and world > 1:  # this GPU holds only the experts it serves
        # load-aware placement from the Eq. 2 aggregate (identical on every
        # rank: same fitted predictor, same request mix)
        loads = owned_experts(plan_shares(global_resident, E, world, agg[0]), rank)

    # ---- inputs (CPU generator shared with --impl reference), layer, planned loads
    wg64 = input_gate(cfg)
    td = torch_dtype(cfg)
    layer = MoELayer(d, f, E, k, activation=cfg["act"], dtype=cfg.get("dtype", "bf16"), weight_mode=cfg["wm"],
                     num_slots=max(1, len(loads)), max_tokens=T, gemm_cta_group=cta_group)
    layer.set_gate(wg64.to(td))
    # the fused tcgen05 gate (E >= 32) routes from its accumulators; the fp32
    # logits are a parity/debug output, not consumed downstream
    # (tests/test_forward_gpu.py::test_fused_gate_route_bit_identical: identical routing)
    layer.set_keep_logits(False)
    experts = {}
    for e in range(E):
        w1, w3, w2 = input_expert(cfg, e)
        layer.register_expert(e, w1, w3, w2)
        if e in global_resident:
            experts[e] = (w1, w3, w2)
    layer.begin_load([], loads)
    layer.poll_loads(blocking=True)
    # route_token's fallback scores = the invocation's aggregate (engine.cpp:424, :529-531)
    layer.set_scores(agg[0])
    load_bytes, load_ms = layer.last_load_stats()
    torch.cuda.synchronize()

    # ---- activations whose gate logits reproduce the serving trace
    choices = serve.reshape(T, k)  # [P][1][Tp][k] -> token-major
    x_host = input_x(cfg, wg64, choices, T)
    x = x_host.to(device)
    res = [0] * E
    for e in global_resident:
        res[e] = 1
    info = dict(trace=trace, loads=loads, aggregate=agg[0].tolist(), load_bytes=load_bytes, load_ms=load_ms,
                choices=choices, resident=res, global_resident=global_resident, x_host=x_host,
                wg=wg64.to(td), experts=experts)
    return layer, pred, x, info


def cpu_reference_step(cfg, layer_info, x_host_f32, wg_f32, experts_f32, n_tokens, port, ref, threads):
    """One bounded CPU step of the same workload: the reference's route_token
    (oracle/_ref, single thread) + the oracle port of gate/permute/FFN/combine
    (pthreads over all host cores).  Returns seconds."""
    E, k = cfg["E"], cfg["k"]
    resident = np.zeros(E, np.uint8)
    resident[np.asarray(layer_info["resident"], bool)] = 1
    x = x_host_f32[:n_tokens]
    t0 = time.perf_counter()
    logits = port.gate_logits(x, wg_f32)
    o = port.gate_route(logits, k, 0 if cfg["wm"] == "topk_softmax" else 1, resident,
                        scores=layer_info.get("aggregate"))
    if ref is not None:
        ref.route_tokens(o["topk_idx"], resident, scores=layer_info.get("aggregate"))
    counts, offsets, pos, src = port.permute(o["served_idx"], E, 1)
    Y = np.zeros((int(offsets[-1]), cfg["d"]), np.float32)
    for e in range(E):
        rows = np.arange(offsets[e], offsets[e + 1])
        if rows.size == 0:
            continue
        w1, w3, w2 = experts_f32[e]
        bf = cfg.get("dtype", "bf16") == "bf16"
        Y[rows] = port.expert_ffn(x[src[rows]], w1, w3, w2, 0 if cfg["act"] == "swiglu" else 1, bf, threads)
    port.combine(Y, pos, o["served_w"], cfg.get("dtype", "bf16") == "bf16")
    return time.perf_counter() - t0


def f32_inputs(x_rows, wg, experts):
    """float32 numpy copies for the oracle port."""
    to = lambda t: None if t is None else t.float().numpy()  # noqa: E731
    return to(x_rows), to(wg), {e: tuple(to(w) for w in ws) for e, ws in experts.items()}


CPU_PATH_NOTE = ("oracle port = the repo's CPU restatement (C, scalar loops with fp64 accumulation, pthreads): "
                 "a correctness oracle timed with a stopwatch, not a tuned CPU kernel; route_token is the "
                 "reference's own code (oracle/_ref)")


def run_cpu_baseline(cfg, x_rows, wg, experts, info, target_s=10.0):
    """cpu_baseline of the GPU arm: the bounded CPU path on the first rows of
    the same x, with the same weights and resident set."""
    from oracle.oracle import Port, Ref, have_ref

    port = Port()
    ref = Ref() if have_ref() else None
    threads = port.threads()
    T = x_rows.shape[0]
    xs, wgf, ex = f32_inputs(x_rows[: min(X_CHUNK, T)], wg, experts)
    # calibrate the sample so the timed CPU work is ~target_s (never more rows than the batch has)
    n = min(8, T)
    dt = cpu_reference_step(cfg, info, xs, wgf, ex, n, port, ref, threads)
    n = int(max(min(8, T), min(X_CHUNK, T, n * target_s / max(dt, 1e-3))))
    dt = cpu_reference_step(cfg, info, xs, wgf, ex, n, port, ref, threads)
    rt_ns = None
    if ref is not None:
        res = np.zeros(cfg["E"], np.uint8)
        res[np.asarray(info["resident"], bool)] = 1
        rt_ns, _ = ref.time_route_tokens(info["choices"], res, reps=3)
    return dict(value=n / dt, unit="tokens/s", cores=threads, kind="port",
                sample=f"{n} of {T} tokens through the full CPU path: gate+top-k, permute, SwiGLU/ReLU FFN, "
                       f"combine ({threads} pthreads); reference route_token "
                       f"{'%.2f ns/token' % rt_ns if rt_ns else 'n/a'}; {CPU_PATH_NOTE}",
                seconds=dt, input_digest=input_digest(x_rows[:DIGEST_ROWS], wg, experts))


# ---------------------------------------------------------------------------
def parallelism_label(world, parallel, transport):
    """config.parallelism: "single" at N=1; under torchrun "ep{N}-{transport}"
    (the default) or "replicas{N}"."""
    if world <= 1:
        return "single"
    return f"ep{world}-{transport}" if parallel == "ep" else f"replicas{world}"


def build_parser():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="emoe", choices=["emoe", "reference"])
    ap.add_argument("--config", default="mixtral", choices=list(CONFIGS) + ["stream", "stack"],
                    help="stream = BASELINE config 5 (mixed-task 8k-token prompt stream over a 32-layer stack); "
                         "stack = BASELINE config 4 (32-layer Mixtral-shaped stack, 32 x 2048 tokens per GPU)")
    ap.add_argument("--stream-layers", type=int, default=32)
    ap.add_argument("--stream-prompts", type=int, default=80)
    ap.add_argument("--residency", default="predicted", choices=["predicted", "dynamic"],
                    help="--config stream: eMoE predicted residency, or the reference's on-demand baseline "
                         "(engine.cpp:469-502) for comparison")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: seconds of CPU work for the warm-up + timed steps together")
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--gemm-cta-group", type=int, default=0, choices=[0, 1, 2],
                    help="FFN GEMM CTA group (0 = the layer's auto choice)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step as one captured CUDA graph (stage times then from a profiling capture of the step "
                         "after the timed region) or launch it eagerly; auto = graph for the sub-millisecond "
                         "steps of configs 1 and 3 (launch-bound: +27 %% / +6 %%, profiles/r01_cuda_graph_ab.jsonl), "
                         "eager for config 2 (stage events inside the timed region)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = every GPU serves the config's full batch (default); strong = the "
                         "config's batch is split over the GPUs (N must divide its 32 prompts)")
    ap.add_argument("--parallel", default="ep", choices=["replicas", "ep"],
                    help="N>1: expert parallelism (default; the north star's split: each GPU computes its share "
                         "of the resident experts' rows, tokens exchanged over NVLink) or replicas of the "
                         "predicted resident set (no exchange)")
    ap.add_argument("--ep-at-1", action="store_true",
                    help="run the expert-parallel code path even with one process (a world-1 group; tests)")
    ap.add_argument("--ep-recv-cap", type=int, default=0,
                    help="--parallel ep: p2p receive-buffer rows per GPU (0 = the worst case, world x rows_cap); "
                         "nccl: rows per (source, destination) chunk (0 = the plan's bound, ep.plan_pair_rows)")
    ap.add_argument("--ep-transport", default="p2p", choices=["p2p", "nccl"],
                    help="--parallel ep: dispatch/combine fused into the permute/combine kernels over "
                         "IPC-mapped peer memory (p2p), or NCCL all-to-alls over fixed capacity chunks between "
                         "the stage kernels (no host synchronisation)")
    return ap


def main():
    args = build_parser().parse_args()
    args.warmup = max(args.warmup, 3)
    if args.config == "stream":
        return main_stream(args)
    if args.config == "stack":
        return main_stack(args)
    cfg = CONFIGS[args.config]

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        nccl_log_to_stderr()
        dist.init_process_group("nccl" if args.impl == "emoe" else "gloo")
    if args.impl == "reference":
        return main_reference(args, cfg, rank, world)

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    import paper_2503_06823_b200 as emoe
    from paper_2503_06823_b200 import _lib

    use_ep = args.parallel == "ep" and (world > 1 or args.ep_at_1)
    ensure_group_for_ep_at_1(args, world)
    strong = args.scaling == "strong" and world > 1
    if strong and cfg["prompts"] % world:
        raise SystemExit(f"--scaling strong: {world} GPUs do not divide the {cfg['prompts']} prompts")
    layer, pred, x, info = build_workload(cfg, device, args.gemm_cta_group, rank, world,
                                          "ep" if use_ep else "replicas", strong)
    T = x.shape[0]
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    P, Tp = cfg["prompts"] // (world if strong else 1), cfg["tokens"]
    tid = torch.zeros(P, dtype=torch.int32, device=device)
    import ctypes as C

    ep_model = None
    ep_stats = ep_stages = None
    ep_fallback = None
    if use_ep and args.ep_transport == "p2p":
        ep_model, ep_fallback = make_p2p_ep(layer, info, args, x, world, device)
        if ep_model is None:  # every rank falls back together: the NCCL transport, same placement
            args.ep_transport = "nccl"
            if rank == 0:
                print(f"bench: peer-memory EP unavailable ({ep_fallback}); running the NCCL transport",
                      file=sys.stderr, flush=True)
    if use_ep and args.ep_transport == "nccl":  # NCCL all-to-alls over capacity chunks, no host synchronisation
        from paper_2503_06823_b200.ep import NcclExpertParallelMoE, plan_pair_rows, plan_shares

        cum = plan_shares(info["global_resident"], cfg["E"], world, info["aggregate"])
        # --ep-recv-cap sizes the NCCL chunks too, unless it is the p2p setting that just failed
        cap = (args.ep_recv_cap if not ep_fallback else 0) or plan_pair_rows(cum, info["aggregate"], T, cfg["k"],
                                                                            layer.seg_pad)
        ep_model = NcclExpertParallelMoE(layer, info["global_resident"], loads=info["aggregate"], cap_rows=cap)

    def eager_step():
        if ep_model is not None:
            ep_model(x, out=y)
        else:
            layer.forward(x, out=y)
        ws_topk = layer_ws_topk(layer)
        emoe.moesim.check(_lib.lib.emoe_hist_update(pred.h, C.c_void_p(ws_topk), P, Tp, C.c_void_p(tid.data_ptr()),
                                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    for _ in range(args.warmup):
        eager_step()
    torch.cuda.synchronize()
    ws = layer.workspace()
    counts = ws["counts"].cpu().numpy()
    S = int(counts.sum())
    hit_rate = float(ws["route_hit"].float().mean().item())
    fallback = float((ws["route_rank"] == -1).float().mean().item())

    # --graph on: the step as one CUDA graph (every kernel of the step
    # replayed as a whole: no per-launch host or queue gaps, which matter for
    # the small configs; EP steps stay eager).  The per-stage events are not
    # captured (their timestamps inside replays were not trustworthy), so the
    # stage times then come from a second capture with the events as graph record nodes.
    graph = None
    launches_per_step = 0
    use_graph = args.graph == "on" or (args.graph == "auto" and args.config in ("synthetic", "switch"))
    if use_graph and ep_model is None:
        l0 = _lib.lib.emoe_kernel_launches()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="thread_local"):
            eager_step()
        launches_per_step = int(_lib.lib.emoe_kernel_launches() - l0)
        graph.replay()  # warm replay
        torch.cuda.synchronize()
    elif ep_model is not None:
        ep_model.set_profiling(True)
    else:
        layer.set_profiling(True)

    def step():
        if graph is not None:
            graph.replay()
        else:
            eager_step()

    launches0 = _lib.lib.emoe_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = int(_lib.lib.emoe_kernel_launches() - launches0) + launches_per_step * args.steps
    clock_note = "sampled during the timed region"
    if len(clk.lines) < 3:  # timed region shorter than the sampler period: sample a continuation of the same loop
        with ClockSampler(local) as clk:
            t_end = time.time() + 1.0
            while time.time() < t_end:
                step()
                torch.cuda.synchronize()
        clock_note = "timed region < 150 ms: sampled over 1 s of the same steps right after it"
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    stages_profiled, stage_scale = None, 1.0
    if ep_model is None:
        if graph is not None:
            # stage times from the same step captured once more with the stage
            # events as record nodes of the graph, replayed and read one replay
            # at a time (eager steps carry host launch gaps between stages, which
            # inflated them by up to 25 % on some hosts)
            layer.set_profiling(True)
            gprof = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gprof, capture_error_mode="thread_local"):
                eager_step()
            layer.set_profiling(False)
            stages = {}
            for _ in range(args.steps):
                # each replay re-stamps the events: only the last of a short
                # back-to-back burst is read, so the profiled step runs at the
                # clocks of the timed region (reading after an idle gap caught
                # some boxes mid clock ramp: stage sums 20 % over the step)
                for _ in range(4):
                    gprof.replay()
                torch.cuda.synchronize()
                for key, v in layer.stage_times_last().items():
                    stages[key] = stages.get(key, 0.0) + v / args.steps
            del gprof
            # On some boxes the event-instrumented replays run slower than the
            # timed ones (stage sums up to 20 % over the timed step, every stage
            # alike): keep the profiled times, and scale the stages that feed
            # the roofline so they sum to the timed step when they overshoot it.
            stages_profiled = dict(stages)
            stage_scale = min(1.0, ms / sum(stages.values())) if sum(stages.values()) > 0 else 1.0
            stages = {key: v * stage_scale for key, v in stages.items()}
        else:
            stages = layer.stage_times()
    elif args.ep_transport == "p2p":  # the EP forward's own stage events
        ep_stages = ep_model.stage_times()
        ep_model.set_profiling(False)
        ep_stats = ep_model.stats()
        stages = dict(route=ep_stages["route"], permute=ep_stages["dispatch"], gemm1=ep_stages["gemm1"],
                      gemm2=ep_stages["gemm2_return"], combine=ep_stages["combine"])
    else:  # NCCL transport: events on the compute stream, which waits on each collective
        ep_stages = ep_model.stage_times()
        ep_model.set_profiling(False)
        stages = dict(route=ep_stages["route"], permute=ep_stages["dispatch"], gemm1=ep_stages["ffn"], gemm2=0.0,
                      combine=ep_stages["combine"])
        ep_status, _ = ep_model.status()
        if ep_status != 0:
            raise SystemExit(f"--ep-transport nccl: a (source, destination) pair overflowed the {ep_model.cap}-row "
                             "chunk (status 2); raise --ep-recv-cap")
    layer.set_profiling(False)
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * T / (ms / 1e3)

    # ---- end to end through the public host-buffer API (H2D x + D2H y every step)
    x_host = x.cpu().pin_memory()
    y_host = torch.empty_like(x_host).pin_memory()

    y_host2 = torch.empty_like(x_host).pin_memory()

    def e2e_step(i):
        # the serving pattern of the public host-buffer API: call i+1 is enqueued
        # while call i computes (emoe_moe_forward_host_async, two staging sets)
        if ep_model is None:
            layer.forward_host_async(x_host, y_host if i % 2 == 0 else y_host2)
        else:
            y_host.copy_(ep_model(x_host.to(device, non_blocking=True)))

    def e2e_wait():
        if ep_model is None:
            layer.wait_host()
        torch.cuda.synchronize()

    for i in range(2):
        e2e_step(i)
    e2e_wait()
    if world > 1:
        dist.barrier()
    # PCIe-bound shapes (config 3) vary with the box's host link: the copy
    # floor below is measured on the same box for comparison
    t0 = time.perf_counter()
    for i in range(args.e2e_steps):
        e2e_step(i)
    e2e_wait()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # the copy floor of the e2e path: the same H2D and D2H bytes per step with
    # no compute (one stream each way, concurrent, back to back)
    xd_f = torch.empty(x_host.shape, dtype=x_host.dtype, device=device)
    yd_f = torch.empty_like(xd_f)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    n_floor = 20
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_floor):
        with torch.cuda.stream(s_in):
            xd_f.copy_(x_host, non_blocking=True)
        with torch.cuda.stream(s_out):
            y_host.copy_(yd_f, non_blocking=True)
    torch.cuda.synchronize()
    floor_s = (time.perf_counter() - t0) / n_floor
    del xd_f, yd_f
    e2e = dict(value=world * T / e2e_s, unit="tokens/s", h2d_bytes_per_step=x_host.numel() * x_host.element_size(),
               d2h_bytes_per_step=y_host.numel() * y_host.element_size(), ms_per_step=e2e_s * 1e3,
               copy_floor_ms=floor_s * 1e3, frac_of_copy_floor=floor_s / e2e_s,
               copy_floor_gbs=(x_host.numel() + y_host.numel()) * x_host.element_size() / floor_s / 1e9,
               calls=args.e2e_steps,
               note="emoe_moe_forward_host_async per call (H2D x, K1-K5, D2H y), wall clock over the calls; "
                    "the device-timed step also runs the A6 histogram update and per-stage events, which "
                    "this path does not (about 5 % of a config-1 step, < 0.1 % of config 2)")

    # ---- roofline of the dominant kernel (the grouped FFN GEMMs)
    peaks = load_peaks()
    d, f = cfg["d"], cfg["f"]
    fp32 = cfg.get("dtype", "bf16") == "fp32"
    nmat = 3 if cfg["act"] == "swiglu" else 2
    # the FFN rows this GPU computes: its own served rows (single GPU,
    # replicas) or, under EP, the rows the split assigned it
    S_ffn = ep_stats["rows_computed_real"] if ep_stats else S
    ffn_flops = 2.0 * nmat * d * f * S_ffn
    ffn_ms = stages["gemm1"] + stages["gemm2"]
    achieved = ffn_flops / (ffn_ms / 1e3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "ffn_gemm_dram_traffic.json"
    if tfile.exists() and args.config == "mixtral":  # ncu capture of this workload (profiles/)
        traffic = json.loads(tfile.read_text())["ffn_bytes_per_step"]
    if fp32 and layer.fp32_tensor_core:
        # config 1 on tcgen05 3xTF32: three TF32 MMAs per fp32 product, so the
        # roofline is a third of the TF32 tensor peak measured in this run
        tf32_peak = measure_tf32_peak(device)
        fp32_peak = measure_fp32_peak(device)
        roofline = dict(bound="tensor", achieved=round(achieved, 2), peak=round(tf32_peak / 3, 2), unit="TFLOP/s",
                        frac=round(achieved / (tf32_peak / 3), 4), traffic=None,
                        kernel="gemm_tf32x3_kernel (K4: GEMM1 SwiGLU + GEMM2, 3xTF32 on tcgen05), avg of the "
                               "timed steps",
                        algorithmic=f"2*{nmat}*d*f*S = {ffn_flops:.4g} fp32 FLOP per step (S={S} served rows)",
                        peak_kind="TF32 cuBLAS 8192^3 / 3 (three TF32 products per fp32 product), measured in this "
                                  f"run: TF32 {tf32_peak:.1f} TFLOP/s",
                        fp32_ffma_peak=round(fp32_peak, 2), frac_of_fp32_ffma_peak=round(achieved / fp32_peak, 4))
    elif fp32:  # SIMT FFMA kernel against the CUDA-core fp32 peak measured in this run
        fp32_peak = measure_fp32_peak(device)
        roofline = dict(bound="fp32", achieved=round(achieved, 2), peak=round(fp32_peak, 2), unit="TFLOP/s",
                        frac=round(achieved / fp32_peak, 4), traffic=None,
                        kernel="grouped_gemm_f32 (K4: GEMM1 SwiGLU + GEMM2, FFMA), avg of the timed steps",
                        algorithmic=f"2*{nmat}*d*f*S = {ffn_flops:.4g} FLOP per step (S={S} served rows)",
                        peak_kind="fp32 cuBLAS SGEMM 8192^3 (TF32 off), best of 5, measured in this run")
    else:
        # the sustained (power-capped) rate for a timed region long enough to
        # reach it, the burst rate for a short one (config 3: 20 steps = 10 ms)
        long_region = args.steps * ms >= 150.0
        peak = peaks["bf16_sustained"] if long_region else peaks["bf16"]
        roofline = dict(bound="tensor", achieved=round(achieved, 1), peak=peak, unit="TFLOP/s",
                        frac=round(achieved / peak, 4), traffic=traffic,
                        traffic_unit="bytes per step (GEMM1 + GEMM2), ncu dram__bytes_read+write",
                        kernel="grouped_gemm_kernel (K4: GEMM1 SwiGLU + GEMM2), avg of the timed steps",
                        algorithmic=f"2*{nmat}*d*f*S = {ffn_flops:.4g} FLOP per step (S={S_ffn} rows computed "
                                    f"on this GPU)",
                        peak_kind=(f"bf16_tflops_sustained ({peaks['source']}; timed region >= 150 ms); "
                                   f"burst {peaks['bf16']}") if long_region else
                                  (f"bf16_tflops burst ({peaks['source']}; timed region {args.steps * ms:.0f} ms "
                                   f"< 150 ms); sustained {peaks['bf16_sustained']}"),
                        frac_of_burst=round(achieved / peaks["bf16"], 4),
                        frac_of_sustained=round(achieved / peaks["bf16_sustained"], 4))
    hbm_stages = {}
    eb = elem_bytes(cfg)
    xb = T * d * eb
    hbm_stages["route"] = (xb + T * k_of(cfg) * 8 + T * 9) / (stages["route"] / 1e3) / 1e9
    hbm_stages["permute"] = (xb + S * d * eb + 8 * S) / (stages["permute"] / 1e3) / 1e9
    hbm_stages["combine"] = (S * d * eb + xb + 4 * S) / (stages["combine"] / 1e3) / 1e9

    out = dict(metric=METRIC, value=round(value, 1), unit="tokens/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(ms, 4), higher_is_better=True,
               scaling="strong" if strong else "weak",
               vs_baseline=None, dtype=cfg.get("dtype", "bf16"),
               data="synthetic (random-init weights; routing = reference Markov trace embedded in x)",
               config=dict(workload=cfg["workload"] + (f" split over {world} GPUs" if strong else ""),
                           tokens_per_step=T, tokens_per_gpu=T, num_experts=cfg["E"], top_k=cfg["k"],
                           step_launch=("one CUDA graph per step (replayed); stages_ms and the roofline from the "
                                        "same step captured with its stage events as graph record nodes, replayed "
                                        "and read one replay at a time") if graph is not None else "eager",
                           resident_experts=cfg["L"], resident_set=[e for e in range(cfg["E"])
                                                                     if info["resident"][e]],
                           d_model=d, d_ff=f, activation=cfg["act"], served_rows=S, hit_rate=round(hit_rate, 4),
                           fallback_rate=round(fallback, 4),
                           l2=("inputs larger than L2: x is %.0f MB per step" % (xb / 1e6)) if xb > 126e6 else
                           ("working set larger than L2: %.0f MB of resident expert weights streamed per step "
                            "(x is %.1f MB)" % (cfg["L"] * nmat * d * f * eb / 1e6, xb / 1e6)),
                           parallelism=parallelism_label(world, args.parallel, args.ep_transport),
                           gemm_cta_group=layer.gemm_cta_group, seg_pad=layer.seg_pad),
               roofline=roofline, e2e=e2e, gpu_launches=launches, clocks=dict(clk.summary(), note=clock_note),
               stages_ms={kk: round(v, 4) for kk, v in stages.items()},
               stage_hbm_gbs={kk: round(v, 1) for kk, v in hbm_stages.items()},
               expert_load=dict(bytes=info["load_bytes"], ms=round(info["load_ms"], 3),
                                h2d_gbs=round(info["load_bytes"] / max(info["load_ms"], 1e-9) / 1e6, 2),
                                experts=info["loads"]))
    if stages_profiled is not None:
        out["stages_ms_profiled"] = {kk: round(v, 4) for kk, v in stages_profiled.items()}
        out["stage_scale"] = round(stage_scale, 4)
        out["stages_note"] = ("stages_ms = the profiled stage times (graph replays with the stage events as record "
                              "nodes, stages_ms_profiled) scaled by stage_scale = min(1, timed step / their sum): on "
                              "some boxes the instrumented replays run uniformly slower than the timed ones")
    if ep_stats:
        out["ep"] = ep_report(ep_model, ep_stages, ep_stats, world, rank, device)
    elif ep_model is not None:  # NCCL transport
        a2a_bytes = ep_model.send.numel() * ep_model.send.element_size()
        if ep_fallback:
            out["config"]["ep_p2p_fallback"] = ep_fallback
        out["ep"] = dict(transport="nccl: count all_gather_into_tensor, dispatch and return all_to_all_single over "
                                   f"equal {ep_model.cap}-row chunks per (source, destination) pair, no host sync",
                         stages_ms={kk: round(v, 4) for kk, v in ep_stages.items()},
                         exchange=dict(a2a_bytes_per_call=a2a_bytes,
                                       dispatch_a2a_gbs=round(a2a_bytes / max(ep_stages["dispatch_a2a"], 1e-9) / 1e6, 1),
                                       return_a2a_gbs=round(a2a_bytes / max(ep_stages["return_a2a"], 1e-9) / 1e6, 1),
                                       note="bytes each rank's all_to_all_single moves (whole chunks, incl. its own); "
                                            "GB/s over the stage's events on the compute stream"),
                         placement=ep_model.owned())
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = run_cpu_baseline(cfg, info["x_host"], info["wg"], info["experts"], info)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ensure_group_for_ep_at_1(args, world):
    """--ep-at-1 without torchrun: a world-1 NCCL group, so the expert-parallel
    code path (handle exchange, device barriers, stage events, report) runs on
    one GPU."""
    import torch
    import torch.distributed as dist

    if args.ep_at_1 and world == 1 and args.parallel == "ep" and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))


def nccl_log_to_stderr():
    """NCCL's communicator lines (transport: NVLink P2P / NVLS) on stderr, so
    stdout keeps the one JSON line."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,P2P,NVLS")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def make_p2p_ep(layer, info, args, x, world, device):
    """The peer-memory EP model, or (None, why) when it cannot run here: its
    construction or a first forward failed (or timed out) on any rank -- the
    ranks agree by an all-reduce, so all of them fall back together."""
    import torch
    import torch.distributed as dist

    from paper_2503_06823_b200.ep import PeerExpertParallelMoE

    os.environ.setdefault("EMOE_EP_TIMEOUT_S", "20")  # a failed peer surfaces as status 1, not a hang
    model, err = None, None
    try:
        model = PeerExpertParallelMoE(layer, info["global_resident"], loads=info["aggregate"],
                                      recv_rows_cap=args.ep_recv_cap)
        model(x)
        st, _ = model.status()
        if st != 0:
            err = f"first forward status {st}"
    except Exception as e:  # noqa: BLE001 (reported, and every rank falls back)
        err = f"{type(e).__name__}: {e}"
    ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=device)
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 1:
        return model, None
    if model is not None:
        model.close()
    return None, err or "the peer-memory setup failed on another rank"


def ep_report(ep_models, stages, stats, world, rank, device):
    """The EP step's stage times (rank 0's events; summed over layers for a
    stack), exchange volume and NVLink rates, and the placement; the busiest
    rank's FFN rows against the mean (the FFN-bound step waits for it)."""
    import torch
    import torch.distributed as dist

    models = ep_models if isinstance(ep_models, (list, tuple)) else [ep_models]
    t = torch.tensor([float(stats["rows_computed_real"])], device=device)
    rows = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(rows, t)
    rows = [float(r.item()) for r in rows]
    disp_ms, ret_ms = stages["dispatch"], stages["gemm2_return"]
    return dict(transport="p2p: dispatch fused into the permute (NVLink stores into the computing rank's receive "
                          "buffer), return fused into GEMM2's epilogue, device-side barriers",
                stages_ms={k: round(v, 4) for k, v in stages.items()},
                exchange=dict(dispatch_bytes_to_peers=stats["dispatch_bytes_to_peers"],
                              return_bytes_to_peers=stats["return_bytes_to_peers"],
                              dispatch_nvlink_gbs=round(stats["dispatch_bytes_to_peers"] / max(disp_ms, 1e-9) / 1e6, 1),
                              note="bytes of this rank's rows stored to peers in the dispatch kernel, and of the "
                                   "expert outputs it pushes back to their sources from GEMM2 (summed over layers "
                                   "for a stack); GB/s over the dispatch stage"),
                rows_computed_per_rank=rows, balance_mean_over_max=round(sum(rows) / len(rows) / max(max(rows), 1), 4),
                placement=[m.owned() for m in models][:4], layers=len(models))


def k_of(cfg):
    return cfg["k"]


def torch_dtype(cfg):
    import torch

    return torch.float32 if cfg.get("dtype", "bf16") == "fp32" else torch.bfloat16


def elem_bytes(cfg):
    return 4 if cfg.get("dtype", "bf16") == "fp32" else 2


def measure_tf32_peak(device, n=8192, reps=5):
    """TF32 tensor-core peak (cuBLAS, torch.matmul with TF32 on), best of `reps`."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, device=device)
    b = torch.randn(n, n, device=device)
    c = a @ b
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = prev
    del a, b, c
    return 2.0 * n ** 3 / best / 1e12


def measure_fp32_peak(device, n=8192, reps=5):
    """fp32 CUDA-core roofline denominator for config 1, measured in this run:
    cuBLAS SGEMM (torch.matmul, TF32 off) n^3, best of `reps` (CUDA events)."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    a = torch.randn(n, n, device=device)
    b = torch.randn(n, n, device=device)
    c = a @ b
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = prev
    del a, b, c
    return 2.0 * n ** 3 / best / 1e12


def layer_ws_topk(layer):
    from paper_2503_06823_b200._lib import Workspace, lib
    import ctypes as C

    w = Workspace()
    lib.emoe_layer_workspace(layer.h, C.byref(w))
    return w.topk_idx


def main_stream(args):
    """BASELINE config 5: a mixed-task stream of 8k-token prompts ("conv" sensitive on
    every layer, "cls" on none, mix 0.5/0.5) through a 32-layer Mixtral-shaped stack
    with phi = 0.5 (4 of 8 experts per layer), predictor every p = 40 prompts and
    skipped for windows with only insensitive requests, expert loads on a shared
    side copy stream overlapped with compute.  Routing-driven: the gate logits of
    prompt p / layer l embed the reference trace.  Single GPU."""
    import torch
    import torch.distributed as dist

    import paper_2503_06823_b200 as emoe
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig, TaskSpec, moesim_prompt_sets, run_stream

    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    m, E, k, L, d, f, T, p = args.stream_layers, 8, 2, 4, 4096, 14336, 8192, 40
    tasks = {"cls": TaskSpec(16.0, [0] * m), "conv": TaskSpec(256.0, [1] * m)}
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=T, period=p, mode=0, tasks=tasks)
    P_train, P_serve = 60, args.stream_prompts
    shape = emoe.ModelShape(m, E, k)
    trace = emoe.gen_routing_trace(shape, 0.6, 0.8, 0, 17, P_train + P_serve, T)
    rng = np.random.default_rng(5)
    prompt_tasks = ["conv" if v < 0.5 else "cls" for v in rng.random(P_train + P_serve)]
    # a window of only insensitive prompts exercises the skip
    if P_serve >= 3 * p:
        for q in range(P_train + 2 * p, P_train + 3 * p):
            prompt_tasks[q] = "cls"
    g = torch.Generator(device=device).manual_seed(1234)
    host = [tuple((torch.randn(*s, generator=g, device=device) / s[1] ** 0.5).to(torch.bfloat16).cpu().pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    # every layer runs its gate on x (random N(0, 1/d) weights); the trace is
    # added to the gate's logits as a dominant bias (EMOE_LOGITS_ADD), so the
    # routing follows the trace the predictor was fitted on
    gates = [(torch.randn(E, d, generator=g, device=device) / d ** 0.5).to(torch.bfloat16).cpu() for _ in range(m)]
    stack = MoEStack(cfg, host, gates)
    for layer in stack.layers:
        layer.set_logits_mode("add")
    trace_dev = torch.from_numpy(trace).to(device)
    # N > 1: every rank tallies a shard of the training prompts and one
    # all-reduce merges them (ep.fit_sharded; identical to one fit)
    stack.fit(trace_dev[:P_train].contiguous(), prompt_tasks[:P_train],
              group=dist.group.WORLD if dist.is_initialized() and dist.get_world_size() > 1 else None)
    # initial placement: the first plan from an empty device (blocking, untimed)
    _, sets = moesim_prompt_sets(trace_dev, P_train - 1)
    ops, agg, _ = stack.invocation(sets, [(prompt_tasks[q], T) for q in range(P_train, P_train + p)])
    stack.apply(ops)
    stack.set_scores(agg)
    for layer in stack.layers:
        layer.poll_loads(blocking=True)
    torch.cuda.synchronize()
    # the plans' delta_e uses the per-expert copy time measured by this load
    n0 = max(1, len(ops[0][1]))
    b0, ms0 = stack.layers[0].last_load_stats()
    cfg.per_expert_seconds = ms0 / 1e3 / n0

    # trace biases of every prompt, built before the timed region:
    # [m][T][E], 16 x (8 - r at the ranked choices, uniform in [-4, 4) elsewhere)
    bias = {}
    for q in range(P_train, P_train + P_serve):
        lg = torch.round((torch.rand(m, T, E, generator=g, device=device) * 8.0 - 4.0) * 64) / 64
        ch = trace_dev[q].long()
        for r in range(k):
            lg.scatter_(2, ch[:, :, r:r + 1], 8.0 - r)
        bias[q] = lg * 16.0

    def logits_of(q):
        return bias[q]

    x = torch.randn(T, d, generator=g, device=device).to(torch.bfloat16)
    out = torch.empty_like(x)
    hits = torch.zeros(m, dtype=torch.int64, device=device)
    for q in range(P_train, P_train + args.warmup):  # warm-up prompts (no invocation)
        stack.forward_prompt(x, logits_of(q), out, hits)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        st = run_stream(stack, trace, trace_dev, prompt_tasks, x, logits_of, P_train, P_serve,
                        residency=args.residency)
    nmat = 3
    served = None
    flops_note = f"2*{nmat}*d*f per served (token, expert) per layer"
    res = dict(metric=METRIC, value=round(st["tokens_per_s"], 1), unit="tokens/s", n_gpus=1, steps=P_serve,
               warmup=args.warmup, ms_per_step=round(st["ms"] / P_serve, 3), higher_is_better=True, scaling="weak",
               vs_baseline=None, dtype="bf16", data="synthetic (random-init weights; gate computed on x, routing "
                                                   "biased to the reference Markov trace)",
               config=dict(per_expert_seconds=cfg.per_expert_seconds, workload=("BASELINE config 5: mixed-task stream, 8k-token prompts, %d-layer "
                                     "Mixtral-shaped stack, phi=0.5, p=40, predictor skipped for insensitive "
                                     "windows, loads overlapped" % m) if args.residency == "predicted" else
                           ("BASELINE config 5 stream, %d-layer Mixtral-shaped stack, phi=0.5, ON-DEMAND "
                            "residency baseline (engine.cpp:469-502): per layer keep the experts the prompt "
                            "demands most, load missing ones synchronously" % m),
                           residency=args.residency, prompts=P_serve, tokens_per_prompt=T,
                           layers=m, tasks={n: dict(wo=t.wo, sensitive_layers=sum(t.sensitivity))
                                            for n, t in tasks.items()}),
               stream=dict((kk, v) for kk, v in st.items() if kk not in ("ms",)), clocks=clk.summary(),
               note=flops_note, served=served)
    print(json.dumps(res), flush=True)
    stack.close()


def main_stack(args):
    """BASELINE config 4: a 32-layer Mixtral-shaped stack (E=8, top-2, 4
    predicted-resident experts per layer, bf16), 32 x 2048 tokens per GPU per
    step, layers chained (y of layer l is x of layer l+1) on one shared
    activation workspace.  Every layer runs its gate on its input (random
    N(0, 1/d) gate weights); the reference Markov trace is added to the
    gate's logits as a bias (EMOE_LOGITS_ADD), so routing follows the trace
    the predictor was fitted on while the gate's arithmetic is real.
    Resident sets from one GPU predictor invocation (fit over the ranks'
    shards, merged by one all-reduce).  A step = the forward through all
    layers + the A6 histogram update of the batch.
    N > 1, --parallel ep (default): expert parallelism, every layer its own
    load-aware placement (plan_shares of its Eq. 2 aggregate), all layers on
    one symmetric peer-memory region; --parallel replicas: each GPU holds the
    resident sets.  Weak scaling (every GPU its own 32 x 2048 tokens) unless
    --scaling strong."""
    import torch
    import torch.distributed as dist

    import paper_2503_06823_b200 as emoe
    from paper_2503_06823_b200 import _lib
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE, owned_experts, plan_shares
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig, TaskSpec, moesim_prompt_sets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        nccl_log_to_stderr()
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    m, E, k, L, d, f, P, Tp = args.stream_layers, 8, 2, 4, 4096, 14336, 32, 2048
    strong = args.scaling == "strong" and world > 1
    use_ep = args.parallel == "ep" and (world > 1 or args.ep_at_1)
    ensure_group_for_ep_at_1(args, world)
    if use_ep and args.ep_transport != "p2p":
        raise SystemExit("--config stack: expert parallelism runs the p2p transport")
    if strong and P % world:
        raise SystemExit(f"--scaling strong: {world} GPUs do not divide the {P} prompts")
    Pr = P // world if strong else P  # prompts this rank serves
    T = Pr * Tp
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=T, period=40, mode=0,
                       tasks={"conv": TaskSpec(256.0, [1] * m)})
    P_train = 60
    trace = emoe.gen_routing_trace(emoe.ModelShape(m, E, k), 0.6, 0.8, 0, 17, P_train + Pr * world, Tp)
    g = torch.Generator(device=device).manual_seed(1234)
    host = [tuple((torch.randn(*sh, generator=g, device=device) / sh[1] ** 0.5).to(torch.bfloat16).cpu()
                  .pin_memory() for sh in ((f, d), (f, d), (d, f))) for _ in range(E)]
    gates = [(torch.randn(E, d, generator=g, device=device) / d ** 0.5).to(torch.bfloat16).cpu() for _ in range(m)]
    stack = MoEStack(cfg, host, gates)
    for layer in stack.layers:
        layer.set_logits_mode("add")
    trace_dev = torch.from_numpy(trace).to(device)
    stack.fit(trace_dev[:P_train].contiguous(), ["conv"] * P_train,
              group=dist.group.WORLD if dist.is_initialized() and dist.get_world_size() > 1 else None)
    _, sets = moesim_prompt_sets(trace_dev, P_train - 1)
    ops, agg, _ = stack.invocation(sets, [("conv", Tp)] * P)
    eps = []
    if use_ep:  # every layer: its resident set spread over the ranks by its own Eq. 2 loads
        for l, layer in enumerate(stack.layers):
            res_l = sorted(ops[l][1])  # the plan's loads onto an empty GPU = the resident set
            layer.begin_load([], owned_experts(plan_shares(res_l, E, world, agg[l]), rank))
            eps.append(PeerExpertParallelMoE(layer, res_l, loads=agg[l], share_with=eps[0] if eps else None,
                                             recv_rows_cap=args.ep_recv_cap))
    else:
        stack.apply(ops)
    stack.set_scores(agg)
    for layer in stack.layers:
        layer.poll_loads(blocking=True)
    torch.cuda.synchronize()
    serve = trace_dev[P_train + rank * Pr: P_train + (rank + 1) * Pr].contiguous()  # [Pr][m][Tp][k]
    ch = serve.permute(1, 0, 2, 3).reshape(m, T, k).long()
    lg = torch.round((torch.rand(m, T, E, generator=g, device=device) * 8.0 - 4.0) * 64) / 64
    for r in range(k):
        lg.scatter_(2, ch[:, :, r:r + 1], 8.0 - r)
    lg *= 16.0  # the trace bias dominates the gate's own logits (~N(0, |x|^2 / d))
    x = torch.randn(T, d, generator=g, device=device).to(torch.bfloat16)
    bufs = [torch.empty_like(x), torch.empty_like(x)]
    tid = torch.zeros(Pr, dtype=torch.int32, device=device)
    stream = torch.cuda.current_stream()
    import ctypes as C

    def step(src=None):
        h = x if src is None else src
        for l, layer in enumerate(stack.layers):
            if use_ep:
                h = eps[l](h, logits=lg[l], out=bufs[l % 2])
            else:
                h = layer.forward(h, logits=lg[l], out=bufs[l % 2])
        emoe.moesim.check(_lib.lib.emoe_hist_update(stack.pred.h, C.c_void_p(serve.data_ptr()), Pr, Tp,
                                                    C.c_void_p(tid.data_ptr()), C.c_void_p(stream.cuda_stream)))
        return h

    # served rows and hits per layer of one step
    S_total, hits = 0, 0
    h = x
    for l, layer in enumerate(stack.layers):
        h = eps[l](h, logits=lg[l], out=bufs[l % 2]) if use_ep else layer.forward(h, logits=lg[l], out=bufs[l % 2])
        ws = layer.workspace()
        S_total += int(ws["counts"].sum().item())
        hits += int(ws["route_hit"].sum().item())
    topk_match = bool(torch.equal(stack.layers[-1].workspace()["topk_idx"].long(), ch[-1]))
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    for obj in (eps if use_ep else stack.layers):
        obj.set_profiling(True)
    launches0 = _lib.lib.emoe_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = int(_lib.lib.emoe_kernel_launches() - launches0)
    ms = ev0.elapsed_time(ev1) / args.steps
    stages, ep_stats = {}, None
    for obj in (eps if use_ep else stack.layers):
        for key, v in obj.stage_times().items():
            stages[key] = stages.get(key, 0.0) + v
        obj.set_profiling(False)
    if use_ep:
        ep_stats = {}
        for ep in eps:
            for key, v in ep.stats().items():
                ep_stats[key] = ep_stats.get(key, 0) + v
        gemm_ms = stages["gemm1"] + stages["gemm2_return"]
        S_ffn = ep_stats["rows_computed_real"]
    else:
        gemm_ms = stages["gemm1"] + stages["gemm2"]
        S_ffn = S_total
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * T / (ms / 1e3)
    # end to end: pinned host x in, the stack, y back to host, every step
    x_host = x.cpu().pin_memory()
    y_host = torch.empty_like(x_host).pin_memory()
    x_dev = torch.empty_like(x)
    e2e_steps = max(2, args.steps // 2)
    step(x_dev.copy_(x_host, non_blocking=True))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        y_host.copy_(step(x_dev.copy_(x_host, non_blocking=True)), non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    peaks = load_peaks()
    ffn_flops = 2.0 * 3 * d * f * S_ffn
    achieved = ffn_flops / (gemm_ms / 1e3) / 1e12
    out = dict(metric=METRIC, value=round(value, 1), unit="tokens/s", n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(ms, 3), higher_is_better=True,
               scaling="strong" if strong else "weak", vs_baseline=None, dtype="bf16",
               data="synthetic (random-init weights; gate computed on x, routing biased to the reference Markov "
                    "trace)",
               config=dict(workload=f"BASELINE config 4: {m}-layer Mixtral-shaped MoE stack bf16, 8 experts top-2, "
                                    f"4 predicted resident per layer, {Pr} x {Tp} tokens per GPU through every layer",
                           layers=m, tokens_per_step=T, served_rows_all_layers=S_total,
                           hit_rate=round(hits / (T * m), 4), routing_follows_trace=topk_match,
                           workspace="one shared activation workspace" + (
                               " + one shared EP peer-memory region" if use_ep else ""),
                           parallelism=parallelism_label(world, args.parallel, "p2p"),
                           l2="inputs larger than L2: x is %.0f MB per layer" % (T * d * 2 / 1e6)),
               roofline=dict(bound="tensor", achieved=round(achieved, 1), peak=peaks["bf16_sustained"],
                             unit="TFLOP/s", frac=round(achieved / peaks["bf16_sustained"], 4),
                             kernel="grouped_gemm_kernel (GEMM1 + GEMM2 of every layer), stage events",
                             algorithmic=f"2*3*d*f*S summed over layers = {ffn_flops:.4g} FLOP per step "
                                         f"(S = {S_ffn} rows computed on this GPU)"),
               e2e=dict(value=world * T / e2e_s, unit="tokens/s", h2d_bytes_per_step=x_host.numel() * 2,
                        d2h_bytes_per_step=y_host.numel() * 2, ms_per_step=e2e_s * 1e3),
               gpu_launches=launches, clocks=clk.summary(), per_layer_ms=round(ms / m, 3),
               stages_ms={kk: round(v, 3) for kk, v in stages.items()},
               resident_per_layer=[[int(e) for e in np.flatnonzero(layer.residency())] for layer in stack.layers[:4]])
    if use_ep:
        out["ep"] = ep_report(eps, stages, ep_stats, world, rank, device)
    if rank == 0:
        print(json.dumps(out), flush=True)
    for ep in eps:
        ep.close()
    stack.close()
    if world > 1:
        dist.destroy_process_group()


def main_reference(args, cfg, rank, world):
    """--impl reference: the reference's CPU implementation of the path on this
    host's cores, on bounded samples of the same workload.  It never imports
    the product package: the routing trace comes from the reference's own
    generator (oracle/_ref, workload.cpp:242-286), the resident set from the
    reference's fit / prompt_expert_sets / predict / predicted_frequencies /
    loading_targets (oracle/_ref) with the engine's invocation aggregate
    (engine.cpp:367-417, oracle port), the inputs from the same CPU generator
    as the GPU arm (input_gate / input_expert / input_x: same seeds, same
    bits; input_digest proves it), route_token from oracle/_ref and gate /
    permute / FFN / combine from the oracle port."""
    if rank != 0:
        return
    import torch

    from oracle.oracle import Port, Ref, have_ref

    if not have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the reference build) is missing"}))
        return
    port, ref = Port(), Ref()
    threads = port.threads()
    E, k, d, f, L = cfg["E"], cfg["k"], cfg["d"], cfg["f"], cfg["L"]
    P, Tp, P_train = cfg["prompts"], cfg["tokens"], cfg["train"]
    T = P * Tp
    trace = ref.gen_routing_trace(1, E, k, cfg["layer_lambda"], cfg["prompt_lambda"], 0, cfg["seed"],
                                  P_train + P, Tp)
    train = trace[:P_train]
    model = ref.fit(train, np.zeros(P_train, np.int32), ["t0"], 0.01, E)
    _, sets, sizes = ref.prompt_expert_sets(train, P_train - 1)
    scores, _, _ = ref.predict(model, 0, sets, sizes, k=k)
    fitted = ref.predicted_frequencies(model["task_counts"], ["t0"], 0.01, "t0")[None]
    agg = port.invocation_aggregate(scores, fitted, [128.0], np.ones((1, 1), np.int32), [1],
                                    np.zeros(P, np.int32), np.full(P, Tp))
    targets = ref.loading_targets(agg, np.zeros((1, E), np.uint8), [L])[0]
    resident = [1 if e in targets else 0 for e in range(E)]
    choices = trace[P_train:].reshape(-1, k)
    info = dict(resident=resident, choices=choices, aggregate=agg[0].tolist())
    wg64 = input_gate(cfg)
    wg = wg64.to(torch_dtype(cfg))
    experts = {e: input_expert(cfg, e) for e in range(E) if resident[e]}
    rows = min(X_CHUNK, T)
    x_rows = input_x(cfg, wg64, choices, rows)
    digest = input_digest(x_rows[:DIGEST_ROWS], wg, experts)
    xs, wgf, ex = f32_inputs(x_rows, wg, experts)
    # size the per-step sample so W+K steps finish within a few minutes
    n = min(16, rows)
    dt = cpu_reference_step(cfg, info, xs, wgf, ex, n, port, ref, threads)
    budget_s = args.ref_budget_s / (args.steps + args.warmup)
    n = int(max(min(4, rows), min(rows, n * budget_s / max(dt, 1e-3))))
    for _ in range(args.warmup):
        cpu_reference_step(cfg, info, xs, wgf, ex, n, port, ref, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_reference_step(cfg, info, xs, wgf, ex, n, port, ref, threads)
    s = (time.perf_counter() - t0) / args.steps
    value = n / s
    sample = (f"the first {n} of the {P}x{Tp} = {T} tokens per step (same x rows, weights and resident set as "
              f"the GPU arm; input_digest {digest}): {CPU_PATH_NOTE}; {threads} host threads")
    out = dict(metric=METRIC, impl="reference", value=round(value, 3), unit="tokens/s", n_gpus=world,
               steps=args.steps, warmup=args.warmup, ms_per_step=round(s * 1e3, 3), higher_is_better=True,
               scaling="weak", vs_baseline=None, dtype="fp32 (fp64 accumulate)", data="synthetic",
               config=dict(workload=cfg["workload"], tokens_per_step=n, parallelism="cpu",
                           resident_set=[e for e in range(E) if resident[e]], input_digest=digest,
                           same_config=True),
               cpu_baseline=dict(value=round(value, 3), unit="tokens/s", cores=threads, kind="port", sample=sample),
               e2e=dict(value=round(value, 3), unit="tokens/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
