"""Expert parallelism: the exchange logic (plan, segment-size exchange,
dispatch/return all-to-all, per-(source, expert) segments) is checked with
world-size 2 and 4 gloo groups on CPU using the oracle as the local compute,
and on the GPU with 2 ranks sharing cuda:0 over gloo (real kernels).  EP=G
output must be bit-identical to EP=1 on the same tokens."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2503_06823_b200.ep import (SHARE_ONE, ExpertParallelMoE, RoutedBatch, owned_experts,  # noqa: E402
                                      p2p_layout, plan_shares)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleBackend:
    """Local compute through the CPU oracle (tests only)."""

    def __init__(self, port, E, k, d, f, global_resident, pad=4, seed=0):
        rng = np.random.default_rng(seed)
        self.port, self.E, self.k, self.d, self.f, self.pad = port, E, k, d, f, pad
        self.wg = (rng.standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
        self.experts = [((rng.standard_normal((f, d)) / np.sqrt(d)).astype(np.float32),
                         (rng.standard_normal((f, d)) / np.sqrt(d)).astype(np.float32),
                         (rng.standard_normal((d, f)) / np.sqrt(f)).astype(np.float32)) for _ in range(E)]
        self.resident = np.zeros(E, np.uint8)
        self.resident[list(global_resident)] = 1

    def route_permute(self, x):
        xn = x.numpy()
        o = self.port.gate_route(self.port.gate_logits(xn, self.wg), self.k, 0, self.resident)
        counts, offsets, pos, src = self.port.permute(o["served_idx"], self.E, self.pad)
        rows = np.zeros((int(offsets[-1]), self.d), np.float32)
        valid = src >= 0
        rows[valid] = xn[src[valid]]
        return RoutedBatch(offsets, torch.from_numpy(rows), torch.from_numpy(pos.astype(np.int32)),
                           torch.from_numpy(o["served_w"]), x.shape[0], counts.astype(np.int64))

    def ffn(self, rows, seg_offsets, seg_expert):
        y = np.zeros((rows.shape[0], self.d), np.float32)
        rn = rows.numpy()
        for i, e in enumerate(seg_expert):
            a, b = int(seg_offsets[i]), int(seg_offsets[i + 1])
            w1, w3, w2 = self.experts[e]
            y[a:b] = self.port.expert_ffn(rn[a:b], w1, w3, w2, 0, False, 1)
        return torch.from_numpy(y)

    def combine(self, y_rows, batch):
        return torch.from_numpy(self.port.combine(y_rows.numpy(), batch.pos.numpy().astype(np.int64),
                                                  batch.served_w.numpy(), False))


def single(backend, x):
    b = backend.route_permute(x)
    seg = b.seg_offsets
    nz = [e for e in range(backend.E) if seg[e + 1] > seg[e]]
    so = np.array([seg[e] for e in nz] + [seg[-1]], np.int64)
    y = backend.ffn(b.rows, so, np.array(nz, np.int32))
    return backend.combine(y, b)


def _cpu_worker(rank, world, port_no, resident, out_dir, loads=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port

    be = OracleBackend(Port(), E=8, k=2, d=64, f=128, global_resident=resident)
    x = torch.from_numpy(np.random.default_rng(100 + rank).standard_normal((37 + 5 * rank, 64)).astype(np.float32))
    ep = ExpertParallelMoE(be, resident, loads=loads)
    y_ep = ep(x)
    y_1 = single(be, x)
    np.save(Path(out_dir) / f"r{rank}.npy", np.stack([y_ep.numpy(), y_1.numpy()]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,resident,skew", [(2, [0, 2, 5, 7], False), (4, [1, 6], False),
                                                  (4, [0, 1, 2, 3, 4, 5, 6, 7], False), (2, [3], False),
                                                  (4, [0, 2, 5, 7], True)])
def test_ep_gloo_cpu_bit_identical(world, resident, skew, tmp_path):
    loads = [1, 0, 1, 0, 0, 1, 0, 20] if skew else None  # skew: expert 7 spans most ranks
    mp.spawn(_cpu_worker, args=(world, free_port(), resident, str(tmp_path), loads), nprocs=world, join=True)
    for r in range(world):
        y_ep, y_1 = np.load(tmp_path / f"r{r}.npy")
        assert np.array_equal(y_ep, y_1), f"rank {r}: EP output differs from EP=1"


STACK = [([0, 2, 5, 7], [1, 0, 1, 0, 0, 1, 0, 20]), ([1, 6], None), ([0, 1, 2, 3, 4, 5, 6, 7], list(range(1, 9)))]


def _cpu_stack_worker(rank, world, port_no, out_dir):
    """A 3-layer stack (config 4's shape in miniature): every layer its own
    resident set and load-aware plan, y of layer l is x of layer l+1."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port

    port = Port()
    layers = [OracleBackend(port, E=8, k=2, d=64, f=128, global_resident=res, seed=l)
              for l, (res, _) in enumerate(STACK)]
    eps = [ExpertParallelMoE(be, res, loads=loads) for be, (res, loads) in zip(layers, STACK)]
    x = torch.from_numpy(np.random.default_rng(300 + rank).standard_normal((53 + 9 * rank, 64)).astype(np.float32))
    h_ep, h_1 = x, x
    for be, ep in zip(layers, eps):
        h_ep = ep(h_ep)
        h_1 = single(be, h_1)
    np.save(Path(out_dir) / f"s{rank}.npy", np.stack([h_ep.numpy(), h_1.numpy()]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_stack_gloo_cpu_bit_identical(world, tmp_path):
    mp.spawn(_cpu_stack_worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        y_ep, y_1 = np.load(tmp_path / f"s{r}.npy")
        assert np.array_equal(y_ep, y_1), f"rank {r}: stack EP output differs from EP=1"


SKEW = np.array([1, 0, 1, 0, 0, 1, 0, 20], np.float64)  # expert 7 carries most rows


def _rank_ranges(cum):
    """[first, last] rank of every resident expert."""
    out = {}
    for e in range(cum.shape[0]):
        if cum[e, 0] < 0:
            continue
        prev = np.concatenate([[0], cum[e, :-1]])
        q = np.flatnonzero(cum[e] > prev)
        out[e] = (int(q[0]), int(q[-1]))
    return out


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("resident", [[0, 2, 5, 7], list(range(8)), [7], [1, 6]])
def test_plan_shares(world, resident):
    rng = np.random.default_rng(world * 31 + len(resident))
    for loads in (None, SKEW, rng.random(8) * 100, np.zeros(8), np.array([0, 0, 5, 0, 0, 0, 0, 0.0])):
        cum = plan_shares(resident, 8, world, loads)
        for e in range(8):
            if e not in resident:
                assert (cum[e] == -1).all()
                continue
            assert (np.diff(cum[e]) >= 0).all() and cum[e, -1] == SHARE_ONE and cum[e, 0] >= 0
        rr = _rank_ranges(cum)
        # consecutive experts never go back to an earlier rank (contiguous NCCL chunks)
        es = sorted(rr)
        assert all(rr[a][1] <= rr[b][0] for a, b in zip(es, es[1:])), rr
        # every rank's expected load within min_share of a fair share
        w = np.ones(len(resident)) if loads is None or np.sum([loads[e] for e in resident]) <= 0 else \
            np.array([loads[e] for e in resident], float)
        w = w / w.sum() * world
        per = np.zeros(world)
        for i, e in enumerate(sorted(resident)):
            frac = np.diff(np.concatenate([[0], cum[e]])) / SHARE_ONE
            per += frac * w[i]
        assert per.max() <= 1.0 + 2 * 0.05 + 1e-6 or len(resident) * 1 < 1, (per, loads)
        assert sum(len(owned_experts(cum, q)) for q in range(world)) >= len(resident)
    # a heavy expert spans several ranks; light ones share one
    cum = plan_shares([0, 2, 5, 7], 8, 8, SKEW)
    assert sum(7 in owned_experts(cum, q) for q in range(8)) >= 6
    cum = plan_shares([0, 5, 6, 7], 8, 8)  # 4 resident, 8 ranks, equal: two ranks per expert, half each
    assert [owned_experts(cum, q) for q in range(8)] == [[0], [0], [5], [5], [6], [6], [7], [7]]
    assert all(cum[e, 2 * i] == SHARE_ONE // 2 for i, e in enumerate([0, 5, 6, 7]))


def test_split_balances_per_source_skew():
    """Token-level split: whatever the per-source skew of a replicated expert's
    rows, its ranks compute their share of the total (within one pad)."""
    rng = np.random.default_rng(3)
    W, E, pad = 8, 8, 4
    cum = plan_shares([0, 5, 6, 7], E, W, SKEW)
    for _ in range(20):
        counts = np.zeros((W, E), np.int64)
        for e in [0, 5, 6, 7]:
            counts[:, e] = rng.integers(0, 200, W) * (1 + 9 * (e == 7)) * rng.integers(1, 4, W)
        lays = [p2p_layout(counts, cum, q, pad) for q in range(W)]
        tot = lays[0]["tot"]
        cp = (counts + pad - 1) // pad * pad
        for e in [0, 5, 6, 7]:
            frac = np.diff(np.concatenate([[0], cum[e]])) / SHARE_ONE
            got = np.zeros(W, np.int64)
            for q in range(W):
                segs, exp = lays[q]["recv_segs"], lays[q]["seg_expert"]
                got[q] = sum(segs[i + 1] - segs[i] for i in range(len(exp)) if exp[i] == e)
            assert got.sum() == cp[:, e].sum()
            assert np.all(np.abs(got - frac * cp[:, e].sum()) <= pad + 1e-9), (e, got, frac)
        assert np.array_equal(tot.sum(axis=0), [lays[q]["recv_segs"][-1] for q in range(W)])


def _gpu_worker(rank, world, port_no, resident, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import LayerBackend

    mine = owned_experts(plan_shares(resident, 8, world), rank)
    # EP layer: only this rank's experts in HBM, routing against the global set
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(mine), mine, max_tokens=2048)
    ep = ExpertParallelMoE(LayerBackend(layer, resident), resident)
    x = torch.randn(1500 + 100 * rank, 256, generator=torch.Generator().manual_seed(rank)).to(torch.bfloat16).cuda()
    y_ep = ep(x).cpu()
    # EP=1 reference: one layer holding the whole resident set
    full, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(resident), resident,
                             max_tokens=2048)
    y_1 = full.forward(x).cpu()
    torch.save(dict(y_ep=y_ep, y_1=y_1, last=ep.last), Path(out_dir) / f"g{rank}.pt")
    layer.close()
    full.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("resident", [[0, 2, 5, 7], [3]])
def test_ep_two_ranks_one_gpu_bit_identical(resident, tmp_path):
    mp.spawn(_gpu_worker, args=(2, free_port(), resident, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        d = torch.load(tmp_path / f"g{r}.pt", weights_only=False)
        assert torch.equal(d["y_ep"], d["y_1"]), f"rank {r}: EP output differs from the single-GPU forward"


# ---------------------------------------------------------------------------
# expert parallelism over peer memory (csrc/ep.cu)
# ---------------------------------------------------------------------------
def _simulate_p2p(backends, xs, cum):
    """CPU restatement of the peer-memory protocol: every rank publishes its
    counts, computes p2p_layout, 'stores' its rows piece by piece into the
    computing ranks' receive buffers, those run the FFN over their (source,
    expert) segments and push the outputs back into each source's permuted
    layout, and each source combines locally."""
    W = len(backends)
    E, pad = backends[0].E, backends[0].pad
    batches = [b.route_permute(x) for b, x in zip(backends, xs)]
    counts = np.stack([bt.counts for bt in batches])
    lays = [p2p_layout(counts, cum, r, pad) for r in range(W)]
    recv = [np.full((int(lays[q]["recv_segs"][-1]), backends[0].d), np.nan, np.float32) for q in range(W)]
    for r, bt in enumerate(batches):
        assert np.array_equal(lays[r]["seg_offsets"], bt.seg_offsets)
        pe, ps = lays[r]["piece_end"], lays[r]["piece_shift"]
        for e in range(E):
            start = int(bt.seg_offsets[e])
            for q in range(W):
                end = int(pe[e, q])
                if end > start:
                    recv[q][start + ps[e, q]:end + ps[e, q]] = bt.rows[start:end].numpy()
                start = max(start, end)
            assert start == bt.seg_offsets[e + 1], "pieces must cover the segment"
    y_local = [np.full((int(bt.seg_offsets[-1]), backends[0].d), np.nan, np.float32) for bt in batches]
    for q in range(W):
        lay = lays[q]
        segs, exp, src, out_shift = lay["recv_segs"], lay["seg_expert"], lay["seg_src"], lay["out_shift"]
        if not len(exp):
            continue
        out = backends[q].ffn(torch.from_numpy(np.nan_to_num(recv[q])), segs, exp).numpy()
        for i in range(len(exp)):
            a, b = int(segs[i]), int(segs[i + 1])
            if b > a:
                y_local[src[i]][a + out_shift[i]:b + out_shift[i]] = out[a:b]
    ys = []
    for r, bt in enumerate(batches):
        pos = bt.pos.numpy().astype(np.int64)
        served = pos[pos >= 0]
        assert not np.isnan(y_local[r][served]).any(), "a served row was never returned"
        ys.append(backends[r].combine(torch.from_numpy(np.nan_to_num(y_local[r])),
                                      RoutedBatch(bt.seg_offsets, None, torch.from_numpy(pos), bt.served_w, bt.T)))
    return ys, lays


@pytest.mark.parametrize("world,resident,loads", [(2, [0, 2, 5, 7], None), (4, [1, 6], None),
                                                   (4, list(range(8)), None), (2, [3], None),
                                                   (2, [0, 2, 5, 7], SKEW), (4, [0, 2, 5, 7], SKEW),
                                                   (3, list(range(8)), SKEW), (8, [0, 5, 6, 7], SKEW)])
def test_p2p_layout_protocol_bit_identical(world, resident, loads, port):
    be = [OracleBackend(port, E=8, k=2, d=64, f=128, global_resident=resident) for _ in range(world)]
    xs = [torch.from_numpy(np.random.default_rng(200 + r).standard_normal((41 + 7 * r, 64)).astype(np.float32))
          for r in range(world)]
    cum = plan_shares(resident, 8, world, loads)
    ys, lays = _simulate_p2p(be, xs, cum)
    for r in range(world):
        assert np.array_equal(ys[r].numpy(), single(be[r], xs[r]).numpy()), f"rank {r}: P2P layout output differs"
    for q, lay in enumerate(lays):
        segs = lay["recv_segs"]
        assert np.all(np.diff(segs) >= 0) and np.all(segs % be[0].pad == 0)
        assert len(lay["seg_expert"]) == world * len(owned_experts(cum, q))


def test_p2p_layout_disjoint_writes():
    """Within every receiver, the row ranges written by different (source,
    expert, piece) writes are disjoint and tile [0, total); the return pushes
    tile each source's own padded segments exactly."""
    rng = np.random.default_rng(5)
    pad = 4
    for world, resident, loads in [(2, [0, 2, 5, 7], None), (4, [1, 6], None), (8, [0, 5, 6, 7], None),
                                   (8, list(range(8)), None), (8, [0, 2, 5, 7], SKEW), (4, list(range(8)), SKEW),
                                   (8, [3], None), (5, [0, 1, 7], rng.random(8))]:
        cum = plan_shares(resident, 8, world, loads)
        for _ in range(5):
            counts = rng.integers(0, 17, (world, 8)) * (cum[:, 0] >= 0)
            lays = [p2p_layout(counts, cum, q, pad) for q in range(world)]
            written = {q: [] for q in range(world)}
            for r in range(world):
                seg, pe, ps = lays[r]["seg_offsets"], lays[r]["piece_end"], lays[r]["piece_shift"]
                for e in range(8):
                    start = int(seg[e])
                    for q in range(world):
                        end = int(pe[e, q])
                        if end > start:
                            written[q].append((start + ps[e, q], end + ps[e, q]))
                        start = max(start, end)
            pushed = {r: [] for r in range(world)}
            for q in range(world):
                segs, src, osh = lays[q]["recv_segs"], lays[q]["seg_src"], lays[q]["out_shift"]
                iv = sorted(written[q])
                assert all(a[1] == b[0] for a, b in zip(iv, iv[1:])), (world, q, iv)
                assert (iv[0][0] if iv else 0) == 0 and (iv[-1][1] if iv else 0) == segs[-1]
                for i in range(len(src)):
                    if segs[i + 1] > segs[i]:
                        pushed[int(src[i])].append((segs[i] + osh[i], segs[i + 1] + osh[i]))
            for r in range(world):
                seg = lays[r]["seg_offsets"]
                got = sorted(pushed[r])
                assert all(x[1] <= y[0] for x, y in zip(got, got[1:])), (world, r, got)  # no overlap
                assert _merge(got) == _merge([(seg[e], seg[e + 1]) for e in range(8) if seg[e + 1] > seg[e]])


def _merge(iv):
    out = []
    for a, b in sorted(iv):
        if out and out[-1][1] == a:
            out[-1] = (out[-1][0], b)
        else:
            out.append((a, b))
    return out


def _gpu_p2p_worker(rank, world, port_no, resident, out_dir, loads=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    os.environ.setdefault("EMOE_EP_TIMEOUT_S", "120")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE

    cum = plan_shares(resident, 8, world, loads)
    mine = owned_experts(cum, rank)
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(mine), mine, max_tokens=2048)
    ep = PeerExpertParallelMoE(layer, resident, loads=loads)
    assert np.array_equal(ep.cum, cum)
    full, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(resident), resident,
                             max_tokens=2048)
    res = []
    for it, T in enumerate([1500 + 100 * rank, 700 - 50 * rank, 2048]):  # epochs reuse the buffers
        x = torch.randn(T, 256, generator=torch.Generator().manual_seed(10 * it + rank)).to(torch.bfloat16).cuda()
        y_ep = ep(x)
        st, rows = ep.status()
        # the device layout (ep_bar0_kernel) against its numpy restatement on
        # the all-gathered counts
        counts = layer.workspace()["counts"].cpu().to(torch.int64)
        table = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(table, counts)
        want = p2p_layout(torch.stack(table).numpy(), cum, rank, layer.seg_pad)
        got = ep.layout()
        same = all(np.array_equal(got[key], want[key]) for key in ("piece_end", "piece_shift", "recv_segs",
                                                                    "out_shift"))
        stats = ep.stats()
        y_1 = full.forward(x)
        torch.cuda.synchronize()
        res.append(dict(y_ep=y_ep.cpu(), y_1=y_1.cpu(), status=st, rows=rows, layout_same=same, stats=stats,
                        tot=want["tot"]))
    torch.save(res, Path(out_dir) / f"p{rank}.pt")
    dist.barrier()
    ep.close()
    layer.close()
    full.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("resident,loads", [([0, 2, 5, 7], None), ([3], None), ([0, 2, 5, 7], SKEW),
                                           ([1, 6], [0, 1, 0, 0, 0, 0, 3, 0])])
def test_ep_p2p_two_ranks_one_gpu_bit_identical(resident, loads, tmp_path):
    """SKEW: expert 7 is split token by token over both ranks while experts
    0, 2 and 5 live on rank 0; [3]: one expert split in half."""
    mp.spawn(_gpu_p2p_worker, args=(2, free_port(), resident, str(tmp_path), loads), nprocs=2, join=True)
    for r in range(2):
        for i, d in enumerate(torch.load(tmp_path / f"p{r}.pt", weights_only=False)):
            assert d["status"] == 0, f"rank {r} forward {i}: status {d['status']}"
            assert d["rows"] > 0 and d["rows"] == d["tot"][:, r].sum()
            assert d["layout_same"], f"rank {r} forward {i}: device layout differs from p2p_layout"
            assert 0 <= d["stats"]["rows_sent_to_peers"] <= d["stats"]["rows_routed"]
            assert torch.equal(d["y_ep"], d["y_1"]), f"rank {r} forward {i}: P2P EP output differs from 1 GPU"


def _gpu_p2p_fault_worker(rank, world, port_no, case, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no), EMOE_EP_TIMEOUT_S="2")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE

    resident = [0, 2, 5, 7]
    mine = owned_experts(plan_shares(resident, 8, world), rank)
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(mine), mine, max_tokens=2048)
    ep = PeerExpertParallelMoE(layer, resident, recv_rows_cap=256 if case == "overflow" else 0)
    x = torch.randn(1500, 256, generator=torch.Generator().manual_seed(rank)).to(torch.bfloat16).cuda()
    res = {}
    if case == "overflow" or rank == 0:  # "timeout": rank 1 never joins the forward
        y = ep(x)
        res["status"], res["rows"] = ep.status()
        res["finite"] = bool(torch.isfinite(y.float()).all())
    torch.save(res, Path(out_dir) / f"f{rank}.pt")
    dist.barrier()
    ep.close()
    layer.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["overflow", "timeout"])
def test_ep_p2p_fault_status(case, tmp_path):
    """A receive buffer too small for the routed rows drops them and reports
    status 2 on every rank (all ranks derive the same layout); a peer that
    never arrives makes the barrier give up after EMOE_EP_TIMEOUT_S with
    status 1 instead of hanging the GPU."""
    mp.spawn(_gpu_p2p_fault_worker, args=(2, free_port(), case, str(tmp_path)), nprocs=2, join=True)
    r0 = torch.load(tmp_path / "f0.pt", weights_only=False)
    if case == "overflow":
        r1 = torch.load(tmp_path / "f1.pt", weights_only=False)
        assert r0["status"] == 2 and r1["status"] == 2
        assert r0["finite"] and r1["finite"]
    else:
        assert r0["status"] == 1


def _gpu_p2p_single_worker(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE

    resident = [1, 2, 6]
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 3, resident, max_tokens=1024)
    ep = PeerExpertParallelMoE(layer, resident)
    full, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 3, resident, max_tokens=1024)
    x = torch.randn(1000, 256, generator=torch.Generator().manual_seed(2)).to(torch.bfloat16).cuda()
    y_ep = ep(x)
    st, rows = ep.status()
    torch.save(dict(y_ep=y_ep.cpu(), y_1=full.forward(x).cpu(), status=st), Path(out_dir) / "s.pt")
    ep.close()
    layer.close()
    full.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_ep_p2p_single_rank(tmp_path):
    """World size 1: the peer-memory path degenerates to local stores and a
    self-barrier and still equals the plain forward."""
    mp.spawn(_gpu_p2p_single_worker, args=(1, free_port(), str(tmp_path)), nprocs=1, join=True)
    d = torch.load(tmp_path / "s.pt", weights_only=False)
    assert d["status"] == 0
    assert torch.equal(d["y_ep"], d["y_1"])


# ---------------------------------------------------------------------------
# a layer stack under expert parallelism (config 4's shape in miniature)
# ---------------------------------------------------------------------------
GPU_STACK = [([0, 2, 5, 7], SKEW), ([1, 6], None), ([3, 4, 5, 6], [0, 0, 0, 1, 2, 3, 4, 0])]


def _gpu_stack_worker(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no), EMOE_EP_TIMEOUT_S="120")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE
    from paper_2503_06823_b200.serving import MoEStack, StreamConfig

    m, E, k, d, f = len(GPU_STACK), 8, 2, 256, 512
    cfg = StreamConfig(m=m, E=E, k=k, L=4, d=d, f=f, tokens_per_prompt=2048, period=4, mode=0, tasks={})
    g = torch.Generator().manual_seed(11)  # the same weights on every rank
    host = [tuple((torch.randn(*s, generator=g) / s[1] ** 0.5).to(torch.bfloat16).pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    gates = [(torch.randn(E, d, generator=g) / d ** 0.5).to(torch.bfloat16) for _ in range(m)]
    ep_stack, ref_stack = MoEStack(cfg, host, gates), MoEStack(cfg, host, gates)
    eps = []
    for l, (res, loads) in enumerate(GPU_STACK):
        ep_stack.layers[l].load_initial(owned_experts(plan_shares(res, E, world, loads), rank))
        eps.append(PeerExpertParallelMoE(ep_stack.layers[l], res, loads=loads, share_with=eps[0] if eps else None))
        ref_stack.layers[l].load_initial(res)
    out = []
    for it, T in enumerate([1500 + 100 * rank, 900 - 300 * rank, 2048]):
        x = torch.randn(T, d, generator=torch.Generator().manual_seed(50 * it + rank)).to(torch.bfloat16).cuda()
        h_ep, h_1, same = x, x, []
        for l in range(m):
            h_ep = eps[l](h_ep)
            h_1 = ref_stack.layers[l].forward(h_1)
            same.append(bool(torch.equal(h_ep, h_1)))
        st, rows = eps[-1].status()
        out.append(dict(same=same, status=st))
    torch.save(out, Path(out_dir) / f"st{rank}.pt")
    dist.barrier()
    for ep in reversed(eps):
        ep.close()
    ep_stack.close()
    ref_stack.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_ep_stack_two_ranks_one_gpu_bit_identical(tmp_path):
    """Three chained layers, each with its own resident set and load-aware
    split, all on one shared symmetric region: every layer's output on every
    rank equals the single-GPU stack's, over forwards of different sizes."""
    mp.spawn(_gpu_stack_worker, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        for i, d in enumerate(torch.load(tmp_path / f"st{r}.pt", weights_only=False)):
            assert d["status"] == 0, f"rank {r} forward {i}: status {d['status']}"
            assert all(d["same"]), f"rank {r} forward {i}: per-layer EP == EP=1: {d['same']}"


# ---------------------------------------------------------------------------
# NCCL transport without host synchronisation (emoe_epx_*, capacity chunks)
# ---------------------------------------------------------------------------
def _gpu_epx_worker(rank, world, port_no, resident, out_dir, loads, cap):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import NcclExpertParallelMoE

    cum = plan_shares(resident, 8, world, loads)
    mine = owned_experts(cum, rank)
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(mine), mine, max_tokens=2048)
    ep = NcclExpertParallelMoE(layer, resident, loads=loads, cap_rows=cap)
    full, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(resident), resident,
                             max_tokens=2048)
    res = []
    for it, T in enumerate([1500 + 100 * rank, 700 - 50 * rank, 2048]):
        x = torch.randn(T, 256, generator=torch.Generator().manual_seed(10 * it + rank)).to(torch.bfloat16).cuda()
        y_ep = ep(x)
        st, rows = ep.status()
        y_1 = full.forward(x)
        torch.cuda.synchronize()
        res.append(dict(same=bool(torch.equal(y_ep, y_1)), status=st, rows=rows))
    torch.save(res, Path(out_dir) / f"x{rank}.pt")
    dist.barrier()
    ep.close()
    layer.close()
    full.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("resident,loads,cap", [([0, 2, 5, 7], None, 0), ([0, 2, 5, 7], SKEW, 0), ([3], None, 0),
                                               ([1, 6], [0, 1, 0, 0, 0, 0, 3, 0], 4352), ([0, 2, 5, 7], None, 128)])
def test_epx_two_ranks_one_gpu(resident, loads, cap, tmp_path):
    """The NCCL chunk transport (here over gloo, 2 ranks sharing one B200):
    bit-identical to the single-GPU forward over three forwards; a capacity
    too small for a pair (cap = 128 rows) drops the forward on both ranks with
    status 2 instead of returning a wrong output silently."""
    mp.spawn(_gpu_epx_worker, args=(2, free_port(), resident, str(tmp_path), loads, cap), nprocs=2, join=True)
    for r in range(2):
        for i, d in enumerate(torch.load(tmp_path / f"x{r}.pt", weights_only=False)):
            if cap == 128:
                assert d["status"] == 2, f"rank {r} forward {i}: overflow not reported"
            else:
                assert d["status"] == 0 and d["rows"] > 0, f"rank {r} forward {i}: status {d['status']}"
                assert d["same"], f"rank {r} forward {i}: NCCL chunk EP output differs from 1 GPU"


def _nccl_graph_worker(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    from helpers import build_layer
    from paper_2503_06823_b200.ep import NcclExpertParallelMoE

    resident = [0, 2, 5, 7]
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", 4, resident, max_tokens=2048)
    ep = NcclExpertParallelMoE(layer, resident)
    x = torch.randn(1800, 256, generator=torch.Generator().manual_seed(4)).to(torch.bfloat16).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ep(x, out=y)  # warm-up (lazy NCCL communicator setup happens outside the capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):  # any host synchronisation inside would abort the capture
        ep(x, out=y)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    ref = layer.forward(x)
    torch.cuda.synchronize()
    torch.save(dict(same=bool(torch.equal(y, ref))), Path(out_dir) / "g.pt")
    ep.close()
    layer.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_epx_nccl_forward_has_no_host_sync(tmp_path):
    """The whole NCCL-transport forward -- route, device count all-gather,
    device layout + dispatch permute, equal-split all_to_all, FFN, return
    all_to_all, combine -- is captured into one CUDA graph on an NCCL group
    (world 1 on this single-GPU box): a host synchronisation anywhere would
    abort the capture.  The replay equals the plain forward."""
    mp.spawn(_nccl_graph_worker, args=(1, free_port(), str(tmp_path)), nprocs=1, join=True)
    assert torch.load(tmp_path / "g.pt", weights_only=False)["same"]
