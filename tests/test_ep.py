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

from paper_2503_06823_b200.ep import ExpertParallelMoE, RoutedBatch, owned_experts, plan_destinations  # noqa: E402


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
                           torch.from_numpy(o["served_w"]), x.shape[0])

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
    loads = [1, 0, 1, 0, 0, 1, 0, 20] if skew else None  # skew: load-aware placement replicates expert 7
    mp.spawn(_cpu_worker, args=(world, free_port(), resident, str(tmp_path), loads), nprocs=world, join=True)
    for r in range(world):
        y_ep, y_1 = np.load(tmp_path / f"r{r}.npy")
        assert np.array_equal(y_ep, y_1), f"rank {r}: EP output differs from EP=1"


def test_plan_destinations():
    d = plan_destinations([0, 5, 6, 7], 8, 8)  # 4 resident on 8 ranks -> 2 replica groups
    assert d[0].tolist() == [0, -1, -1, -1, -1, 1, 2, 3]
    assert d[1].tolist() == [4, -1, -1, -1, -1, 5, 6, 7]
    assert all(owned_experts(d, q) == [[0, 5, 6, 7][q % 4]] for q in range(8))
    d = plan_destinations(list(range(8)), 8, 2)  # 8 resident on 2 ranks -> blocks of 4
    assert d[0].tolist() == [0, 0, 0, 0, 1, 1, 1, 1] and d[1].tolist() == d[0].tolist()
    for src in range(8):  # monotone in expert order -> contiguous send chunks
        row = [q for q in plan_destinations([1, 2, 4], 8, 8)[src] if q >= 0]
        assert row == sorted(row)


SKEW = np.array([1, 0, 1, 0, 0, 1, 0, 20], np.float64)  # expert 7 carries most rows


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("resident", [[0, 2, 5, 7], list(range(8)), [7], [1, 6]])
def test_plan_destinations_load_aware(world, resident):
    rng = np.random.default_rng(world * 31 + len(resident))
    for loads in (SKEW, rng.random(8) * 100, np.zeros(8)):
        d = plan_destinations(resident, 8, world, loads)
        for src in range(world):
            row = d[src]
            assert all(row[e] == -1 for e in range(8) if e not in resident)
            assert all(0 <= row[e] < world for e in resident)
            live = [row[e] for e in sorted(resident)]
            assert live == sorted(live), "load-aware plan must stay monotone in expert order"
    # the heavy expert is spread over the ranks, the light ones share a rank
    d = plan_destinations([0, 2, 5, 7], 8, 2, SKEW)
    assert d[:, 7].tolist() == [0, 1] and d[0, :7].max() == 0
    d = plan_destinations([0, 2, 5, 7], 8, 8, SKEW)
    assert len(set(d[:, 7].tolist())) >= 6
    # modelled busiest-rank load: never worse than the equal plan on the skew
    for world in (2, 4, 8):
        def busiest(dd):
            per = np.zeros(world)
            for src in range(world):
                for e in [0, 2, 5, 7]:
                    per[dd[src, e]] += SKEW[e]
            return per.max()
        assert busiest(plan_destinations([0, 2, 5, 7], 8, world, SKEW)) <= busiest(
            plan_destinations([0, 2, 5, 7], 8, world))


def _gpu_worker(rank, world, port_no, resident, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import LayerBackend

    dest = plan_destinations(resident, 8, world)
    mine = owned_experts(dest, rank)
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
        d = torch.load(tmp_path / f"g{r}.pt")
        assert torch.equal(d["y_ep"], d["y_1"]), f"rank {r}: EP output differs from the single-GPU forward"


# ---------------------------------------------------------------------------
# expert parallelism over peer memory (csrc/ep.cu)
# ---------------------------------------------------------------------------
def _simulate_p2p(backends, xs, dest):
    """CPU restatement of the peer-memory protocol: every rank publishes its
    padded counts, computes p2p_layout, 'stores' its rows into the owners'
    receive buffers, owners run the FFN over their (source, expert)
    segments, and each source combines from the owners' outputs."""
    from paper_2503_06823_b200.ep import p2p_layout

    W = len(backends)
    E = backends[0].E
    batches = [b.route_permute(x) for b, x in zip(backends, xs)]
    counts = np.stack([np.diff(bt.seg_offsets) for bt in batches])
    layouts = [p2p_layout(counts, dest, r, batches[r].seg_offsets) for r in range(W)]
    recv = [np.zeros((int(layouts[q][0][-1]), backends[0].d), np.float32) for q in range(W)]
    for r, bt in enumerate(batches):
        shift = layouts[r][2]
        for e in range(E):
            a, b = int(bt.seg_offsets[e]), int(bt.seg_offsets[e + 1])
            if b > a:
                q = dest[r, e]
                recv[q][a + shift[e]:b + shift[e]] = bt.rows[a:b].numpy()
    # every owner pushes each received segment's outputs back into the
    # source's own permuted layout (GEMM2's epilogue on the GPU)
    y_local = [np.zeros((int(bt.seg_offsets[-1]), backends[0].d), np.float32) for bt in batches]
    for q in range(W):
        segs, exp, _, src, out_shift = layouts[q]
        if not len(exp):
            continue
        out = backends[q].ffn(torch.from_numpy(recv[q]), segs, exp).numpy()
        for i in range(len(exp)):
            a, b = int(segs[i]), int(segs[i + 1])
            if b > a:
                y_local[src[i]][a + out_shift[i]:b + out_shift[i]] = out[a:b]
    ys = []
    for r, bt in enumerate(batches):
        pos = bt.pos.numpy().astype(np.int64)
        ys.append(backends[r].combine(torch.from_numpy(y_local[r]),
                                      RoutedBatch(bt.seg_offsets, None, torch.from_numpy(pos), bt.served_w, bt.T)))
    return ys, layouts


@pytest.mark.parametrize("world,resident,loads", [(2, [0, 2, 5, 7], None), (4, [1, 6], None),
                                                   (4, list(range(8)), None), (2, [3], None),
                                                   (2, [0, 2, 5, 7], SKEW), (4, [0, 2, 5, 7], SKEW),
                                                   (3, list(range(8)), SKEW)])
def test_p2p_layout_protocol_bit_identical(world, resident, loads, port):
    be = [OracleBackend(port, E=8, k=2, d=64, f=128, global_resident=resident) for _ in range(world)]
    xs = [torch.from_numpy(np.random.default_rng(200 + r).standard_normal((41 + 7 * r, 64)).astype(np.float32))
          for r in range(world)]
    dest = plan_destinations(resident, 8, world, loads)
    ys, layouts = _simulate_p2p(be, xs, dest)
    for r in range(world):
        assert np.array_equal(ys[r].numpy(), single(be[r], xs[r]).numpy()), f"rank {r}: P2P layout output differs"
    # receive segments are contiguous, padded and cover exactly the rows sent to each rank
    for q, (segs, exp, _, _, _) in enumerate(layouts):
        assert np.all(np.diff(segs) >= 0) and np.all(segs % be[0].pad == 0)
        assert len(exp) == world * len(owned_experts(dest, q))


def test_p2p_layout_disjoint_writes(port):
    """Within every receiver, the row ranges written by different (source,
    expert) segments are disjoint and tile [0, total)."""
    from paper_2503_06823_b200.ep import p2p_layout

    rng = np.random.default_rng(5)
    for world, resident, loads in [(2, [0, 2, 5, 7], None), (4, [1, 6], None), (8, [0, 5, 6, 7], None),
                                   (8, list(range(8)), None), (8, [0, 2, 5, 7], SKEW), (4, list(range(8)), SKEW)]:
        dest = plan_destinations(resident, 8, world, loads)
        counts = rng.integers(0, 5, (world, 8)) * 4 * (dest >= 0)
        seg = [np.concatenate([[0], np.cumsum(counts[r])]) for r in range(world)]
        written = {q: [] for q in range(world)}
        for r in range(world):
            _, _, shift, _, _ = p2p_layout(counts, dest, r, seg[r])
            for e in range(8):
                if counts[r, e]:
                    written[dest[r, e]].append((seg[r][e] + shift[e], seg[r][e + 1] + shift[e]))
        pushed = {r: [] for r in range(world)}
        for q in range(world):
            segs, _, _, src, out_shift = p2p_layout(counts, dest, q, seg[q])
            iv = sorted(written[q])
            assert all(a[1] == b[0] for a, b in zip(iv, iv[1:])), (world, q, iv)
            assert (iv[0][0] if iv else 0) == 0 and (iv[-1][1] if iv else 0) == segs[-1]
            for i in range(len(src)):
                if segs[i + 1] > segs[i]:
                    pushed[int(src[i])].append((segs[i] + out_shift[i], segs[i + 1] + out_shift[i]))
        # the return pushes land exactly on each source's own padded segments
        for r in range(world):
            want = sorted((seg[r][e], seg[r][e + 1]) for e in range(8) if counts[r, e])
            assert sorted(pushed[r]) == want, (world, r)


def _gpu_p2p_worker(rank, world, port_no, resident, out_dir, loads=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    os.environ.setdefault("EMOE_EP_TIMEOUT_S", "120")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE

    dest = plan_destinations(resident, 8, world, loads)
    mine = owned_experts(dest, rank)
    layer, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(mine), mine, max_tokens=2048)
    ep = PeerExpertParallelMoE(layer, resident, loads=loads)
    full, _, _ = build_layer(8, 256, 512, 2, "bf16", "swiglu", "topk_softmax", len(resident), resident,
                             max_tokens=2048)
    res = []
    for it, T in enumerate([1500 + 100 * rank, 700 - 50 * rank, 2048]):  # epochs reuse the buffers
        x = torch.randn(T, 256, generator=torch.Generator().manual_seed(10 * it + rank)).to(torch.bfloat16).cuda()
        y_ep = ep(x)
        st, rows = ep.status()
        y_1 = full.forward(x)
        torch.cuda.synchronize()
        res.append(dict(y_ep=y_ep.cpu(), y_1=y_1.cpu(), status=st, rows=rows))
    torch.save(res, Path(out_dir) / f"p{rank}.pt")
    dist.barrier()
    ep.close()
    layer.close()
    full.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("resident,loads", [([0, 2, 5, 7], None), ([3], None), ([0, 2, 5, 7], SKEW)])
def test_ep_p2p_two_ranks_one_gpu_bit_identical(resident, loads, tmp_path):
    """SKEW: expert 7 is replicated on both ranks (each computes its own
    source's rows of it) while experts 0, 2 and 5 live on rank 0."""
    mp.spawn(_gpu_p2p_worker, args=(2, free_port(), resident, str(tmp_path), loads), nprocs=2, join=True)
    for r in range(2):
        for i, d in enumerate(torch.load(tmp_path / f"p{r}.pt")):
            assert d["status"] == 0, f"rank {r} forward {i}: status {d['status']}"
            assert d["rows"] > 0
            assert torch.equal(d["y_ep"], d["y_1"]), f"rank {r} forward {i}: P2P EP output differs from 1 GPU"


def _gpu_p2p_fault_worker(rank, world, port_no, case, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no), EMOE_EP_TIMEOUT_S="2")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import build_layer
    from paper_2503_06823_b200.ep import PeerExpertParallelMoE

    resident = [0, 2, 5, 7]
    dest = plan_destinations(resident, 8, world)
    mine = owned_experts(dest, rank)
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
    r0 = torch.load(tmp_path / "f0.pt")
    if case == "overflow":
        r1 = torch.load(tmp_path / "f1.pt")
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
    d = torch.load(tmp_path / "s.pt")
    assert d["status"] == 0
    assert torch.equal(d["y_ep"], d["y_1"])
