"""A6 under data parallelism: per-rank histogram tallies
merged with one all-reduce must equal a single fit over all prompts.

CPU (gloo, world 2-4): ep.HistogramSync over a host stand-in whose tallies
come from the reference's own fit (oracle/_ref, predictor.cpp:137-185) on
each rank's shard; the merged tallies are compared bit-exactly with the
reference fit over the whole trace.  GPU: ep.fit_sharded on real
emoe_predictor handles, 2 ranks sharing one B200.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2503_06823_b200.ep import HistogramSync, shard_range  # noqa: E402

E, M, T, K, P = 8, 3, 16, 2, 13
NAMES = ("cls", "conv")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def make_trace(seed=3):
    rng = np.random.default_rng(seed)
    trace = np.zeros((P, M, T, K), np.int32)
    for p in range(P):
        for l in range(M):
            for t in range(T):
                trace[p, l, t] = rng.choice(E, K, replace=False)
    return trace, rng.integers(0, len(NAMES), P).astype(np.int32)


def flat(model, tasks_seen):
    """[layer | prompt | task] with one task row per name in NAMES (the
    reference model holds rows only for the tasks it saw, in std::map order)."""
    tc = np.zeros((len(NAMES), M, E))
    seen = sorted({NAMES[i] for i in tasks_seen})
    for row, name in zip(model["task_counts"], seen):
        tc[NAMES.index(name)] = row
    return torch.from_numpy(np.concatenate([model["layer_counts"].ravel(), model["prompt_counts"].ravel(),
                                            tc.ravel()]).astype(np.int64))


class HostCounts:
    """Stand-in for PredictorCounts: the caller sets the tallies."""

    def __init__(self, n):
        self.t = torch.zeros(n, dtype=torch.int64)

    def export(self):
        return self.t.clone()

    def import_(self, t):
        self.t = t.clone()


def _worker(rank, world, port_no, prime, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Ref

    ref = Ref()
    trace, tasks = make_trace()

    def fit(lo, hi):
        return flat(ref.fit(trace[lo:hi], tasks[lo:hi], NAMES, num_experts=E), tasks[lo:hi])

    io = HostCounts(fit(0, 1).numel())
    sync = HistogramSync(io)
    a, b = shard_range(P, world, rank)
    if b > a:
        lo = a
        if prime and a > 0:  # replay the previous shard's last prompt for the chain only
            lo = a - 1
            io.import_(fit(lo, a))
            sync.mark_local()
        io.import_(fit(lo, b))
    merged = sync.merge()
    assert torch.equal(io.export(), merged)
    torch.save(merged, Path(out_dir) / f"m{rank}.pt")
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_histogram_sync_equals_single_fit(world, tmp_path):
    from oracle.oracle import Ref, have_ref

    if not have_ref():
        pytest.skip("oracle/_ref not built")
    mp.spawn(_worker, args=(world, free_port(), True, str(tmp_path)), nprocs=world, join=True)
    trace, tasks = make_trace()
    want = flat(Ref().fit(trace, tasks, NAMES, num_experts=E), tasks)
    for r in range(world):
        assert torch.equal(torch.load(tmp_path / f"m{r}.pt"), want), f"rank {r}: merged tallies differ from one fit"


def test_histogram_sync_without_priming_drops_boundary_transitions(tmp_path):
    """Control: without replaying the previous shard's last prompt the merged
    tallies miss the W-1 prompt transitions across shard boundaries."""
    from oracle.oracle import Ref, have_ref

    if not have_ref():
        pytest.skip("oracle/_ref not built")
    world = 3
    mp.spawn(_worker, args=(world, free_port(), False, str(tmp_path)), nprocs=world, join=True)
    trace, tasks = make_trace()
    model = Ref().fit(trace, tasks, NAMES, num_experts=E)
    got = torch.load(tmp_path / "m0.pt")
    want = flat(model, tasks)
    nl = model["layer_counts"].size
    npc = model["prompt_counts"].size
    assert torch.equal(got[:nl], want[:nl]) and torch.equal(got[nl + npc:], want[nl + npc:])
    assert int(want[nl:nl + npc].sum() - got[nl:nl + npc].sum()) == (world - 1) * M


def _gpu_worker(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_06823_b200 import moesim
    from paper_2503_06823_b200.ep import PredictorCounts, fit_sharded

    trace, tasks = make_trace()
    pred = moesim._Pred(M, E, K, len(NAMES), 0.01)
    fit_sharded(pred.h, torch.from_numpy(trace).cuda(), torch.from_numpy(tasks).cuda())
    torch.save(PredictorCounts(pred.h).export().cpu(), Path(out_dir) / f"g{rank}.pt")
    dist.barrier()
    del pred
    dist.destroy_process_group()


@pytest.mark.gpu
def test_fit_sharded_two_ranks_one_gpu(tmp_path):
    from oracle.oracle import Ref, have_ref

    mp.spawn(_gpu_worker, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    trace, tasks = make_trace()
    from paper_2503_06823_b200 import moesim
    from paper_2503_06823_b200.ep import PredictorCounts

    single = moesim._Pred(M, E, K, len(NAMES), 0.01)
    import ctypes as C

    from paper_2503_06823_b200._lib import lib

    d = torch.from_numpy(trace).cuda()
    tid = torch.from_numpy(tasks).cuda()
    moesim.check(lib.emoe_hist_update(single.h, C.c_void_p(d.data_ptr()), P, T, C.c_void_p(tid.data_ptr()), None))
    want = PredictorCounts(single.h).export().cpu()
    if have_ref():
        assert torch.equal(want, flat(Ref().fit(trace, tasks, NAMES, num_experts=E), tasks))
    for r in range(2):
        assert torch.equal(torch.load(tmp_path / f"g{r}.pt"), want), f"rank {r}: sharded fit differs"
