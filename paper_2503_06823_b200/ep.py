"""Expert parallelism for the predicted-residency MoE layer.

Tokens are data-parallel: every rank routes its own tokens against the GLOBAL
resident set (the reference Placement, replicated), while the resident experts'
weights are sharded across ranks.  When there are fewer resident experts than
ranks (e.g. 4 resident Mixtral experts on 8 GPUs) groups of L ranks each hold a
full replica of the resident set and source ranks are spread over the groups.

One step on every rank:
  1. route + permute locally (K1 + K3): padded per-expert segments of x
  2. segment-size all-to-all (tiny) so every rank knows what it receives
  3. dispatch all-to-all(v) of the padded segments, chunks ordered by
     (source rank, expert, token)
  4. grouped FFN (K4) on the received segments, one segment per (source, expert)
  5. return all-to-all(v) of the expert outputs into the source's layout
  6. combine at the source in slot order (K5)
Each row's FFN is the same kernel with the same weights wherever it runs, and
the combine order is fixed at the source, so the EP=G output is bit-identical
to EP=1 (tests/test_ep.py checks it with gloo on CPU and on the GPU).

The exchange is NCCL all_to_all_single over NVLink for device tensors; with a
gloo group (CPU tests, or several ranks sharing one GPU) tensors are staged
through host memory.

PeerExpertParallelMoE is the fused form (csrc/ep.cu): the permute kernel
stores each row straight into its owner's receive buffer and GEMM2's epilogue
stores each expert output row straight back into its source's permuted
layout, over CUDA-IPC-mapped peer memory (NVLink between GPUs), with
device-side barriers and no host synchronisation; the combine is local.  The receive layout is the same (source rank, expert,
token) order, so its output is bit-identical too.  `p2p_layout` restates the
layout the device computes (tests check it on CPU).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def plan_destinations(resident: Sequence[int], num_experts: int, world: int, loads=None) -> np.ndarray:
    """dest[src, e] = rank that computes source `src`'s rows of resident expert e
    (-1 for non-resident experts).  Monotone in e for every source, so each
    source's permuted buffer is already grouped by destination (the NCCL
    transport sends contiguous chunks).

    loads None: resident experts in contiguous equal-count blocks (L >= W), or
    W // L full replicas of the resident set with sources spread over them
    (L < W).  loads[e] (e.g. the ranks' summed Eq. 2 expected tokens): the
    busiest rank is what an FFN-bound EP step waits for, so the resident
    experts' loads are laid end to end on [0, W) in expert order and cut into
    W unit intervals (one per rank); source s sends its rows of e to the rank
    under the point c_e + (s + 1/2) w_e / W of e's interval [c_e, c_e + w_e).
    A heavy expert is thereby replicated over the ranks its interval covers
    and light neighbours share a rank; the points are non-decreasing in e, so
    the plan stays monotone (tools/ep_balance_model.py on the config-2
    routing: 0.49 -> 0.79 of W GPUs' FFN throughput at W = 8)."""
    res = sorted(int(e) for e in resident)
    L = len(res)
    dest = np.full((world, num_experts), -1, np.int64)
    if L == 0:
        return dest
    if loads is not None:
        w = np.array([max(float(loads[e]), 0.0) for e in res])
        if w.sum() > 0:
            w = w / w.sum() * world
            c = np.concatenate([[0.0], np.cumsum(w)])
            for src in range(world):
                for i, e in enumerate(res):
                    p = c[i] + (src + 0.5) * w[i] / world
                    dest[src, e] = min(world - 1, int(np.floor(p)))
            return dest
    if L >= world:
        for i, e in enumerate(res):  # contiguous blocks of resident experts per rank
            dest[:, e] = i * world // L
        return dest
    groups = world // L  # full replicas of the resident set
    for src in range(world):
        g = src % groups
        for i, e in enumerate(res):
            dest[src, e] = g * L + i
    return dest

def owned_experts(dest: np.ndarray, rank: int) -> list:
    return sorted({int(e) for e in np.flatnonzero((dest == rank).any(axis=0))})


@dataclass
class RoutedBatch:
    seg_offsets: np.ndarray  # [E+1] host, padded segment starts
    rows: torch.Tensor       # [seg_offsets[E], d] permuted activations
    pos: torch.Tensor        # [T, k]
    served_w: torch.Tensor   # [T, k]
    T: int


class LayerBackend:
    """The sm_100a kernels through the C ABI (paper_2503_06823_b200.MoELayer)."""

    def __init__(self, layer, global_resident: Sequence[int]):
        self.layer = layer
        res = np.zeros(layer.E, np.uint8)
        res[list(global_resident)] = 1
        layer.set_route_residency(res)
        self.d, self.f, self.E = layer.d, layer.f, layer.E
        self.dtype = layer.torch_dtype
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._ws = None

    def route_permute(self, x: torch.Tensor) -> RoutedBatch:
        self.layer.route_permute(x)
        ws = self.layer.workspace()
        self.pad = self.layer.seg_pad
        seg = ws["seg_offsets"].cpu().numpy()  # host needs the split sizes (syncs the stream)
        return RoutedBatch(seg, ws["x_perm"][: int(seg[-1])], ws["pos"], ws["served_w"], x.shape[0])

    def ffn(self, rows: torch.Tensor, seg_offsets: np.ndarray, seg_expert: np.ndarray) -> torch.Tensor:
        R = rows.shape[0]
        y = torch.empty(R, self.d, dtype=self.dtype, device=self.device)
        if len(seg_expert) == 0 or R == 0:
            return y
        h = torch.empty(R, self.f, dtype=self.dtype, device=self.device)
        so = torch.from_numpy(np.ascontiguousarray(seg_offsets, np.int64)).to(self.device)
        se = torch.from_numpy(np.ascontiguousarray(seg_expert, np.int32)).to(self.device)
        self.layer.ffn_segments(rows, so, se, h, y)
        return y

    def combine(self, y_rows: torch.Tensor, batch: RoutedBatch) -> torch.Tensor:
        out = torch.empty(batch.T, self.d, dtype=self.dtype, device=self.device)
        self.layer.combine(y_rows, batch.pos, batch.served_w, out)
        return out


class ExpertParallelMoE:
    """EP forward over a process group; `backend` provides the local kernels."""

    def __init__(self, backend, global_resident: Sequence[int], group=None, loads=None):
        self.backend = backend
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dest = plan_destinations(global_resident, backend.E, self.world, loads)
        self.stage_on_host = dist.get_backend(group) != "nccl"
        self.last = {}

    def owned(self) -> list:
        return owned_experts(self.dest, self.rank)

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits) -> torch.Tensor:
        if self.stage_on_host and inp.is_cuda:
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
            return out
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        b = self.backend
        E, W, r = b.E, self.world, self.rank
        batch = b.route_permute(x)
        psz = np.diff(batch.seg_offsets)  # padded rows per expert
        # rows this rank sends each destination, per expert
        send_meta = np.zeros((W, E), np.int64)
        for e in np.flatnonzero(psz):
            q = self.dest[r, e]
            if q < 0:
                raise RuntimeError(f"expert {e} has rows but is not in the global resident set")
            send_meta[q, e] = psz[e]
        meta_out = torch.empty(W * E, dtype=torch.int64)
        meta_in = torch.from_numpy(send_meta.reshape(-1)).clone()
        if self.stage_on_host:
            dist.all_to_all_single(meta_out, meta_in, group=self.group)
        else:  # NCCL exchanges device tensors
            dev = torch.device("cuda", torch.cuda.current_device())
            o = meta_out.to(dev)
            dist.all_to_all_single(o, meta_in.to(dev), group=self.group)
            meta_out.copy_(o.cpu())
        recv_meta = meta_out.numpy().reshape(W, E)
        send_rows = send_meta.sum(axis=1).tolist()
        recv_rows = recv_meta.sum(axis=1).tolist()
        R = int(sum(recv_rows))
        recv = torch.empty(R, b.d, dtype=batch.rows.dtype, device=batch.rows.device)
        self._a2a(recv, batch.rows, recv_rows, send_rows)
        # one segment per (source, expert), sources in rank order
        seg_off, seg_exp, off = [0], [], 0
        for src in range(W):
            for e in range(E):
                n = int(recv_meta[src, e])
                if n:
                    off += n
                    seg_off.append(off)
                    seg_exp.append(e)
        y_recv = b.ffn(recv, np.asarray(seg_off, np.int64), np.asarray(seg_exp, np.int32))
        y_back = torch.empty_like(batch.rows)
        self._a2a(y_back, y_recv, send_rows, recv_rows)
        self.last = dict(send_rows=send_rows, recv_rows=recv_rows, segments=len(seg_exp))
        return b.combine(y_back, batch)

    __call__ = forward


def p2p_layout(counts: np.ndarray, dest: np.ndarray, rank: int, seg_offsets: np.ndarray):
    """The receive segments and send shifts ep_bar0_kernel computes on rank
    `rank` (csrc/ep.cu).  counts[s, e] = padded rows source s holds for expert
    e; seg_offsets = this rank's local padded segment starts [E+1].
    Returns (recv_segs, seg_expert, row_shift, seg_src, out_shift): rank
    `rank` receives segment i = (seg_src[i], seg_expert[i]) at recv_segs[i]
    in (source, expert) order and pushes its outputs back to row r +
    out_shift[i] of the source's own permuted layout; it writes its own
    segment e to row seg_offsets[e] + row_shift[e] of rank dest[rank, e]'s
    receive buffer."""
    W, E = dest.shape
    owned = owned_experts(dest, rank)
    tot = np.zeros((W, W), np.int64)  # [source][receiver]
    for s in range(W):
        for e in range(E):
            if dest[s, e] >= 0:
                tot[s, dest[s, e]] += counts[s, e]
    shift = np.zeros(E, np.int64)
    for e in range(E):
        q = dest[rank, e]
        if q < 0:
            continue
        base = tot[:rank, q].sum() + sum(counts[rank, e2] for e2 in range(e) if dest[rank, e2] == q)
        shift[e] = base - seg_offsets[e]
    segs, exp, src, out, off = [], [], [], [], 0
    for s in range(W):
        for e in owned:
            segs.append(off)
            exp.append(e)
            src.append(s)
            out.append(int(counts[s, :e].sum()) - off)  # source s's padded segment e starts at its count prefix
            if dest[s, e] == rank:
                off += counts[s, e]
    segs.append(off)
    return (np.asarray(segs, np.int64), np.asarray(exp, np.int32), shift, np.asarray(src, np.int32),
            np.asarray(out, np.int64))


class PeerExpertParallelMoE:
    """Expert parallelism over peer memory through the C ABI (emoe_ep_*).

    `layer` is this rank's MoELayer holding the experts it computes; the
    group only carries the IPC-handle exchange at construction (gloo or
    NCCL) -- the forward itself uses no collective.  `loads` (identical on
    every rank) selects the load-aware placement of plan_destinations."""

    def __init__(self, layer, global_resident: Sequence[int], group=None, recv_rows_cap: int = 0, loads=None):
        import ctypes as C

        from ._lib import IPC_HANDLE_BYTES, lib
        from .moesim import check

        self._lib, self._check, self._C = lib, check, C
        self.layer = layer
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.E = layer.E
        self.dest = plan_destinations(global_resident, layer.E, self.world, loads)
        res = np.zeros(layer.E, np.uint8)
        res[list(global_resident)] = 1
        layer.set_route_residency(res)
        dest32 = np.ascontiguousarray(self.dest, np.int32)
        h = C.c_void_p()
        check(lib.emoe_ep_create(layer.h, self.world, self.rank, dest32.ctypes.data_as(C.c_void_p),
                                 int(recv_rows_cap), C.byref(h)))
        self.h = h
        buf = (C.c_uint8 * IPC_HANDLE_BYTES)()
        check(lib.emoe_ep_ipc_handle(h, buf))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(buf), group=group)
        allh = np.frombuffer(b"".join(handles), np.uint8).copy()
        check(lib.emoe_ep_open_peers(h, allh.ctypes.data_as(C.c_void_p)))
        dist.barrier(group=group)  # every rank mapped every peer before the first forward

    def owned(self) -> list:
        return owned_experts(self.dest, self.rank)

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        C = self._C
        assert x.is_cuda and x.dtype == torch.bfloat16 and x.shape[1] == self.layer.d
        x = x.contiguous()
        y = torch.empty_like(x)
        s = stream if stream is not None else torch.cuda.current_stream()
        self._check(self._lib.emoe_ep_forward(self.h, C.c_void_p(x.data_ptr()), None, C.c_void_p(y.data_ptr()),
                                              x.shape[0], C.c_void_p(s.cuda_stream)))
        return y

    __call__ = forward

    def status(self, stream=None):
        """(status, rows received last forward); synchronises the stream.
        status 1 = a peer barrier timed out, 2 = a receive buffer overflowed."""
        C = self._C
        s = stream if stream is not None else torch.cuda.current_stream()
        st, rr = C.c_int(), C.c_int64()
        self._check(self._lib.emoe_ep_status(self.h, C.c_void_p(s.cuda_stream), C.byref(st), C.byref(rr)))
        return st.value, rr.value

    def close(self):
        if getattr(self, "h", None):
            self._lib.emoe_ep_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


# ---------------------------------------------------------------------------
# predictor under multi-GPU: per-rank histograms merged by one all-reduce
# ---------------------------------------------------------------------------
def _all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM over the group; gloo groups stage CUDA tensors through the host."""
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)
    return t


class PredictorCounts:
    """Device int64 view of an emoe_predictor's tallies [layer | prompt | task]
    (emoe_predictor_counts_dev / emoe_predictor_set_counts_dev)."""

    def __init__(self, pred_handle, device=None):
        import ctypes as C

        from ._lib import lib
        from .moesim import check

        self._lib, self._check, self._C = lib, check, C
        self.h = pred_handle
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        n = C.c_int64()
        check(lib.emoe_predictor_count_size(self.h, C.byref(n)))
        self.n = int(n.value)

    def export(self) -> torch.Tensor:
        C = self._C
        t = torch.empty(self.n, dtype=torch.int64, device=self.device)
        s = torch.cuda.current_stream(self.device)
        self._check(self._lib.emoe_predictor_counts_dev(self.h, C.c_void_p(t.data_ptr()), C.c_void_p(s.cuda_stream)))
        return t

    def import_(self, t: torch.Tensor) -> None:
        C = self._C
        assert t.dtype == torch.int64 and t.is_cuda and t.numel() == self.n
        t = t.contiguous()
        s = torch.cuda.current_stream(self.device)
        self._check(self._lib.emoe_predictor_set_counts_dev(self.h, C.c_void_p(t.data_ptr()),
                                                            C.c_void_p(s.cuda_stream)))


class HistogramSync:
    """A6 under data parallelism: every rank tallies its own
    prompts, and merge() replaces every rank's tallies by the common state
    plus the SUM of all ranks' local deltas, in exact int64 (counts commute,
    test_predictor.cpp:284-296).  A7/A8 then run identically on every rank,
    so the residency tables stay replicated.

    `io` has export() -> int64 tensor and import_(tensor) (PredictorCounts for
    an emoe_predictor).  The ranks' tallies must be identical when the sync
    is created (e.g. fresh predictors).  mark_local() excludes the updates
    made since the last merge from this rank's delta -- used to prime the
    prompt chain with the previous shard's last prompt, whose own tallies
    belong to the rank that owns it (fit_sharded)."""

    def __init__(self, io, group=None):
        self.io = io
        self.group = group
        self.common = io.export().clone()
        self.mark = self.common.clone()

    def mark_local(self) -> None:
        self.mark = self.io.export().clone()

    def merge(self) -> torch.Tensor:
        delta = self.io.export() - self.mark
        _all_reduce_sum(delta, self.group)
        merged = self.common + delta
        self.io.import_(merged)
        self.common = merged.clone()
        self.mark = merged.clone()
        return merged


def shard_range(P: int, world: int, rank: int):
    """Contiguous prompt shard [a, b) of rank `rank`."""
    return P * rank // world, P * (rank + 1) // world


def fit_sharded(pred_handle, trace_dev: torch.Tensor, task_ids_dev, group=None) -> None:
    """fit over all P prompts of trace_dev [P, m, T, k] with each rank of the
    group tallying a contiguous shard, then one all-reduce: the merged
    tallies equal a single fit over the whole trace (bit-exact), because
    rank r first replays prompt a_r - 1 (only to continue the prompt chain;
    mark_local drops its tallies) and so counts the boundary transition
    a_r - 1 -> a_r itself."""
    import ctypes as C

    from ._lib import lib
    from .moesim import check

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    P, m, T, k = trace_dev.shape
    sync = HistogramSync(PredictorCounts(pred_handle, trace_dev.device), group)
    a, b = shard_range(P, world, rank)
    s = torch.cuda.current_stream(trace_dev.device)

    def update(lo, hi):
        tid = None if task_ids_dev is None else C.c_void_p(task_ids_dev[lo:hi].data_ptr())
        check(lib.emoe_hist_update(pred_handle, C.c_void_p(trace_dev[lo:hi].data_ptr()), hi - lo, T, tid,
                                   C.c_void_p(s.cuda_stream)))

    if b > a:
        if a > 0:
            update(a - 1, a)
            sync.mark_local()
        update(a, b)
    sync.merge()

