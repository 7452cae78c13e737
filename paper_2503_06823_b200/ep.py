"""Expert parallelism for the predicted-residency MoE layer.

Tokens are data-parallel: every rank routes its own tokens against the GLOBAL
resident set (the reference Placement, replicated), while the resident experts'
weights are spread over the ranks by plan_shares: each expert runs on a run of
consecutive ranks with a fixed share of its rows (token-level split), so a hot
expert occupies several GPUs and light ones share one (e.g. 4 resident
Mixtral experts on 8 GPUs: two ranks per expert, half its rows each).

One step on every rank:
  1. route + permute locally (K1 + K3): padded per-expert segments of x
  2. segment-size all-to-all (tiny) so every rank knows what it receives
  3. dispatch all-to-all(v) of the padded segments, chunks ordered by
     (source rank, expert, token)
  4. grouped FFN (K4) on the received segments, one segment per (source, expert)
     piece
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


SHARE_ONE = 1 << 24  # fixed-point unit of the cumulative shares (emoe_ep_create)


def plan_shares(resident: Sequence[int], num_experts: int, world: int, loads=None,
                min_share: float = 0.05) -> np.ndarray:
    """cum[e][q] (int64 [E][W], fixed point SHARE_ONE = 1): the cumulative
    share of resident expert e's rows computed on ranks <= q; -1 rows for
    experts that are not resident.

    The busiest rank is what an FFN-bound EP step waits for, so the resident
    experts' expected loads (loads[e], e.g. the predictor's Eq. 2 aggregate,
    identical on every rank; None = equal) are laid end to end on [0, W) in
    expert order and cut into W unit intervals, one per rank: expert e runs on
    the ranks its interval [c_e, c_e + w_e) covers, each with the covered
    fraction.  Every forward then splits e's rows (all sources, in source
    order) at those fractions rounded to the segment padding (ep.cu bar0,
    restated in p2p_layout), so a hot expert is shared token by token and a
    light one shares a rank with its neighbours.  A rank's share of an expert
    below `min_share` of a rank's capacity moves to the expert's neighbouring
    rank (one expert copy fewer for at most that much imbalance).  Ranks of
    consecutive experts are non-decreasing, so each source's permuted buffer
    is already grouped by destination (the NCCL transport sends contiguous
    chunks)."""
    res = sorted(int(e) for e in resident)
    cum = np.full((num_experts, world), -1, np.int64)
    if not res:
        return cum
    w = np.ones(len(res)) if loads is None else np.array([max(float(loads[e]), 0.0) for e in res])
    if w.sum() <= 0:
        w = np.ones(len(res))
    w = w / w.sum() * world
    c = np.concatenate([[0.0], np.cumsum(w)])
    for i, e in enumerate(res):
        amt = np.array([max(0.0, min(q + 1.0, c[i] + w[i]) - max(float(q), c[i])) for q in range(world)])
        if amt.sum() <= 0:  # zero expected load: the rank under its (point) interval takes it
            amt[min(world - 1, int(np.floor(c[i])))] = 1.0
        nz = np.flatnonzero(amt > 0)
        while len(nz) > 1 and amt[nz[0]] < min_share:  # tiny head share -> next rank
            amt[nz[1]] += amt[nz[0]]
            amt[nz[0]] = 0.0
            nz = nz[1:]
        while len(nz) > 1 and amt[nz[-1]] < min_share:  # tiny tail share -> previous rank
            amt[nz[-2]] += amt[nz[-1]]
            amt[nz[-1]] = 0.0
            nz = nz[:-1]
        frac = np.cumsum(amt) / amt.sum()
        row = np.minimum(np.round(frac * SHARE_ONE).astype(np.int64), SHARE_ONE)
        row[nz[-1]:] = SHARE_ONE
        cum[e] = np.maximum.accumulate(row)
    return cum


def owned_experts(cum: np.ndarray, rank: int) -> list:
    """Experts with a non-zero share on `rank` (the weights it must hold)."""
    out = []
    for e in range(cum.shape[0]):
        if cum[e, 0] < 0:
            continue
        prev = cum[e, rank - 1] if rank > 0 else 0
        if cum[e, rank] > prev:
            out.append(e)
    return out


def split_bounds(counts: np.ndarray, cum: np.ndarray, pad: int):
    """The per-forward split every rank derives from the replicated count table
    (ep.cu ep_bar0_kernel): counts[s][e] real rows of source s.
    Returns (cp, pre, bnd): padded counts [W][E], rows of e held by earlier
    sources [W][E], and split ends B_e(q) [E][W] (rank q computes e's rows
    [B_e(q-1), B_e(q)) of the source-ordered sequence)."""
    W, E = counts.shape
    cp = (counts.astype(np.int64) + pad - 1) // pad * pad
    pre = np.zeros((W, E), np.int64)
    pre[1:] = np.cumsum(cp, axis=0)[:-1]
    n = cp.sum(axis=0)
    bnd = np.zeros((E, W), np.int64)
    for e in range(E):
        for q in range(W):
            cq = int(cum[e, q])
            if q == W - 1 or cq < 0:
                b = int(n[e])
            else:
                b = pad * ((int(n[e]) // pad * cq + (SHARE_ONE >> 1)) >> 24)
            bnd[e, q] = min(b, int(n[e]))
    return cp, pre, bnd


def p2p_layout(counts: np.ndarray, cum: np.ndarray, rank: int, pad: int) -> dict:
    """Everything ep_bar0_kernel computes on rank `rank` (csrc/ep.cu), restated.
    counts[s][e] = real rows source s routes to expert e.
      piece_end[e][q], piece_shift[e][q]: this rank's local rows
          [piece_end[e][q-1], piece_end[e][q]) of segment e go to rank q at
          receive row (local row + piece_shift[e][q]);
      recv_segs [W*n_owned+1], seg_expert, seg_src, out_shift: the receive
          segments (source, owned expert) in order, receive row r of segment i
          returning to row r + out_shift[i] of source seg_src[i]'s layout;
      tot[s][q]: rows source s sends rank q; seg_offsets: this rank's padded
          local segment starts [E+1]."""
    W, E = counts.shape
    cp, pre, bnd = split_bounds(counts, cum, pad)
    loc = np.zeros((W, E + 1), np.int64)
    loc[:, 1:] = np.cumsum(cp, axis=1)

    def piece(s, e, q):
        p0, p1 = pre[s, e], pre[s, e] + cp[s, e]
        lo = max(p0, bnd[e, q - 1] if q > 0 else 0)
        hi = min(p1, bnd[e, q])
        return lo, max(hi, lo)

    tot = np.zeros((W, W), np.int64)
    for s in range(W):
        for q in range(W):
            tot[s, q] = sum(piece(s, e, q)[1] - piece(s, e, q)[0] for e in range(E))
    piece_end = np.zeros((E, W), np.int64)
    piece_shift = np.zeros((E, W), np.int64)
    for q in range(W):
        recv_off = int(tot[:rank, q].sum())
        for e in range(E):
            lo, hi = piece(rank, e, q)
            p0, seg = pre[rank, e], loc[rank, e]
            end_g = min(max(bnd[e, q], p0), p0 + cp[rank, e])
            piece_end[e, q] = seg + (end_g - p0)
            piece_shift[e, q] = recv_off - seg - (lo - p0)
            recv_off += hi - lo
    owned = owned_experts(cum, rank)
    segs, exp, src, out, off = [], [], [], [], 0
    for s in range(W):
        for e in owned:
            lo, hi = piece(s, e, rank)
            segs.append(off)
            exp.append(e)
            src.append(s)
            out.append(int(loc[s, e] + (lo - pre[s, e]) - off))
            off += hi - lo
    segs.append(off)
    return dict(piece_end=piece_end, piece_shift=piece_shift, recv_segs=np.asarray(segs, np.int64),
                seg_expert=np.asarray(exp, np.int32), seg_src=np.asarray(src, np.int32),
                out_shift=np.asarray(out, np.int64), tot=tot, seg_offsets=loc[rank])


@dataclass
class RoutedBatch:
    seg_offsets: np.ndarray  # [E+1] host, padded segment starts
    rows: torch.Tensor       # [seg_offsets[E], d] permuted activations
    pos: torch.Tensor        # [T, k]
    served_w: torch.Tensor   # [T, k]
    T: int
    counts: Optional[np.ndarray] = None  # [E] real rows per expert


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
        self.layer.workspace()
        self.pad = self.layer.seg_pad

    def route_permute(self, x: torch.Tensor) -> RoutedBatch:
        self.layer.route_permute(x)
        ws = self.layer.workspace()
        seg = ws["seg_offsets"].cpu().numpy()  # host needs the split sizes (syncs the stream)
        return RoutedBatch(seg, ws["x_perm"][: int(seg[-1])], ws["pos"], ws["served_w"], x.shape[0],
                           ws["counts"].cpu().numpy().astype(np.int64))

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
    """EP forward over a process group with all-to-all collectives (the NCCL
    transport); `backend` provides the local kernels.  Same split and receive
    layout as the peer-memory path (p2p_layout), so the output is
    bit-identical to it and to EP=1."""

    def __init__(self, backend, global_resident: Sequence[int], group=None, loads=None):
        self.backend = backend
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cum = plan_shares(global_resident, backend.E, self.world, loads)
        self.stage_on_host = dist.get_backend(group) != "nccl"
        self.last = {}

    def owned(self) -> list:
        return owned_experts(self.cum, self.rank)

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
        counts = torch.from_numpy(np.ascontiguousarray(batch.counts, np.int64))
        table = [torch.empty(E, dtype=torch.int64) for _ in range(W)]
        if self.stage_on_host:
            dist.all_gather(table, counts, group=self.group)
        else:  # NCCL exchanges device tensors
            dev = torch.device("cuda", torch.cuda.current_device())
            t_dev = [torch.empty(E, dtype=torch.int64, device=dev) for _ in range(W)]
            dist.all_gather(t_dev, counts.to(dev), group=self.group)
            table = [t.cpu() for t in t_dev]
        cnt = torch.stack(table).numpy()
        lay = p2p_layout(cnt, self.cum, r, b.pad)
        send_rows = lay["tot"][r].tolist()
        recv_rows = lay["tot"][:, r].tolist()
        R = int(sum(recv_rows))
        recv = torch.empty(R, b.d, dtype=batch.rows.dtype, device=batch.rows.device)
        self._a2a(recv, batch.rows, recv_rows, send_rows)
        y_recv = b.ffn(recv, lay["recv_segs"], lay["seg_expert"])
        y_back = torch.empty_like(batch.rows)
        self._a2a(y_back, y_recv, send_rows, recv_rows)
        self.last = dict(send_rows=send_rows, recv_rows=recv_rows, segments=len(lay["seg_expert"]))
        return b.combine(y_back, batch)

    __call__ = forward


class NcclExpertParallelMoE:
    """Expert parallelism over NCCL all-to-all with no host synchronisation
    (the capacity-padded form of SURVEY.md §8e) through emoe_epx_*: the count
    exchange is one all_gather_into_tensor of [E] int32 on the device, the
    split layout is computed on the device from it (the same split as the
    peer-memory path), and every (source, destination) pair owns a fixed chunk
    of `cap` rows, so both all_to_all_single calls take equal splits.  The
    price is wire bytes: every chunk travels whole (cap rows), so cap should
    be a bound on the rows one source sends one destination
    (plan_pair_rows); a pair over cap drops the forward's rows on every rank
    and status() reports 2.  Bit-identical to the peer-memory path and EP=1."""

    def __init__(self, layer, global_resident: Sequence[int], group=None, loads=None, cap_rows: int = 0,
                 min_share: float = 0.05):
        import ctypes as C

        from ._lib import lib
        from .moesim import check

        self._lib, self._check, self._C = lib, check, C
        self.layer = layer
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.E = layer.E
        self.cum = plan_shares(global_resident, layer.E, self.world, loads, min_share)
        res = np.zeros(layer.E, np.uint8)
        res[list(global_resident)] = 1
        layer.set_route_residency(res)
        cum = np.ascontiguousarray(self.cum, np.int64)
        h = C.c_void_p()
        check(lib.emoe_epx_create(layer.h, self.world, self.rank, cum.ctypes.data_as(C.c_void_p), int(cap_rows),
                                  C.byref(h)))
        self.h = h
        cap = C.c_int64()
        check(lib.emoe_epx_cap_rows(h, C.byref(cap)))
        self.cap = int(cap.value)
        dev = torch.device("cuda", torch.cuda.current_device())
        rows = self.world * self.cap
        self.send = torch.empty(rows, layer.d, dtype=torch.bfloat16, device=dev)
        self.recv = torch.empty_like(self.send)
        self.ret = torch.empty_like(self.send)
        self.back = torch.empty_like(self.send)
        self.table = torch.empty(self.world * layer.E, dtype=torch.int32, device=dev)
        self.stage_on_host = dist.get_backend(group) != "nccl"
        self._prof = False
        self._ev_sets = []  # one list of len(NCCL_STAGES) + 1 events per profiled forward

    def set_profiling(self, enable: bool = True) -> None:
        """Record CUDA events between the forward's stages (on the compute
        stream, which waits on each collective, so a stage's time includes its
        all-to-all); read them with stage_times()."""
        self._prof = bool(enable)
        self._ev_sets = []

    def _mark(self, evs, s):
        if evs is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            evs.append(e)

    def stage_times(self) -> dict:
        """ms per stage (NCCL_STAGES), averaged over the profiled forwards;
        synchronises the device."""
        torch.cuda.synchronize()
        tot = dict.fromkeys(NCCL_STAGES, 0.0)
        for evs in self._ev_sets:
            for i, name in enumerate(NCCL_STAGES):
                tot[name] += evs[i].elapsed_time(evs[i + 1])
        n = max(1, len(self._ev_sets))
        return {k: v / n for k, v in tot.items()}

    def owned(self) -> list:
        return owned_experts(self.cum, self.rank)

    def _a2a(self, out, inp):
        if self.stage_on_host:  # gloo (tests, ranks sharing one GPU): staged through the host
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, group=self.group)

    def forward(self, x: torch.Tensor, logits: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
        C = self._C
        assert x.is_cuda and x.dtype == torch.bfloat16 and x.shape[1] == self.layer.d and x.is_contiguous()
        y = torch.empty_like(x) if out is None else out
        s = stream if stream is not None else torch.cuda.current_stream()
        sp = C.c_void_p(s.cuda_stream)
        lp = None if logits is None else C.c_void_p(logits.contiguous().data_ptr())
        T = x.shape[0]
        evs = [] if self._prof else None
        self._mark(evs, s)
        self._check(self._lib.emoe_epx_route(self.h, C.c_void_p(x.data_ptr()), lp, T, sp))
        self._mark(evs, s)
        counts = self.layer.workspace()["counts"]
        if self.stage_on_host:
            parts = [torch.empty(self.E, dtype=torch.int32) for _ in range(self.world)]
            dist.all_gather(parts, counts.cpu(), group=self.group)
            self.table.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(self.table, counts, group=self.group)
        self._mark(evs, s)
        self._check(self._lib.emoe_epx_dispatch(self.h, C.c_void_p(self.table.data_ptr()), C.c_void_p(x.data_ptr()),
                                                T, C.c_void_p(self.send.data_ptr()), sp))
        self._mark(evs, s)
        self._a2a(self.recv, self.send)
        self._mark(evs, s)
        self._check(self._lib.emoe_epx_ffn(self.h, C.c_void_p(self.recv.data_ptr()), C.c_void_p(self.ret.data_ptr()),
                                           sp))
        self._mark(evs, s)
        self._a2a(self.back, self.ret)
        self._mark(evs, s)
        self._check(self._lib.emoe_epx_combine(self.h, C.c_void_p(self.back.data_ptr()), C.c_void_p(y.data_ptr()), T,
                                               sp))
        self._mark(evs, s)
        if evs is not None:
            self._ev_sets.append(evs)
        return y

    __call__ = forward

    def status(self, stream=None):
        """(status, rows computed last forward); synchronises the stream.
        status 2 = a (source, destination) pair exceeded cap rows."""
        C = self._C
        s = stream if stream is not None else torch.cuda.current_stream()
        st, rr = C.c_int(), C.c_int64()
        self._check(self._lib.emoe_epx_status(self.h, C.c_void_p(s.cuda_stream), C.byref(st), C.byref(rr)))
        return st.value, rr.value

    def close(self):
        if getattr(self, "h", None):
            self._lib.emoe_epx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def plan_pair_rows(cum: np.ndarray, loads, tokens: int, top_k: int, pad: int, slack: float = 1.25) -> int:
    """A capacity for NcclExpertParallelMoE: the rows the busiest (source,
    destination) pair is expected to carry when every source routes `tokens`
    tokens (<= top_k rows each) with the experts' load shares `loads`
    (e.g. the Eq. 2 aggregate), times `slack`, plus one pad per expert."""
    W = cum.shape[1]
    res = [e for e in range(cum.shape[0]) if cum[e, 0] >= 0]
    w = np.array([max(float(loads[e]), 0.0) for e in res]) if loads is not None else np.ones(len(res))
    w = w / w.sum() if w.sum() > 0 else np.ones(len(res)) / len(res)
    rows = tokens * top_k
    per_q = np.zeros(W)
    for i, e in enumerate(res):
        frac = np.diff(np.concatenate([[0], cum[e]])) / SHARE_ONE
        per_q += frac * w[i] * rows
    return int(np.ceil(per_q.max() * slack)) + len(res) * pad


STAGES = ["route", "count_exchange", "dispatch", "dispatch_wait", "gemm1", "gemm2_return", "return_wait", "combine"]
# NcclExpertParallelMoE: route + permute, count all-gather, dispatch packing,
# dispatch all-to-all, both GEMMs, return all-to-all, combine
NCCL_STAGES = ["route", "count_exchange", "dispatch", "dispatch_a2a", "ffn", "return_a2a", "combine"]


class PeerExpertParallelMoE:
    """Expert parallelism over peer memory through the C ABI (emoe_ep_*).

    `layer` is this rank's MoELayer holding the experts it computes
    (owned_experts of plan_shares(...)); the group only carries the
    IPC-handle exchange at construction (gloo or NCCL) -- the forward itself
    uses no collective.  `loads` (identical on every rank) weights the
    placement.  `share_with`: another PeerExpertParallelMoE of this rank
    (a stack's first layer) whose symmetric region this one reuses."""

    def __init__(self, layer, global_resident: Sequence[int], group=None, recv_rows_cap: int = 0, loads=None,
                 share_with: Optional["PeerExpertParallelMoE"] = None, min_share: float = 0.05):
        import ctypes as C

        from ._lib import IPC_HANDLE_BYTES, lib
        from .moesim import check

        self._lib, self._check, self._C = lib, check, C
        self.layer = layer
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.E = layer.E
        self.cum = plan_shares(global_resident, layer.E, self.world, loads, min_share)
        res = np.zeros(layer.E, np.uint8)
        res[list(global_resident)] = 1
        layer.set_route_residency(res)
        cum = np.ascontiguousarray(self.cum, np.int64)
        h = C.c_void_p()
        check(lib.emoe_ep_create(layer.h, self.world, self.rank, cum.ctypes.data_as(C.c_void_p), int(recv_rows_cap),
                                 share_with.h if share_with is not None else None, C.byref(h)))
        self.h = h
        self._share = share_with  # keeps the region owner alive
        if share_with is None:
            buf = (C.c_uint8 * IPC_HANDLE_BYTES)()
            check(lib.emoe_ep_ipc_handle(h, buf))
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(buf), group=group)
            allh = np.frombuffer(b"".join(handles), np.uint8).copy()
            check(lib.emoe_ep_open_peers(h, allh.ctypes.data_as(C.c_void_p)))
            dist.barrier(group=group)  # every rank mapped every peer before the first forward

    def owned(self) -> list:
        return owned_experts(self.cum, self.rank)

    def forward(self, x: torch.Tensor, logits: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
        C = self._C
        assert x.is_cuda and x.dtype == torch.bfloat16 and x.shape[1] == self.layer.d and x.is_contiguous()
        y = torch.empty_like(x) if out is None else out
        lp = None
        if logits is not None:
            assert logits.is_cuda and logits.dtype == torch.float32 and logits.shape == (x.shape[0], self.E)
            lp = C.c_void_p(logits.contiguous().data_ptr())
        s = stream if stream is not None else torch.cuda.current_stream()
        self._check(self._lib.emoe_ep_forward(self.h, C.c_void_p(x.data_ptr()), lp, C.c_void_p(y.data_ptr()),
                                              x.shape[0], C.c_void_p(s.cuda_stream)))
        return y

    __call__ = forward

    def status(self, stream=None):
        """(status, rows computed last forward); synchronises the stream.
        status 1 = a peer barrier timed out, 2 = a receive buffer overflowed."""
        C = self._C
        s = stream if stream is not None else torch.cuda.current_stream()
        st, rr = C.c_int(), C.c_int64()
        self._check(self._lib.emoe_ep_status(self.h, C.c_void_p(s.cuda_stream), C.byref(st), C.byref(rr)))
        return st.value, rr.value

    def stats(self, stream=None) -> dict:
        """Exchange volume of the last forward (synchronises the stream)."""
        C = self._C
        s = stream if stream is not None else torch.cuda.current_stream()
        out = np.zeros(5, np.int64)
        self._check(self._lib.emoe_ep_stats(self.h, C.c_void_p(s.cuda_stream), out.ctypes.data_as(C.c_void_p)))
        row = self.layer.d * 2
        return dict(rows_computed=int(out[0]), rows_sent_to_peers=int(out[1]), rows_recv_from_peers=int(out[2]),
                    rows_routed=int(out[3]), rows_computed_real=int(out[4]), dispatch_bytes_to_peers=int(out[1]) * row,
                    return_bytes_to_peers=int(out[2]) * row)

    def layout(self, stream=None) -> dict:
        """The last forward's send pieces and receive layout (tests)."""
        C = self._C
        s = stream if stream is not None else torch.cuda.current_stream()
        W, E, n = self.world, self.E, len(self.owned())
        pe, ps = np.zeros((E, W), np.int64), np.zeros((E, W), np.int64)
        rs, osh = np.zeros(W * n + 1, np.int64), np.zeros(max(1, W * n), np.int64)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self._lib.emoe_ep_layout(self.h, C.c_void_p(s.cuda_stream), p(pe), p(ps), p(rs), p(osh)))
        return dict(piece_end=pe, piece_shift=ps, recv_segs=rs, out_shift=osh[: W * n])

    def set_profiling(self, enable: bool = True) -> None:
        self._check(self._lib.emoe_ep_set_profiling(self.h, int(enable)))

    def stage_times(self) -> dict:
        ms = (self._C.c_float * 8)()
        self._check(self._lib.emoe_ep_stage_times(self.h, ms))
        return dict(zip(STAGES, [float(v) for v in ms]))

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

