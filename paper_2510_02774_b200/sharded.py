"""Multi-GPU GRNND build: replicated vectors, contiguous-ID-range vertex ownership, one
message exchange per round.

The reference has no distributed path (paper future work PAPER.md:3927).
Each rank owns pools [lo, hi) = [r*N/P, (r+1)*N/P).  A round is

    emit   grnnd_round_emit   pair phase (or reverse selection) of owned vertices; the
                              messages are bucketed by the owner rank of their target and
                              packed (GRNND_MSG_WORDS int32 each: key, tgt, id, dist);
    swap   one all-to-all of the counts, ONE all-to-all of the packed payload (NCCL over
           NVLink), received in source-rank order;
    apply  grnnd_round_apply  unpack, group by target, sort each segment by key,
                              three-stage insert (own entries spliced as on 1 GPU).

A message's key is source * R + emission index -- its position in the reference's global
vertex-major order -- so the receiving side restores exactly the single-GPU per-pool
order: a P-rank build is bit-identical to the 1-GPU build (and so to the reference).

The round driver (``ShardedBuild.rounds``) is a generator that yields at each exchange;
``ShardedBuild.run(exchange)`` drives it with any exchange callable.  The NCCL exchange
(``nccl_exchange``) reads the P send counts to the host once per round -- the variable
split sizes of ``all_to_all_single`` are host integers; a fixed-size padded exchange would
avoid that sync but move every rank's worst-case bucket each round, costing far more than
the ~10 us round-trip.  ``build_virtual_shards`` drives P ``ShardedBuild`` instances of
one process on one GPU in lock-step through the same generator with a concatenation
exchange: it is the single-GPU test of the exact code the NCCL path runs.
``exchange_all_to_all`` is the host logic of the NCCL exchange, also run on CPU (gloo,
world_size 2) by tests/test_sharded.py.
"""

from __future__ import annotations

import ctypes as C
from typing import Callable

import numpy as np
import torch

from . import _lib
from .builder import (
    _ORDER_CODES,
    MASK64,
    STREAM_ROUND_BASE,
    RoundStats,
    _device,
    _DevicePools,
    _finalize_device,
    _on_device,
    _stream,
    check_finite_device,
    check_metric,
    effective_params,
    normalize_rows_,
    num_rounds,
    upload,
)
from .core import BuildParams, Dataset, Graph, validate_params
from .errors import DeviceError, ParamError

MSG_WORDS = _lib.MSG_WORDS


def shard_bounds(n: int, world: int) -> list[int]:
    """Contiguous ownership ranges: rank r owns [b[r], b[r+1])."""
    return [n * r // world for r in range(world + 1)]


def pack_messages(key, tgt, mid, dist) -> torch.Tensor:
    """Host-side packing of (key, tgt, id, dist) into [m, MSG_WORDS] int32 records (the
    layout rank_scatter_kernel writes; used by the CPU tests)."""
    k = key.to(torch.int64)
    out = torch.empty((k.shape[0], MSG_WORDS), dtype=torch.int32, device=k.device)
    out[:, 0] = (k & 0xFFFFFFFF).to(torch.int64).to(torch.int32)
    out[:, 1] = (k >> 32).to(torch.int32)
    out[:, 2] = tgt.to(torch.int32)
    out[:, 3] = mid.to(torch.int32)
    out[:, 4] = dist.to(torch.float32).view(torch.int32)
    return out


def unpack_messages(p: torch.Tensor):
    """Inverse of pack_messages: (key int64, tgt int32, id int32, dist fp32)."""
    lo = p[:, 0].to(torch.int64) & 0xFFFFFFFF
    key = lo | (p[:, 1].to(torch.int64) << 32)
    return key, p[:, 2].clone(), p[:, 3].clone(), p[:, 4].clone().view(torch.float32)


class ShardPools(_DevicePools):
    """One rank's pools plus views of the workspace's packed send / receive buffers."""

    def __init__(self, data_dev, dim, cap, lo, hi, n_total, world, msg_capacity=None):
        rows = hi - lo
        # outgoing <= sum(k) of owned rows; incoming is data dependent (hubs): 2x headroom.
        # Overflow is detected on the device and raised (GRNND_ST_LOST), never truncated.
        mc = msg_capacity if msg_capacity is not None else max(2 * rows * cap, 1024)
        super().__init__(data_dev, dim, cap, lo=lo, hi=hi, n_total=n_total, msg_capacity=mc)
        self.world = world
        p = self.struct()
        po, pi = C.c_void_p(), C.c_void_p()
        _lib.call("grnnd_round_buffers", C.byref(p), C.byref(po), C.byref(pi))
        base = self.workspace.data_ptr()
        nbytes = self.msg_capacity * MSG_WORDS * 4

        def view(ptr):
            off = ptr.value - base
            return self.workspace[off: off + nbytes].view(torch.int32).view(self.msg_capacity, MSG_WORDS)

        self.out = view(po)
        self.inb = view(pi)
        self.send_counts = torch.zeros(world, dtype=torch.int64, device=self.dev)

    @_on_device
    def emit(self, kind: int, seed: int, stream_id: int, order: int, rho: float, bounds_dev: torch.Tensor,
             stats: torch.Tensor) -> None:
        p = self.struct(stats, kind != 0 or self.filtered_round(stream_id))
        _lib.call("grnnd_round_emit", C.byref(p), kind, seed & MASK64, stream_id & MASK64, order, float(rho),
                  bounds_dev.data_ptr(), self.world, self.send_counts.data_ptr(), _stream(self.dev))

    @_on_device
    def apply(self, kind: int, n_in: int, stats: torch.Tensor) -> None:
        if n_in > self.msg_capacity:
            raise DeviceError(f"rank receives {n_in} messages > capacity {self.msg_capacity}")
        p = self.struct(stats)
        _lib.call("grnnd_round_apply", C.byref(p), kind, int(n_in), _stream(self.dev))
        self.swap()


def exchange_all_to_all(out: torch.Tensor, send_counts: list[int], inb: torch.Tensor, group=None) -> int:
    """The per-round exchange over torch.distributed (NCCL on GPUs, gloo on CPU): counts
    all-to-all, then ONE all-to-all of the packed [m, MSG_WORDS] payload, received in
    source-rank order into ``inb``.  Returns the number of messages received."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if out.is_cuda and dist.get_backend(group) == "gloo":
        # gloo's all-to-all moves host tensors: stage through the host (functional multi-rank
        # runs on one GPU, where NCCL refuses two ranks per device)
        inb_h = torch.empty(inb.shape, dtype=inb.dtype)
        n_in = exchange_all_to_all(out.cpu(), send_counts, inb_h, group)
        inb[:n_in].copy_(inb_h[:n_in])
        return n_in
    dev = out.device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.cpu().tolist()]
    n_out, n_in = sum(send_counts), sum(recv_counts)
    if n_in > inb.shape[0]:
        raise DeviceError(f"rank receives {n_in} messages > capacity {inb.shape[0]}")
    dist.all_to_all_single(inb[:n_in], out[:n_out], output_split_sizes=recv_counts,
                           input_split_sizes=send_counts, group=group)
    return n_in


def nccl_exchange(group=None) -> Callable:
    """The exchange callable of a real multi-rank build."""

    def ex(sb: "ShardedBuild") -> int:
        sc = [int(x) for x in sb.pools.send_counts.cpu().tolist()]  # the one host sync per round
        return exchange_all_to_all(sb.pools.out, sc, sb.pools.inb, group)

    return ex


class ShardedBuild:
    """This rank's part of a sharded build."""

    def __init__(self, data_dev: torch.Tensor, dim: int, params: BuildParams, rank: int, world: int,
                 pair_order: str = "disordered", group=None, msg_capacity=None, metric: str = "l2"):
        n = int(data_dev.shape[0])
        self.params = effective_params(params, n)
        validate_params(self.params, n)
        if pair_order not in _ORDER_CODES:
            raise ParamError(f"pair_order must be one of {sorted(_ORDER_CODES)}")
        check_metric(metric)
        self.order = _ORDER_CODES[pair_order]
        self.rank, self.world, self.group = rank, world, group
        self.metric, self.raw, self.dim = metric, data_dev, dim
        self.bounds = shard_bounds(n, world)
        self.bounds_dev = torch.tensor(self.bounds, dtype=torch.int64, device=data_dev.device)
        work = torch.empty_like(data_dev) if metric == "ip" else data_dev
        self.pools = ShardPools(work, dim, self.params.R, self.bounds[rank], self.bounds[rank + 1], n, world,
                                msg_capacity)
        self.stats = torch.zeros((num_rounds(self.params), _lib.NSTATS), dtype=torch.int64, device=data_dev.device)
        self.kinds: list[str] = []

    def rounds(self, phase_events: list | None = None):
        """Generator over one build: yields once per round after the emit (the caller
        performs the exchange and sends back the number of messages received), returns
        (offsets, nbrs, bad, fail) of this rank's rows."""
        p, pools = self.params, self.pools
        self.stats.zero_()
        self.kinds = []
        if self.metric == "ip":
            pools.data.copy_(self.raw)
            normalize_rows_(pools.data, self.dim)
        pools.compute_norms()
        fail = pools.init(p.S, p.seed)
        i = ri = 0
        for t1 in range(1, p.T1 + 1):
            for kind in [0] * p.T2 + ([1] if t1 != p.T1 else []):
                ev = None
                if phase_events is not None and kind == 0:
                    ev = tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
                    phase_events.append(ev)
                    ev[0].record()
                pools.emit(kind, p.seed, STREAM_ROUND_BASE + ri, self.order, p.rho, self.bounds_dev, self.stats[i])
                if ev:
                    ev[1].record()
                n_in = yield kind
                pools.apply(kind, n_in, self.stats[i])
                if ev:
                    ev[2].record()
                if kind == 0:
                    ri += 1
                self.kinds.append("update" if kind == 0 else "reverse")
                i += 1
        offsets, nbrs, bad = _finalize_device(pools)
        return offsets, nbrs, bad, fail

    def run(self, phase_events: list | None = None, exchange: Callable | None = None):
        """One sharded build; same contract as builder.DeviceBuild.run (offsets, nbrs,
        bad, fail for this rank's rows).  ``exchange(self) -> n_incoming`` moves the
        round's packed messages (default: NCCL all-to-all in ``self.group``)."""
        ex = exchange or nccl_exchange(self.group)
        gen = self.rounds(phase_events)
        next(gen)
        while True:
            try:
                gen.send(ex(self))
            except StopIteration as stop:
                return stop.value

    def search_data(self) -> torch.Tensor:
        return self.pools.data

    def round_stats(self) -> list[RoundStats]:
        rows = self.stats.cpu().numpy()
        return [RoundStats.from_counters(k, c) for k, c in zip(self.kinds, rows)]


def _gather_graph(parts, n: int, cap: int) -> Graph:
    offs, nbrs = [], []
    base = 0
    for off, nb in parts:
        offs.append(off[:-1] + base)
        nbrs.append(nb[: off[-1]])
        base += int(off[-1])
    offsets = np.concatenate(offs + [np.array([base], np.int64)])
    return Graph(num_vertices=n, offsets=offsets, neighbor_ids=np.concatenate(nbrs), max_degree_bound=cap)


def _prepare(dataset: Dataset, params: BuildParams, dev):
    dataset.validate_shape()
    params = effective_params(params, dataset.num_points)
    with torch.cuda.device(dev):
        data_dev = upload(dataset.data, dev)
        check_finite_device(data_dev, dataset.dim)
    validate_params(params, dataset.num_points)
    return params, data_dev


def build_sharded(dataset: Dataset, params: BuildParams, pair_order: str = "disordered", *, group=None,
                  report_stats: list | None = None, metric: str = "l2") -> Graph:
    """Collective: every rank calls it with the same dataset; returns the full Graph on
    every rank.  One rank per GPU (torch.distributed initialised with NCCL)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device(None)
    params, data_dev = _prepare(dataset, params, dev)
    sb = ShardedBuild(data_dev, dataset.dim, params, rank, world, pair_order, group, metric=metric)
    offsets, nbrs, bad, fail = sb.run()
    if int(fail.item()) or int(bad.item()):
        raise DeviceError("sharded build: init sampling failed or invalid graph")
    local_off = offsets.cpu().numpy()
    local_nb = nbrs[: int(local_off[-1])].cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (local_off, local_nb), group=group)
    stats = sb.stats.clone()
    dist.all_reduce(stats, group=group)
    rs = [RoundStats.from_counters(kind, c) for kind, c in zip(sb.kinds, stats.cpu().numpy())]
    if report_stats is not None:
        report_stats.extend(rs)
    return _gather_graph(parts, dataset.num_points, sb.params.R)


def concat_exchange(shards: list[ShardedBuild]) -> list[int]:
    """The all-to-all of P in-process ranks by device copies, in source-rank order.  Every
    destination's inbox is filled before any rank applies (a rank's send buffer doubles as
    its segment-sort scratch during apply)."""
    counts = [[int(x) for x in s.pools.send_counts.cpu().tolist()] for s in shards]
    offs = [np.concatenate([[0], np.cumsum(c)]) for c in counts]
    n_in = []
    for d, dst in enumerate(shards):
        m = 0
        for r, src in enumerate(shards):
            a, b = int(offs[r][d]), int(offs[r][d + 1])
            if m + (b - a) > dst.pools.msg_capacity:
                raise DeviceError(f"rank {d} receives more than {dst.pools.msg_capacity} messages")
            dst.pools.inb[m: m + (b - a)].copy_(src.pools.out[a:b])
            m += b - a
        n_in.append(m)
    return n_in


def build_virtual_shards(dataset: Dataset, params: BuildParams, world: int, pair_order: str = "disordered",
                         *, device=None, report_stats: list | None = None, metric: str = "l2",
                         msg_capacity: int | None = None) -> Graph:
    """P ranks in one process on one GPU: P ``ShardedBuild`` round generators -- the code
    the NCCL path runs -- driven in lock-step with ``concat_exchange``.  Bit-identical to
    build(): the single-GPU check of the multi-GPU path."""
    dev = _device(device)
    params, data_dev = _prepare(dataset, params, dev)
    shards = [ShardedBuild(data_dev, dataset.dim, params, r, world, pair_order, msg_capacity=msg_capacity,
                           metric=metric) for r in range(world)]
    gens = [s.rounds() for s in shards]
    with torch.cuda.device(dev):
        for gen in gens:
            next(gen)
        results = [None] * world
        while results[0] is None:
            n_in = concat_exchange(shards)
            for r, gen in enumerate(gens):
                try:
                    gen.send(n_in[r])
                except StopIteration as stop:
                    results[r] = stop.value
    parts = []
    for offsets, nbrs, bad, fail in results:
        if int(bad.item()) or int(fail.item()):
            raise DeviceError("sharded build produced an invalid graph")
        off = offsets.cpu().numpy()
        parts.append((off, nbrs[: int(off[-1])].cpu().numpy()))
    tot = sum(s.stats for s in shards).cpu().numpy()
    rs = [RoundStats.from_counters(kind, c) for kind, c in zip(shards[0].kinds, tot)]
    if report_stats is not None:
        report_stats.extend(rs)
    return _gather_graph(parts, dataset.num_points, params.R)
