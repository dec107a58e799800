"""Multi-GPU GRNND build: replicated vectors, contiguous-ID-range vertex ownership, one
message exchange per round.

The reference has no distributed path (paper future work PAPER.md:3927).
Each rank owns pools [lo, hi) = [r*N/P, (r+1)*N/P).  A round is

    emit   grnnd_round_emit   pair phase (or reverse selection) of owned vertices, the
                              messages bucketed by the owner rank of their target;
    swap   counts all-to-all, then key / tgt / id / dist all-to-all (NCCL over NVLink);
    apply  grnnd_round_apply  group the received messages by target, sort each segment
                              by key, three-stage insert (own entries spliced as on 1 GPU).

A message's key is source * R + emission index -- its position in the reference's global
vertex-major order -- so the receiving side restores exactly the single-GPU per-pool
order: a P-rank build is bit-identical to the 1-GPU build (and so to the reference).

``build_virtual_shards`` runs P ranks in one process on one GPU with the exchange done by
concatenation; it exercises the sharded kernels end to end where only one GPU exists.
``exchange_all_to_all`` is the host logic of the NCCL path and is also covered on CPU
(gloo, world_size 2) by tests/test_sharded.py.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .builder import (
    _ORDER_CODES,
    MASK64,
    STREAM_ROUND_BASE,
    RoundStats,
    _accumulate,
    _DevicePools,
    _device,
    _finalize_device,
    _stream,
    check_finite_device,
    effective_params,
    num_rounds,
    upload,
)
from .core import BuildParams, Dataset, Graph, validate_params
from .errors import DeviceError, ParamError

FIELDS = (("key", torch.int64), ("tgt", torch.int32), ("id", torch.int32), ("dist", torch.float32))


def shard_bounds(n: int, world: int) -> list[int]:
    """Contiguous ownership ranges: rank r owns [b[r], b[r+1])."""
    return [n * r // world for r in range(world + 1)]


class ShardPools(_DevicePools):
    """One rank's pools plus typed views of the workspace's send / receive lists."""

    def __init__(self, data_dev, dim, cap, lo, hi, n_total, world, msg_capacity=None):
        rows = hi - lo
        # outgoing <= sum(k) of owned rows; incoming is data dependent (hubs): 2x headroom,
        # overflow is detected and reported (never silently truncated)
        mc = msg_capacity if msg_capacity is not None else max(2 * rows * cap, 1024)
        super().__init__(data_dev, dim, cap, lo=lo, hi=hi, n_total=n_total, msg_capacity=mc)
        self.world = world
        p = self.struct()
        ptrs = [C.c_void_p() for _ in range(8)]
        _lib.call("grnnd_round_buffers", C.byref(p), *[C.byref(x) for x in ptrs])
        base = self.workspace.data_ptr()

        def view(ptr, dtype):
            off = ptr.value - base
            nbytes = self.msg_capacity * torch.empty(0, dtype=dtype).element_size()
            return self.workspace[off : off + nbytes].view(dtype)

        self.out = {f: view(ptrs[i], dt) for i, (f, dt) in enumerate(FIELDS)}
        self.inb = {f: view(ptrs[4 + i], dt) for i, (f, dt) in enumerate(FIELDS)}
        self.send_counts = torch.zeros(world, dtype=torch.int64, device=self.dev)

    def emit(self, kind: int, seed: int, stream_id: int, order: int, rho: float, bounds_dev: torch.Tensor,
             stats: torch.Tensor) -> None:
        p = self.struct(stats, kind != 0 or self.filtered_round(stream_id))
        _lib.call("grnnd_round_emit", C.byref(p), kind, seed & MASK64, stream_id & MASK64, order, float(rho),
                  bounds_dev.data_ptr(), self.world, self.send_counts.data_ptr(), _stream(self.dev))

    def apply(self, kind: int, n_in: int, stats: torch.Tensor) -> None:
        if n_in > self.msg_capacity:
            raise DeviceError(f"rank receives {n_in} messages > capacity {self.msg_capacity}")
        p = self.struct(stats)
        _lib.call("grnnd_round_apply", C.byref(p), kind, int(n_in), _stream(self.dev))
        self.swap()


def exchange_all_to_all(out: dict, send_counts: list[int], inb: dict, group=None) -> int:
    """The per-round exchange over torch.distributed (NCCL on GPUs, gloo on CPU):
    counts all-to-all, then one all-to-all per message field, received in source-rank
    order into ``inb``.  Returns the number of messages received."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = out["key"].device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.cpu().tolist()]
    n_out, n_in = sum(send_counts), sum(recv_counts)
    if n_in > inb["key"].numel():
        raise DeviceError(f"rank receives {n_in} messages > capacity {inb['key'].numel()}")
    for f, _ in FIELDS:
        dist.all_to_all_single(inb[f][:n_in], out[f][:n_out], output_split_sizes=recv_counts,
                               input_split_sizes=send_counts, group=group)
    return n_in


class ShardedBuild:
    """This rank's part of a sharded build (torch.distributed already initialised)."""

    def __init__(self, data_dev: torch.Tensor, dim: int, params: BuildParams, rank: int, world: int,
                 pair_order: str = "disordered", group=None, msg_capacity=None):
        n = int(data_dev.shape[0])
        self.params = effective_params(params, n)
        validate_params(self.params, n)
        if pair_order not in _ORDER_CODES:
            raise ParamError(f"pair_order must be one of {sorted(_ORDER_CODES)}")
        self.order = _ORDER_CODES[pair_order]
        self.rank, self.world, self.group = rank, world, group
        self.bounds = shard_bounds(n, world)
        self.bounds_dev = torch.tensor(self.bounds, dtype=torch.int64, device=data_dev.device)
        self.pools = ShardPools(data_dev, dim, self.params.R, self.bounds[rank], self.bounds[rank + 1], n, world,
                                msg_capacity)
        self.stats = torch.zeros((num_rounds(self.params), _lib.NSTATS), dtype=torch.int64, device=data_dev.device)
        self.kinds: list[str] = []

    def run(self, phase_events: list | None = None):
        """One sharded build; same contract as builder.DeviceBuild.run (offsets, nbrs,
        bad, fail for this rank's rows).  phase_events gets (start, emitted, applied)
        CUDA-event triples of the update rounds (the emitted->applied span includes the
        exchange)."""
        p, pools = self.params, self.pools
        self.stats.zero_()
        self.kinds = []
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
                sc = [int(x) for x in pools.send_counts.cpu().tolist()]
                n_in = exchange_all_to_all(pools.out, sc, pools.inb, self.group)
                pools.apply(kind, n_in, self.stats[i])
                if ev:
                    ev[2].record()
                if kind == 0:
                    ri += 1
                self.kinds.append("update" if kind == 0 else "reverse")
                i += 1
        offsets, nbrs, bad = _finalize_device(pools)
        return offsets, nbrs, bad, fail

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


def build_sharded(dataset: Dataset, params: BuildParams, pair_order: str = "disordered", *, group=None,
                  report_stats: list | None = None) -> Graph:
    """Collective: every rank calls it with the same dataset; returns the full Graph on
    every rank.  One rank per GPU (torch.distributed initialised with NCCL)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device(None)
    dataset.validate_shape()
    data_dev = upload(dataset.data, dev)
    check_finite_device(data_dev, dataset.dim)
    sb = ShardedBuild(data_dev, dataset.dim, params, rank, world, pair_order, group)
    offsets, nbrs, bad, fail = sb.run()
    if int(fail.item()) or int(bad.item()):
        raise DeviceError("sharded build: init sampling failed or invalid graph")
    local_off = offsets.cpu().numpy()
    local_nb = nbrs[: int(local_off[-1])].cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (local_off, local_nb), group=group)
    stats = sb.stats.clone()
    dist.all_reduce(stats, group=group)
    if report_stats is not None:
        for kind, c in zip(sb.kinds, stats.cpu().numpy()):
            report_stats.append(RoundStats.from_counters(kind, c))
    return _gather_graph(parts, dataset.num_points, sb.params.R)


def build_virtual_shards(dataset: Dataset, params: BuildParams, world: int, pair_order: str = "disordered",
                         *, device=None, report_stats: list | None = None) -> Graph:
    """P ranks in one process on one GPU: the sharded kernels (owned ranges, rank
    bucketing, keyed regrouping) with the all-to-all done by concatenation in source-rank
    order.  Bit-identical to build() -- the single-GPU check of the multi-GPU path."""
    dev = _device(device)
    params = effective_params(params, dataset.num_points)
    validate_params(params, dataset.num_points)
    order = _ORDER_CODES[pair_order]
    data_dev = upload(dataset.data, dev)
    check_finite_device(data_dev, dataset.dim)
    n = dataset.num_points
    bounds = shard_bounds(n, world)
    bounds_dev = torch.tensor(bounds, dtype=torch.int64, device=dev)
    shards = [ShardPools(data_dev, dataset.dim, params.R, bounds[r], bounds[r + 1], n, world) for r in range(world)]
    rounds = num_rounds(params)
    stats = torch.zeros((world, rounds, _lib.NSTATS), dtype=torch.int64, device=dev)
    for s in shards:
        s.init(params.S, params.seed)
    kinds = []
    ri = 0
    for t1 in range(1, params.T1 + 1):
        sched = [0] * params.T2 + ([1] if t1 != params.T1 else [])
        for kind in sched:
            i = len(kinds)
            for r, s in enumerate(shards):
                s.emit(kind, params.seed, STREAM_ROUND_BASE + ri, order, params.rho, bounds_dev, stats[r, i])
            sends = [[int(x) for x in s.send_counts.cpu().tolist()] for s in shards]
            offs = [np.concatenate([[0], np.cumsum(sc)]) for sc in sends]
            for d, dst in enumerate(shards):
                n_in = 0
                for src_r, src in enumerate(shards):
                    a, b = int(offs[src_r][d]), int(offs[src_r][d + 1])
                    for f, _ in FIELDS:
                        dst.inb[f][n_in : n_in + (b - a)].copy_(src.out[f][a:b])
                    n_in += b - a
                dst.apply(kind, n_in, stats[d, i])
            if kind == 0:
                ri += 1
            kinds.append("update" if kind == 0 else "reverse")
    parts = []
    for s in shards:
        offsets, nbrs, bad = _finalize_device(s)
        if int(bad.item()):
            raise DeviceError("sharded build produced an invalid graph")
        off = offsets.cpu().numpy()
        parts.append((off, nbrs[: int(off[-1])].cpu().numpy()))
    if report_stats is not None:
        tot = stats.sum(0).cpu().numpy()
        for kind, c in zip(kinds, tot):
            report_stats.append(RoundStats.from_counters(kind, c))
    return _gather_graph(parts, n, params.R)
