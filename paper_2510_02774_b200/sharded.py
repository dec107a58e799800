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
    MSG_PER_ROW,
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
    optimistic_msg_capacity,
    padded_ld,
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
        # send buffer and inbox: MSG_PER_ROW slots per owned row (the single-GPU build's
        # optimistic capacity; C2's largest round needs ~20).  An emission beyond it is
        # counted on the device (GRNND_ST_LOST); an inbox beyond it is seen by every rank
        # in the counts exchange -- either way build_sharded redoes the build at the
        # worst-case capacity, never on truncated messages.
        mc = msg_capacity if msg_capacity is not None else max(optimistic_msg_capacity(rows, cap), 1024)
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
            raise CapacityError(f"rank receives {n_in} messages > capacity {self.msg_capacity}")
        p = self.struct(stats)
        _lib.call("grnnd_round_apply", C.byref(p), kind, int(n_in), _stream(self.dev))
        self.swap()


class CapacityError(DeviceError):
    """A round needs more message slots than the workspace holds (raised on every rank)."""


def exchange_all_to_all(out: torch.Tensor, send_counts: list[int], inb: torch.Tensor, group=None) -> int:
    """The per-round exchange over torch.distributed (NCCL on GPUs, gloo on CPU): ONE
    all-gather of every rank's P send counts (so each rank sees every inbox size and an
    over-full inbox anywhere stops all ranks together, before the payload moves), then
    ONE all-to-all of the packed [m, MSG_WORDS] payload, received in source-rank order
    into ``inb``.  Returns the number of messages received."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if out.is_cuda and dist.get_backend(group) == "gloo":
        # gloo's all-to-all moves host tensors: stage through the host (functional multi-rank
        # runs on one GPU, where NCCL refuses two ranks per device)
        inb_h = torch.empty(inb.shape, dtype=inb.dtype)
        n_in = exchange_all_to_all(out.cpu(), send_counts, inb_h, group)
        inb[:n_in].copy_(inb_h[:n_in])
        return n_in
    dev = out.device
    sc = torch.tensor(list(send_counts) + [inb.shape[0]], dtype=torch.int64, device=dev)
    allc = torch.empty(world * (world + 1), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, sc, group=group)
    m = allc.cpu().view(world, world + 1)  # [source, destination] counts + each rank's inbox capacity
    recv_counts = [int(x) for x in m[:, rank].tolist()]
    n_out, n_in = sum(send_counts), sum(recv_counts)
    inbox = m[:, :world].sum(0)
    over = [r for r in range(world) if int(inbox[r]) > int(m[r, world])]
    if over:
        raise CapacityError(f"rank(s) {over} receive more messages than their inbox holds "
                            f"({[int(inbox[r]) for r in over]} > {[int(m[r, world]) for r in over]})")
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
                 pair_order: str = "disordered", group=None, msg_capacity=None, metric: str = "l2",
                 normalize_in_place: bool = False):
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
        # IP works on L2-normalised rows: a working copy keeps the caller's rows for reruns;
        # normalize_in_place (C5: no room for a second 38.4 GB copy) normalises them once
        self.copy_rows = metric == "ip" and not normalize_in_place
        if metric == "ip" and normalize_in_place:
            normalize_rows_(data_dev, dim)
        work = torch.empty_like(data_dev) if self.copy_rows else data_dev
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
        if self.copy_rows:
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


def run_sharded(data_dev: torch.Tensor, dim: int, params: BuildParams, rank: int, world: int,
                pair_order: str = "disordered", group=None, *, metric: str = "l2", exchange: Callable | None = None,
                phase_events: list | None = None):
    """This rank's build with the optimistic message capacity; if any rank's round
    outgrows it (an emission the device counted as lost, or an over-full inbox seen in the
    counts exchange) every rank redoes the build at the worst-case capacity -- the same
    rule as the single-GPU build().  Returns (ShardedBuild, offsets, nbrs, bad, fail)."""
    import torch.distributed as dist

    for attempt in range(2):
        mc = None if attempt == 0 else max(2 * (shard_bounds(int(data_dev.shape[0]), world)[rank + 1]
                                                - shard_bounds(int(data_dev.shape[0]), world)[rank]) * params.R, 1024)
        sb = ShardedBuild(data_dev, dim, params, rank, world, pair_order, group, msg_capacity=mc, metric=metric)
        try:
            offsets, nbrs, bad, fail = sb.run(phase_events, exchange)
            lost = int(sb.stats[:, _lib.ST_LOST].sum().item())
        except CapacityError:
            if attempt:
                raise
            lost = 1
        flag = torch.tensor([lost], dtype=torch.int64, device=data_dev.device)
        if dist.is_initialized():
            dist.all_reduce(flag, group=group)
        if attempt == 0 and int(flag.item()):
            del sb
            continue
        if int(flag.item()):
            raise CapacityError("sharded build lost messages at the worst-case capacity")
        return sb, offsets, nbrs, bad, fail


def memory_plan(n: int, dim: int, R: int, world: int = 1, metric: str = "l2", *,
                msg_per_row: int = MSG_PER_ROW, normalize_in_place: bool = False) -> dict:
    """Per-rank device bytes of a sharded build (the largest shard): replicated vectors
    (fp32 [N, ld]; IP keeps a normalised working copy next to the caller's rows unless the
    caller normalises in place), the row norms of the tensor-core filter, the one pool
    buffer of the owned rows, the workspace (grnnd_workspace_bytes: messages, pair records,
    masks, staging) and the CSR emitted at the end.  SURVEY 8(d) C5: 100M x 96 at P=8."""
    rows = max(hi - lo for lo, hi in zip(shard_bounds(n, world), shard_bounds(n, world)[1:]))
    ld = padded_ld(dim)
    mc = max(min(max(rows * R, 1), max(msg_per_row * rows, 1 << 16)), 1024)
    plan = {
        "vectors": n * ld * 4,
        "vectors_ip_copy": n * ld * 4 if metric == "ip" and not normalize_in_place else 0,
        "norms": n * 4,
        "pools": rows * R * 8 + rows * 4,
        "workspace": int(_lib.lib.grnnd_workspace_bytes(rows, R, mc)),
        "csr": (rows + 1) * 8 + rows * R * 4,
    }
    plan["total"] = sum(plan.values())
    plan.update(rows=rows, msg_capacity=mc)
    return plan


def generate_device(n: int, dim: int, seed: int = 1, device=None) -> torch.Tensor:
    """Seeded standard-normal fp32 [n, ld] (zero-padded) generated on the device (torch's
    counter-based Philox), for corpora with no host twin (C5: 38.4 GB); every rank that
    calls it with the same arguments gets the same rows."""
    dev = _device(device)
    ld = padded_ld(dim)
    out = torch.zeros((n, ld), dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    chunk = max(1, (1 << 28) // ld)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b, :dim].normal_(generator=gen)
    return out


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
    sb, offsets, nbrs, bad, fail = run_sharded(data_dev, dataset.dim, params, rank, world, pair_order, group,
                                               metric=metric)
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
                raise CapacityError(f"rank {d} receives more than {dst.pools.msg_capacity} messages")
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
