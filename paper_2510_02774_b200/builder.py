"""GRNND graph construction on B200: the drop-in for the reference builder.

Public surface and semantics follow /root/reference/pkg/src/grnnd/builder.py:
``build`` (:365-390), the stepwise ``init_neighbors`` (:221-257),
``update_round`` (:283-312), ``reverse_edge_sampling`` (:315-339),
``finalize_graph`` (:342-362), ``validate_state`` (:393-422), the scalar
specs ``rng_redirect_check`` (:52-63) / ``cooperative_insert`` (:66-99),
``RoundStats`` (:102-114) and ``effective_params`` (:209-218).

What differs is where the work runs: the pools live in HBM as torch tensors
(PyTorch is the device allocator and stream provider only) and every round is
one asynchronous call into libgrnnd_b200.so (hand-written sm_100a kernels,
include/grnnd_b200.h).  Results are bit-identical to the reference's numba
backend: same RNG streams, same exact fp32 distance arithmetic, same per-pool
message order.  There is no CPU fallback; without a CUDA device the build
raises.
"""

from __future__ import annotations

import ctypes as C
import os
import warnings
from dataclasses import dataclass, field, replace
from typing import Literal, NamedTuple

import numpy as np
import torch

from . import _lib
from .core import TOMBSTONE, BuildParams, Dataset, DoubleBufferPool, Graph, validate_params
from .errors import DeviceError, ParamError, SelfInsert

MASK64 = (1 << 64) - 1
STREAM_ROUND_BASE = 1  # rng.py:17 -- update round r uses stream 1 + r
PairOrder = Literal["disordered", "ascending"]
_ORDER_CODES = {"disordered": 0, "ascending": 1}


# ----------------------------------------------------------------------------------
# scalar specs (host, used by tests as in the reference)
# ----------------------------------------------------------------------------------
class Redirect(NamedTuple):
    far: int
    close: int


def rng_redirect_check(d_vi: float, d_vj: float, d_ij: float) -> Redirect | None:
    """The pair rule: redirect the farther member iff d_ij < max(d_vi, d_vj);
    an exact tie of the owner distances keeps the first member (builder.py:52-63)."""
    if not d_ij < max(d_vi, d_vj):
        return None
    return Redirect(1, 0) if d_vj >= d_vi else Redirect(0, 1)


def cooperative_insert(owner, write_ids, write_dists, count, candidate_id, candidate_dist):
    """Scalar three-stage insert spec (builder.py:66-99): dedupe, append, or
    replace the first farthest slot when strictly closer.  Returns (status, count)."""
    if candidate_id == owner:
        raise SelfInsert(f"pool {owner} asked to insert its own owner")
    if candidate_id in write_ids[:count]:
        return "duplicate", count
    cap = write_ids.shape[0]
    if count < cap:
        write_ids[count] = candidate_id
        write_dists[count] = candidate_dist
        return "inserted", count + 1
    worst = int(np.argmax(write_dists))  # first index of the maximum
    if candidate_dist < write_dists[worst]:
        write_ids[worst] = candidate_id
        write_dists[worst] = np.float32(candidate_dist)
        return "replaced", count
    return "rejected", count


@dataclass
class RoundStats:
    kind: str
    messages: int = 0
    redirects: int = 0
    survivors: int = 0
    reverse_attempts: int = 0
    inserted: int = 0
    duplicate: int = 0
    replaced: int = 0
    rejected: int = 0
    # instrumentation (not in the reference): pair distances computed / evaluated
    pairs: int = field(default=0, compare=False, repr=False)
    pairs_ref: int = field(default=0, compare=False, repr=False)
    candidates: int = field(default=0, compare=False, repr=False)  # filter band re-evaluations
    redirectable: int = field(default=0, compare=False, repr=False)  # pairs meeting the redirect condition
    record_pools: int = field(default=0, compare=False, repr=False)  # pools with >= 1 such pair
    active_entries: int = field(default=0, compare=False, repr=False)  # entries whose pair phase ran

    @classmethod
    def from_counters(cls, kind: str, c) -> "RoundStats":
        c = [int(x) for x in c]
        if c[_lib.ST_LOST]:
            raise DeviceError(f"{kind} round lost {c[_lib.ST_LOST]} message(s): the message capacity of the "
                              "workspace is too small for this round (GRNND_EWORKSPACE)")
        st = cls(
            kind=kind,
            messages=c[_lib.ST_MESSAGES],
            redirects=c[_lib.ST_REDIRECTS],
            survivors=c[_lib.ST_SURVIVORS],
            reverse_attempts=c[_lib.ST_REVERSE_ATTEMPTS],
            inserted=c[_lib.ST_INSERTED],
            duplicate=c[_lib.ST_DUPLICATE],
            replaced=c[_lib.ST_REPLACED],
            rejected=c[_lib.ST_REJECTED],
            pairs=c[_lib.ST_PAIRS],
            pairs_ref=c[_lib.ST_PAIRS_REF],
            candidates=c[_lib.ST_CANDIDATES],
            redirectable=c[_lib.ST_REDIRECTABLE],
            record_pools=c[_lib.ST_RECPOOLS],
            active_entries=c[_lib.ST_ACTIVE_K],
        )
        if kind == "update":
            st.survivors = st.messages - st.redirects
        return st


def _accumulate(totals: RoundStats, s: RoundStats) -> None:
    for f in ("messages", "redirects", "survivors", "reverse_attempts", "inserted",
              "duplicate", "replaced", "rejected", "pairs", "pairs_ref"):
        setattr(totals, f, getattr(totals, f) + getattr(s, f))


def effective_params(params: BuildParams, n: int) -> BuildParams:
    """Clamp S and R for tiny datasets, with a warning (builder.py:209-218)."""
    if n >= 2 and (params.S > n - 1 or params.R > n - 1):
        r = min(params.R, n - 1)
        s = min(params.S, r)
        warnings.warn(f"dataset has only {n} points; clamping S={params.S}->{s}, R={params.R}->{r}")
        params = replace(params, S=s, R=r)
    return params


# ----------------------------------------------------------------------------------
# device plumbing
# ----------------------------------------------------------------------------------
def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("the B200 GRNND builder needs a CUDA device (no CPU fallback)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise DeviceError(f"device must be a CUDA device, got {dev}")
    return dev


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def padded_ld(dim: int) -> int:
    """Row stride of the device copy: a multiple of 4 floats (16-byte rows for
    vectorised gathers); padding columns are zero, which leaves every exact
    squared distance unchanged (adding +0.0 is exact)."""
    return (dim + 3) // 4 * 4


def upload(data: np.ndarray | torch.Tensor, dev: torch.device) -> torch.Tensor:
    """Host (or device) fp32 [N, D] -> device fp32 [N, ld] with zero padding."""
    if isinstance(data, torch.Tensor):
        src = data
    else:
        src = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32))
    n, dim = src.shape
    ld = padded_ld(dim)
    if ld == dim:
        return src.to(dev, dtype=torch.float32, non_blocking=src.is_pinned()).contiguous()
    out = torch.zeros((n, ld), dtype=torch.float32, device=dev)
    out[:, :dim].copy_(src, non_blocking=src.is_pinned())
    return out


def check_finite_device(data_dev: torch.Tensor, dim: int) -> None:
    """Dataset.validate's finiteness scan (core.py:70-71), on the GPU."""
    n, ld = data_dev.shape
    flag = torch.zeros(1, dtype=torch.int64, device=data_dev.device)
    _lib.call("grnnd_check_finite", data_dev.data_ptr(), n, dim, ld, flag.data_ptr(), _stream(data_dev.device))
    if int(flag.item()):
        raise ParamError("dataset contains non-finite values")


EXACT_FIRST_ROUNDS = 3  # update rounds (stream ids 1..3) that run the exact-only pair phase
EXACT_FIRST_ROUNDS_MULTI = 5  # the same for D > 128
METRICS = ("l2", "ip")


def check_metric(metric: str) -> None:
    if metric not in METRICS:
        raise ParamError(f"metric must be one of {METRICS}, got {metric!r}")


def normalize_rows_(data_dev: torch.Tensor, dim: int) -> torch.Tensor:
    """IP metric (SURVEY 7 hard part 6; the reference has L2 only): rows scaled in place to
    unit norm on the device, so the squared L2 the build uses is 2 - 2<a, b>."""
    n, ld = data_dev.shape
    with torch.cuda.device(data_dev.device):
        _lib.call("grnnd_normalize_rows", data_dev.data_ptr(), n, dim, ld, _stream(data_dev.device))
    return data_dev


def _on_device(method):
    """Run a pools method with the pools' device current: the library launches onto that
    device's current stream, and the CUDA runtime's current device must match it."""
    import functools

    @functools.wraps(method)
    def wrapper(self, *a, **k):
        with torch.cuda.device(self.dev):
            return method(self, *a, **k)

    return wrapper


class _DevicePools:
    """The double-buffered pools of owned rows [lo, hi) plus round scratch, in HBM."""

    def __init__(self, data_dev: torch.Tensor, dim: int, cap: int, lo: int = 0, hi: int | None = None,
                 n_total: int | None = None, msg_capacity: int | None = None, filtered: bool | None = None,
                 in_place: bool = True):
        dev = data_dev.device
        self.dev = dev
        self.data = data_dev
        self.n_total = int(n_total if n_total is not None else data_dev.shape[0])
        self.lo = int(lo)
        self.hi = int(hi if hi is not None else self.n_total)
        self.dim = int(dim)
        self.ld = int(data_dev.shape[1])
        self.cap = int(cap)
        if self.cap > _lib.MAX_CAP:
            raise ParamError(f"R={cap} exceeds the {_lib.MAX_CAP} slots the B200 kernels are built for")
        rows = self.hi - self.lo
        self.rows = rows
        self.msg_capacity = int(msg_capacity if msg_capacity is not None else max(rows * cap, 1))
        i32, f32 = torch.int32, torch.float32
        self.read_ids = torch.empty((rows, cap), dtype=i32, device=dev)
        self.read_dists = torch.empty((rows, cap), dtype=f32, device=dev)
        self.read_count = torch.zeros(rows, dtype=i32, device=dev)
        # in place (default): ONE pool buffer.  A round's apply runs after its whole pair
        # phase and rewrites only the pools that changed (incoming messages or tombstones),
        # each from its own row -- the reference's cleared write buffer + swap, without the
        # copy of every unchanged pool.  The double-buffered layout remains for states built
        # with non-empty write buffers (the reference's manual-state tests).
        self.in_place = bool(in_place)
        if self.in_place:
            self.write_ids, self.write_dists, self.write_count = self.read_ids, self.read_dists, self.read_count
        else:
            self.write_ids = torch.empty((rows, cap), dtype=i32, device=dev)
            self.write_dists = torch.empty((rows, cap), dtype=f32, device=dev)
            self.write_count = torch.zeros(rows, dtype=i32, device=dev)
        ws = int(_lib.lib.grnnd_workspace_bytes(rows, cap, self.msg_capacity))
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self.scratch_stats = torch.zeros(_lib.NSTATS, dtype=torch.int64, device=dev)
        self.version = 0  # bumped on every state change (host snapshot cache key)
        # filtered pair phase (FFMA dot pre-screen + exact re-evaluation near the threshold;
        # same graph as the exact-only phase): needs the squared norms of every row
        if filtered is None:
            filtered = os.environ.get("GRNND_EXACT_PAIRS", "0") != "1"
        self.norms = None
        self._filter_ok = None
        self.band_ratio = None
        if filtered:
            self.norms = torch.empty(self.n_total, dtype=f32, device=dev)
            self.compute_norms()

    def compute_norms(self) -> None:
        """Squared row norms of the vectors (the tensor-core pre-screen's |a|^2 terms)."""
        if self.norms is not None:
            with torch.cuda.device(self.dev):
                _lib.call("grnnd_row_norms", self.data.data_ptr(), self.n_total, self.dim, self.ld,
                          self.norms.data_ptr(), _stream(self.dev))

    def struct(self, stats: torch.Tensor | None = None, filtered: "bool | int" = True) -> _lib.Pools:
        """filtered: False / 0 exact pair phase, True / 1 TF32 filter, 2 split-TF32 filter."""
        norms = self.norms if filtered else None
        return _lib.Pools(
            self.data.data_ptr(), self.n_total, self.lo, self.hi, self.dim, self.ld, self.cap,
            self.read_ids.data_ptr(), self.read_dists.data_ptr(), self.read_count.data_ptr(),
            self.write_ids.data_ptr(), self.write_dists.data_ptr(), self.write_count.data_ptr(),
            self.workspace.data_ptr(), self.workspace.numel(), self.msg_capacity,
            (stats if stats is not None else self.scratch_stats).data_ptr(),
            norms.data_ptr() if norms is not None else None,
            1 if (filtered == 2 and norms is not None) else 0,
        )

    BAND_LIMIT = 0.05  # filter band / mean stored distance above which plain TF32 is not used

    def filtered_round(self, stream_id: int) -> int:
        """Pair-phase mode of an update round.  The first rounds start from random pools,
        where most pairs meet the redirect condition (68% / 32% / 17% of all pairs in rounds
        1-3 at C2) and the tensor-core filter settles few of them: those rounds run the
        exact-only pair phase; later rounds the filtered one.  The plain TF32 filter's error
        band (2^-8 (|a|^2 + |b|^2)) is wide when the data lie far from the origin
        relative to their neighbour distances (clustered data: 85% of pairs would be
        candidates); such builds keep the exact pair phase.  (The split-TF32 Gram, band
        2^-15 (|a|^2 + |b|^2), settles those pairs -- candidates drop to the redirect-capable
        ones -- but its three MMAs per k-block made it slower than the exact tile kernel on
        C2c; GRNND_FORCE_FILTER=2 selects it.)  The band is measured once, at the first
        filtered round (one host read per build).  Returns 0 (exact), 1 (TF32) or 2 (split
        TF32); the graph is the same either way."""
        # (D > 128: the tensor-core kernel's exact chains gather both rows of every candidate
        # from L2, so the redirect-dense rounds 4-5 run faster on the exact tile kernel too:
        # C3 1.78 -> 1.67 s)
        first = EXACT_FIRST_ROUNDS if self.dim <= 128 else EXACT_FIRST_ROUNDS_MULTI
        if stream_id <= int(os.environ.get("GRNND_EXACT_FIRST_ROUNDS", first)):
            return 0
        if self.norms is None:
            return 0
        force = os.environ.get("GRNND_FORCE_FILTER")  # tests / A-B runs: 0 exact, 1 TF32, 2 split
        if force in ("0", "1", "2"):
            return int(force)
        if self._filter_ok is None:
            out = torch.zeros(2, dtype=torch.float64, device=self.dev)
            with torch.cuda.device(self.dev):
                _lib.call("grnnd_band_terms", C.byref(self.struct()), out.data_ptr(), _stream(self.dev))
            sr, cnt = (float(x) for x in out.cpu())
            self.band_ratio = 2.0 ** -7 * sr / max(cnt, 1.0)  # mean band / stored distance
            self._filter_ok = 1 if self.band_ratio <= self.BAND_LIMIT else 0
        return self._filter_ok

    def swap(self) -> None:
        """clear_and_swap (builder.py:170-176): the written buffers become the read
        side; the old read side is logically cleared (count 0; slots beyond a row's
        count are never read)."""
        if not self.in_place:
            self.read_ids, self.write_ids = self.write_ids, self.read_ids
            self.read_dists, self.write_dists = self.write_dists, self.read_dists
            self.read_count, self.write_count = self.write_count, self.read_count
            self.write_count.zero_()
        self.version += 1

    # -- the four asynchronous steps --
    @_on_device
    def init(self, S: int, seed: int) -> torch.Tensor:
        fail = torch.zeros(1, dtype=torch.int64, device=self.dev)
        p = self.struct()
        _lib.call("grnnd_init_pools", C.byref(p), S, seed & MASK64, fail.data_ptr(), _stream(self.dev))
        self.version += 1
        self._filter_ok = None  # re-measured by the next build's first filtered round
        return fail

    @_on_device
    def update(self, seed: int, stream_id: int, order_code: int, stats: torch.Tensor) -> None:
        p = self.struct(stats, self.filtered_round(stream_id))
        _lib.call("grnnd_update_round", C.byref(p), seed & MASK64, stream_id & MASK64, order_code,
                  _stream(self.dev))
        self.swap()

    @_on_device
    def reverse(self, rho: float, stats: torch.Tensor) -> None:
        p = self.struct(stats)
        _lib.call("grnnd_reverse_round", C.byref(p), float(rho), _stream(self.dev))
        self.swap()

    @_on_device
    def update_split(self, seed: int, stream_id: int, order_code: int, stats: torch.Tensor,
                     ev: tuple | None = None) -> None:
        """update() as its two halves with optional CUDA events (before emit, after emit,
        after apply) for per-phase timing on the launching stream."""
        p = self.struct(stats, self.filtered_round(stream_id))
        st = _stream(self.dev)
        if ev:
            ev[0].record()
        _lib.call("grnnd_update_emit", C.byref(p), seed & MASK64, stream_id & MASK64, order_code, st)
        if ev:
            ev[1].record()
        _lib.call("grnnd_apply_emitted", C.byref(p), 0, st)
        if ev:
            ev[2].record()
        self.swap()

    @_on_device
    def finalize(self, offsets: torch.Tensor, nbrs: torch.Tensor, bad: torch.Tensor) -> None:
        p = self.struct()
        _lib.call("grnnd_finalize_pools", C.byref(p), offsets.data_ptr(), nbrs.data_ptr(), bad.data_ptr(),
                  _stream(self.dev))

    @_on_device
    def sorted_rows(self) -> torch.Tensor:
        out = torch.empty((self.rows, self.cap), dtype=torch.int32, device=self.dev)
        _lib.call("grnnd_sorted_rows", self.read_ids.data_ptr(), self.read_dists.data_ptr(),
                  self.read_count.data_ptr(), self.rows, self.cap, out.data_ptr(), _stream(self.dev))
        return out


# ----------------------------------------------------------------------------------
# the drop-in build state and stepwise API
# ----------------------------------------------------------------------------------
class BuildState:
    """Device-resident twin of builder.BuildState (builder.py:117-176).

    Two constructors: the internal one (``BuildState(dataset, params, pools)``) and the
    reference's keyword form ``BuildState(data=..., params=..., read_ids=..., read_dists=...,
    read_count=..., write_ids=..., write_dists=..., write_count=..., round_index=0,
    pair_order="disordered")`` (test_builder.py:89), which uploads the arrays.

    ``read_ids`` / ``read_dists`` / ``read_count`` / ``write_*`` are READ-ONLY host
    snapshots (numpy, ``writeable=False``; slots beyond a row's count read as TOMBSTONE /
    inf like the reference's cleared buffers), cached until the next round or swap: one
    device-to-host copy per state change, not per access.  The live tensors are
    ``state.pools.read_ids`` etc.
    """

    def __init__(self, dataset=None, params: BuildParams | None = None, pools: "_DevicePools | None" = None,
                 pair_order: str = "disordered", *, data=None, read_ids=None, read_dists=None, read_count=None,
                 write_ids=None, write_dists=None, write_count=None, round_index: int = 0, totals=None,
                 device=None):
        if pools is None:
            if data is None and dataset is not None:
                data = dataset.data if isinstance(dataset, Dataset) else dataset
            if data is None or read_ids is None or read_dists is None or read_count is None:
                raise ParamError("BuildState needs (dataset, params, pools) or data= and the read_* arrays")
            ds = data if isinstance(data, Dataset) else Dataset(data)
            ri = np.ascontiguousarray(read_ids, dtype=np.int32)
            n, cap = ri.shape
            dev = _device(device)
            with torch.cuda.device(dev):
                wc_given = write_count is not None and np.any(np.asarray(write_count) != 0)
                pools = _DevicePools(upload(ds.data, dev), ds.dim, cap, in_place=not wc_given)
                pools.read_ids.copy_(torch.from_numpy(ri))
                pools.read_dists.copy_(torch.from_numpy(np.ascontiguousarray(read_dists, dtype=np.float32)))
                pools.read_count.copy_(torch.from_numpy(np.ascontiguousarray(read_count, dtype=np.int32)))
                if wc_given:
                    wc = np.ascontiguousarray(write_count, dtype=np.int32)
                    pools.write_count.copy_(torch.from_numpy(wc))
                    if write_ids is not None:
                        pools.write_ids.copy_(torch.from_numpy(np.ascontiguousarray(write_ids, dtype=np.int32)))
                    if write_dists is not None:
                        pools.write_dists.copy_(torch.from_numpy(np.ascontiguousarray(write_dists, dtype=np.float32)))
            dataset = ds
        self.dataset = dataset
        self.params = params
        self.pools = pools
        self.pair_order = pair_order
        self.round_index = round_index
        self.totals = totals if totals is not None else RoundStats(kind="total")
        self._snap: dict = {}
        self._snap_version = -1

    # --- shape ---
    @property
    def num_vertices(self) -> int:
        return self.pools.rows

    @property
    def capacity(self) -> int:
        return self.pools.cap

    @property
    def data(self) -> np.ndarray:
        return self.dataset.data

    # --- host snapshots (read-only, cached per pool version) ---
    def _cached(self, side: str):
        if self._snap_version != self.pools.version:
            self._snap = {}
            self._snap_version = self.pools.version
        if side not in self._snap:
            P = self.pools
            if side == "write" and P.in_place:  # logically cleared between rounds
                n, cap = P.rows, P.cap
                out = (np.full((n, cap), TOMBSTONE, np.int32), np.full((n, cap), np.inf, np.float32),
                       np.zeros(n, np.int32))
            else:
                ids, dists, counts = ((P.read_ids, P.read_dists, P.read_count) if side == "read"
                                      else (P.write_ids, P.write_dists, P.write_count))
                out = self._masked(ids, dists, counts)
            for a in out:
                a.setflags(write=False)
            self._snap[side] = out
        return self._snap[side]

    def _masked(self, ids: torch.Tensor, dists: torch.Tensor, counts: torch.Tensor):
        c = counts.cpu().numpy().astype(np.int32)
        i = ids.cpu().numpy()
        d = dists.cpu().numpy()
        valid = np.arange(self.capacity)[None, :] < c[:, None]
        return np.where(valid, i, TOMBSTONE).astype(np.int32), np.where(valid, d, np.float32(np.inf)).astype(np.float32), c

    @property
    def read_ids(self) -> np.ndarray:
        return self._cached("read")[0]

    @property
    def read_dists(self) -> np.ndarray:
        return self._cached("read")[1]

    @property
    def read_count(self) -> np.ndarray:
        return self._cached("read")[2]

    @property
    def write_ids(self) -> np.ndarray:
        return self._cached("write")[0]

    @property
    def write_dists(self) -> np.ndarray:
        return self._cached("write")[1]

    @property
    def write_count(self) -> np.ndarray:
        return self._cached("write")[2]

    def snapshot(self):
        """(read_ids, read_dists, read_count) host copies (read-only)."""
        return self._cached("read")

    def pool(self, v: int) -> DoubleBufferPool:
        ri, rd, _ = self.snapshot()
        wi, wd, wc = self._cached("write")
        return DoubleBufferPool(owner=v, read_ids=ri[v], read_dists=rd[v], write_ids=wi[v],
                                write_dists=wd[v], write_count=int(wc[v]))

    def clear_and_swap(self) -> None:
        self.pools.swap()

    def fixed_degree(self) -> np.ndarray:
        """The fixed-degree int32 [N, R] adjacency: rows ascending by (dist, id), -1 padded."""
        return self.pools.sorted_rows().cpu().numpy()

    @classmethod
    def from_arrays(cls, data, params: BuildParams, read_ids, read_dists, read_count,
                    pair_order: str = "disordered", device=None) -> "BuildState":
        """A state with caller-set read pools (the reference tests' _manual_state)."""
        return cls(params=params, data=data, read_ids=read_ids, read_dists=read_dists, read_count=read_count,
                   pair_order=pair_order, device=device)


def init_neighbors(dataset: Dataset, params: BuildParams, pair_order: PairOrder = "disordered",
                   *, device=None, metric: str = "l2", msg_capacity: int | None = None) -> BuildState:
    """S distinct random neighbours != owner per vertex (builder.py:221-257).  The
    reference validates the dataset (finiteness included) before the parameters; so does
    this, with the finiteness scan on the device."""
    dataset.validate_shape()
    n = dataset.num_points
    if pair_order not in _ORDER_CODES:
        raise ParamError(f"pair_order must be one of {sorted(_ORDER_CODES)}")
    check_metric(metric)
    dev = _device(device)
    with torch.cuda.device(dev):
        data_dev = upload(dataset.data, dev)
        check_finite_device(data_dev, dataset.dim)
        validate_params(params, n)
        if params.S > n - 1:
            raise ParamError("S <= N-1")
        if metric == "ip":
            normalize_rows_(data_dev, dataset.dim)
    pools = _DevicePools(data_dev, dataset.dim, params.R, msg_capacity=msg_capacity)
    fail = pools.init(params.S, params.seed)
    if int(fail.item()):  # pragma: no cover - probability ~ exp(-64)
        raise RuntimeError("initial neighbor sampling did not converge")
    return BuildState(dataset, params, pools, pair_order)


def _stats_row(state: BuildState) -> torch.Tensor:
    st = state.pools.scratch_stats
    st.zero_()
    return st


def update_round(state: BuildState) -> RoundStats:
    """One pair-propagation round (builder.py:283-312)."""
    st = _stats_row(state)
    state.pools.update(state.params.seed, STREAM_ROUND_BASE + state.round_index,
                       _ORDER_CODES[state.pair_order], st)
    state.round_index += 1
    stats = RoundStats.from_counters("update", st.cpu().numpy())
    _accumulate(state.totals, stats)
    return stats


def reverse_edge_sampling(state: BuildState) -> RoundStats:
    """Reverse edges for each vertex's ceil(rho*k) closest neighbours, then the
    self merge; clear and swap (builder.py:315-339)."""
    st = _stats_row(state)
    state.pools.reverse(state.params.rho, st)
    stats = RoundStats.from_counters("reverse", st.cpu().numpy())
    _accumulate(state.totals, stats)
    return stats


def _finalize_device(pools: _DevicePools):
    """Device CSR: (offsets int64[n+1], nbrs int32[<= n*cap], bad flag)."""
    offsets = torch.empty(pools.rows + 1, dtype=torch.int64, device=pools.dev)
    nbrs = torch.empty(max(pools.rows * pools.cap, 1), dtype=torch.int32, device=pools.dev)
    bad = torch.zeros(1, dtype=torch.int64, device=pools.dev)
    pools.finalize(offsets, nbrs, bad)
    return offsets, nbrs, bad


_BAD_MESSAGES = ((1, "neighbor id out of range"), (2, "self-loop present"),
                 (4, "duplicate neighbor id within one vertex"))


def _to_host_pinned(t: torch.Tensor) -> np.ndarray:
    """Device -> page-locked host memory (torch's caching host allocator), returned as a
    numpy view that keeps the block alive.  A pageable .cpu() of the 84 MB C2 graph costs
    ~40 ms (staging + first-touch page faults of a fresh array); this copy ~2 ms."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h


def _graph_from_device(pools: _DevicePools, offsets, nbrs, bad) -> Graph:
    off_h = _to_host_pinned(offsets)
    flags_h = _to_host_pinned(bad)
    torch.cuda.current_stream(pools.dev).synchronize()
    off = off_h.numpy()
    total = int(off[-1])
    ids_h = _to_host_pinned(nbrs[:total])
    torch.cuda.current_stream(pools.dev).synchronize()
    ids = ids_h.numpy()
    flags = int(flags_h[0])
    for bit, msg in _BAD_MESSAGES:
        if flags & bit:
            raise ParamError(msg)
    return Graph(num_vertices=pools.rows, offsets=off, neighbor_ids=ids, max_degree_bound=pools.cap)


def finalize_graph(state: BuildState) -> Graph:
    """Each read buffer's entries ascending by (dist, id), as CSR (builder.py:342-362).
    The CSR invariants of Graph.validate are checked on the device in the same pass."""
    return _graph_from_device(state.pools, *_finalize_device(state.pools))


def num_rounds(params: BuildParams) -> int:
    return params.T1 * params.T2 + (params.T1 - 1)


def run_rounds(state: BuildState, stats_rows: torch.Tensor | None = None) -> list[str]:
    """All T1 x (T2 update [+ reverse]) rounds, asynchronously; per-round counters
    land in ``stats_rows`` [rounds, NSTATS] (zeroed by the caller).  Returns kinds."""
    p = state.params
    kinds = []
    order = _ORDER_CODES[state.pair_order]
    i = 0
    for t1 in range(1, p.T1 + 1):
        for _ in range(p.T2):
            row = stats_rows[i] if stats_rows is not None else state.pools.scratch_stats
            state.pools.update(p.seed, STREAM_ROUND_BASE + state.round_index, order, row)
            state.round_index += 1
            kinds.append("update")
            i += 1
        if t1 != p.T1:
            row = stats_rows[i] if stats_rows is not None else state.pools.scratch_stats
            state.pools.reverse(p.rho, row)
            kinds.append("reverse")
            i += 1
    return kinds


MSG_PER_ROW = 48  # optimistic message capacity per owned row (see build())


def optimistic_msg_capacity(rows: int, cap: int) -> int:
    """Message slots a build starts with: MSG_PER_ROW per row instead of the worst case
    rows * R (an update round emits one redirect per tombstoned entry, <= sum(k); a reverse
    round ceil(rho k) per row).  At C2 the largest round needs ~20 per row; the worst case
    would cost 60 B x R per row of workspace (5.8 GB at 1M x 96)."""
    return int(min(max(rows * cap, 1), max(MSG_PER_ROW * rows, 1 << 16)))


def build(dataset: Dataset, params: BuildParams, pair_order: PairOrder = "disordered",
          report_stats: list | None = None, *, device=None, metric: str = "l2") -> Graph:
    """Full build (builder.py:365-390): init, T1 x T2 pair rounds with reverse-edge
    sampling between outer iterations, then graph emission.  One host sync for the
    init-failure flag, one at the end; every round is a single asynchronous call.
    ``metric="ip"`` builds over L2-normalised rows (inner product; not in the reference).

    The workspace starts with an optimistic message capacity; a round that outgrows it
    loses messages, which the device counts (GRNND_ST_LOST) -- the stats rows are read
    before the graph is emitted and such a build is redone once at the worst-case
    capacity, so a result is never built on dropped messages."""
    params = effective_params(params, dataset.num_points)
    for attempt in range(2):
        cap_msgs = optimistic_msg_capacity(dataset.num_points, params.R) if attempt == 0 else None
        state = init_neighbors(dataset, params, pair_order, device=device, metric=metric, msg_capacity=cap_msgs)
        rows = torch.zeros((num_rounds(params), _lib.NSTATS), dtype=torch.int64, device=state.pools.dev)
        kinds = run_rounds(state, rows)
        host_rows = rows.cpu().numpy()
        if attempt == 0 and host_rows[:, _lib.ST_LOST].any():
            del state, rows
            continue
        break
    graph = finalize_graph(state)
    for kind, c in zip(kinds, host_rows):
        s = RoundStats.from_counters(kind, c)
        _accumulate(state.totals, s)
        if report_stats is not None:
            report_stats.append(s)
    return graph


class DeviceBuild:
    """A reusable build engine over device-resident vectors (the bench's timed step and
    the building block of the sharded multi-GPU build).  ``run()`` = init + all rounds +
    finalize, entirely asynchronous; results stay in HBM."""

    def __init__(self, data_dev: torch.Tensor, dim: int, params: BuildParams,
                 pair_order: PairOrder = "disordered", metric: str = "l2", msg_capacity: int | None = None):
        self.params = effective_params(params, int(data_dev.shape[0]))
        validate_params(self.params, int(data_dev.shape[0]))
        check_metric(metric)
        self.order = _ORDER_CODES[pair_order]
        self.metric = metric
        self.raw = data_dev
        self.dim = dim
        # IP: every run normalises a copy of the raw vectors (part of the timed build)
        work = torch.empty_like(data_dev) if metric == "ip" else data_dev
        # optimistic message capacity (build()); round_stats() raises if a round outgrew it
        mc = msg_capacity if msg_capacity is not None else optimistic_msg_capacity(int(data_dev.shape[0]),
                                                                                    self.params.R)
        self.pools = _DevicePools(work, dim, self.params.R, msg_capacity=mc)
        self.rounds = num_rounds(self.params)
        self.stats = torch.zeros((self.rounds, _lib.NSTATS), dtype=torch.int64, device=self.pools.dev)
        self.kinds: list[str] = []

    def run(self, phase_events: list | None = None):
        """One full build.  phase_events, if given, receives one (start, emitted, applied)
        CUDA-event triple per update round."""
        p, pools = self.params, self.pools
        self.stats.zero_()
        self.kinds = []
        if self.metric == "ip":
            pools.data.copy_(self.raw)
            normalize_rows_(pools.data, self.dim)
        pools.compute_norms()
        fail = pools.init(p.S, p.seed)
        i = 0
        round_index = 0
        for t1 in range(1, p.T1 + 1):
            for _ in range(p.T2):
                ev = None
                if phase_events is not None:
                    ev = tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
                    phase_events.append(ev)
                pools.update_split(p.seed, STREAM_ROUND_BASE + round_index, self.order, self.stats[i], ev)
                round_index += 1
                self.kinds.append("update")
                i += 1
            if t1 != p.T1:
                pools.reverse(p.rho, self.stats[i])
                self.kinds.append("reverse")
                i += 1
        offsets, nbrs, bad = _finalize_device(pools)
        return offsets, nbrs, bad, fail

    def search_data(self) -> torch.Tensor:
        """The vectors the graph was built over (normalised rows for IP)."""
        return self.pools.data

    def round_stats(self) -> list[RoundStats]:
        rows = self.stats.cpu().numpy()
        return [RoundStats.from_counters(k, c) for k, c in zip(self.kinds, rows)]


def build_fixed_degree(dataset: Dataset, params: BuildParams, pair_order: PairOrder = "disordered",
                       *, device=None, metric: str = "l2") -> np.ndarray:
    """Same build, returned as the fixed-degree int32 [N, R] array (rows ascending by
    (dist, id), -1 padded) -- the layout GPU graph builders hand to search kernels."""
    params = effective_params(params, dataset.num_points)
    state = init_neighbors(dataset, params, pair_order, device=device, metric=metric)
    run_rounds(state)
    return state.fixed_degree()


def validate_state(state: BuildState, tol: float = 1e-4) -> None:
    """Round-boundary invariants (builder.py:393-422) on a host snapshot."""
    n, cap = state.num_vertices, state.capacity
    ids, dists, counts = state.snapshot()
    assert counts.min() >= 0 and counts.max() <= cap, "read count out of range"
    # the device write buffer is cleared logically (count 0; slots beyond a row's count are
    # never read), so "empty" is exactly a zero count (the reference's TOMB fill, :402-404)
    assert np.all(state.write_count == 0), "write buffers not empty at boundary"
    valid = np.arange(cap)[None, :] < counts[:, None]
    assert np.all(ids[valid] >= 0), "tombstone inside the packed prefix"
    assert np.all(ids[~valid] == TOMBSTONE), "valid id beyond the packed prefix"
    owners = np.broadcast_to(np.arange(n, dtype=np.int32)[:, None], (n, cap))
    assert not np.any(ids[valid] == owners[valid]), "self-loop in a pool"
    big = np.int32(2**31 - 1)
    sids = np.sort(np.where(valid, ids, big), axis=1)
    assert not np.any((sids[:, 1:] == sids[:, :-1]) & (sids[:, 1:] != big)), "duplicate id within one pool"
    if np.any(valid):
        rows = np.repeat(np.arange(n), counts)
        diff = state.data[rows].astype(np.float64) - state.data[ids[valid]].astype(np.float64)
        true_sq = (diff * diff).sum(axis=1)
        stored = dists[valid].astype(np.float64)
        err = np.abs(stored - true_sq) / np.maximum(true_sq, 1e-30)
        exact_zero = (true_sq == 0) & (stored == 0)
        assert np.all(exact_zero | (err <= tol)), "stored distance drifted from truth"
