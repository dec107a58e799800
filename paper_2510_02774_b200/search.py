"""Greedy beam search, brute-force ground truth and recall, on the device.

Twin of /root/reference/pkg/src/grnnd/search.py: the same ``SearchParams``
(:26-45), entry selection (:48-56), ``greedy_search`` (:72-87),
``search_batch`` (:90-115), ``brute_force_knn`` / ``brute_force_knn_batch``
(:118-142), ``recall_at_k`` / ``mean_recall`` (:145-159), with the same
argument meaning, padding and exceptions.  The work runs in
libgrnnd_b200.so (``csrc/search.cu``): the results are bit-identical to the
reference's numba kernels (exact sequential fp32 distances, (dist, id) order).

``search_device`` / ``brute_force_device`` take device tensors (the graph as
it leaves ``finalize`` and the vectors already in HBM), which is how the bench
scores recall without a host round trip.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .builder import _device, _stream, padded_ld, upload
from .core import Dataset, Graph
from .errors import DimensionMismatch, EmptyGraph, LengthMismatch, ParamError

MASK64 = (1 << 64) - 1
_STREAM_ENTRY = 0x5EED  # search.py:23
_VISITED_BUDGET = 1 << 31  # bytes of per-query visited bitmaps resident at once


@dataclass(frozen=True)
class SearchParams:
    """L: candidate list capacity (beam width), k: result count; entry: a fixed start
    vertex (default 0) or None for a seeded random entry per query (search.py:26-45)."""

    L: int
    k: int
    entry: int | None = 0
    seed: int = 0

    def validate(self, n: int) -> None:
        if self.k < 1:
            raise ParamError("k >= 1")
        if self.L < self.k:
            raise ParamError("L >= k")
        if self.entry is not None and not (0 <= self.entry < n):
            raise ParamError("entry vertex out of range")


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on uint64 arrays (rng.py:25-31; wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def hash4_vec(seed: int, stream: int, v: np.ndarray, i: int) -> np.ndarray:
    """rng.hash4_vec (rng.py:44-57) on the host (entry selection only)."""
    h = _mix64(np.full(v.shape, seed & MASK64, dtype=np.uint64))
    h = _mix64(h ^ np.uint64(stream & MASK64))
    h = _mix64(h ^ v.astype(np.uint64))
    return _mix64(h ^ np.uint64(i & MASK64))


def _entries_for(sp: SearchParams, n: int, nq: int) -> np.ndarray:
    """search.py:48-56"""
    if sp.entry is not None:
        return np.full(nq, sp.entry, dtype=np.int64)
    qi = np.arange(nq, dtype=np.uint64)
    return (hash4_vec(sp.seed, _STREAM_ENTRY, qi, 0) % np.uint64(n)).astype(np.int64)


def _check_query(dataset: Dataset, q) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float32)
    qdim = q.shape[0] if q.ndim == 1 else q.shape[1]
    if qdim != dataset.dim:
        raise DimensionMismatch(f"query dimension {qdim} does not match dataset dimension {dataset.dim}")
    return q


def _check_graph(graph: Graph, dataset: Dataset) -> None:
    if graph.num_vertices == 0:
        raise EmptyGraph("cannot search an empty graph")
    if graph.num_vertices != dataset.num_points:
        raise DimensionMismatch("graph and dataset disagree on the number of points")


# ----------------------------------------------------------------------------------------
# device-resident entry points
# ----------------------------------------------------------------------------------------
def search_device(offsets: torch.Tensor, nbrs: torch.Tensor, data_dev: torch.Tensor, dim: int,
                  queries_dev: torch.Tensor, L: int, k: int, entries: torch.Tensor,
                  with_dists: bool = False):
    """Greedy search of device queries [nq, ld] over a device CSR graph.  Returns device
    ids int32 [nq, k] (-1 padded), and with ``with_dists`` also fp32 dists and counts."""
    dev = data_dev.device
    n, ld = int(data_dev.shape[0]), int(data_dev.shape[1])
    nq = int(queries_dev.shape[0])
    ids = torch.full((nq, k), -1, dtype=torch.int32, device=dev)
    dists = torch.full((nq, k), float("inf"), dtype=torch.float32, device=dev)
    cnt = torch.zeros(nq, dtype=torch.int64, device=dev)
    if nq == 0:
        return (ids, dists, cnt) if with_dists else ids
    per_q = int(_lib.lib.grnnd_search_visited_bytes(n, 1))
    batch = max(1, min(nq, _VISITED_BUDGET // max(per_q, 1)))
    vis = torch.empty(int(_lib.lib.grnnd_search_visited_bytes(n, batch)), dtype=torch.uint8, device=dev)
    st = _stream(dev)
    for q0 in range(0, nq, batch):
        q1 = min(nq, q0 + batch)
        _lib.call("grnnd_greedy_search", offsets.data_ptr(), nbrs.data_ptr(), n, data_dev.data_ptr(), dim, ld,
                  queries_dev[q0:q1].data_ptr(), q1 - q0, int(L), int(k), entries[q0:q1].data_ptr(),
                  ids[q0:q1].data_ptr(), dists[q0:q1].data_ptr(), cnt[q0:q1].data_ptr(), vis.data_ptr(),
                  vis.numel(), st)
    return (ids, dists, cnt) if with_dists else ids


def brute_force_device(data_dev: torch.Tensor, dim: int, queries_dev: torch.Tensor, k: int,
                       with_dists: bool = False):
    """Exact k nearest ids (ties by ascending id) of device queries [nq, ld]."""
    dev = data_dev.device
    n, ld = int(data_dev.shape[0]), int(data_dev.shape[1])
    nq = int(queries_dev.shape[0])
    ids = torch.full((nq, k), -1, dtype=torch.int32, device=dev)
    dists = torch.full((nq, k), float("inf"), dtype=torch.float32, device=dev)
    if nq:
        ws = torch.empty(max(int(_lib.lib.grnnd_brute_force_workspace_bytes(n, nq, k)), 1), dtype=torch.uint8,
                         device=dev)
        _lib.call("grnnd_brute_force", data_dev.data_ptr(), n, dim, ld, queries_dev.data_ptr(), nq, int(k),
                  ids.data_ptr(), dists.data_ptr(), ws.data_ptr(), ws.numel(), _stream(dev))
    return (ids, dists) if with_dists else ids


def _upload_queries(q: np.ndarray, dev) -> torch.Tensor:
    if q.ndim == 1:
        q = q.reshape(1, -1)
    return upload(q, dev)


def _upload_graph(graph: Graph, dev):
    off = torch.from_numpy(np.ascontiguousarray(graph.offsets, dtype=np.int64)).to(dev)
    nb = graph.neighbor_ids
    nbt = torch.from_numpy(np.ascontiguousarray(nb if len(nb) else np.zeros(1, np.int32), dtype=np.int32)).to(dev)
    return off, nbt


# ----------------------------------------------------------------------------------------
# the reference's host API
# ----------------------------------------------------------------------------------------
def greedy_search(graph: Graph, dataset: Dataset, query, sp: SearchParams, *, device=None) -> np.ndarray:
    """The k nearest visited ids for one query, ascending by distance (search.py:72-87)."""
    _check_graph(graph, dataset)
    sp.validate(graph.num_vertices)
    q = _check_query(dataset, np.asarray(query))
    entry = sp.entry
    if entry is None:
        entry = int(_entries_for(sp, graph.num_vertices, 1)[0])
    dev = _device(device)
    off, nb = _upload_graph(graph, dev)
    ids, _, cnt = search_device(off, nb, upload(dataset.data, dev), dataset.dim, _upload_queries(q, dev),
                                sp.L, sp.k, torch.tensor([entry], dtype=torch.int64, device=dev), with_dists=True)
    c = int(cnt[0].item())
    return ids[0, :c].cpu().numpy()


def search_batch(graph: Graph, dataset: Dataset, queries, sp: SearchParams, threads: int = 1,
                 *, device=None) -> tuple[np.ndarray, float]:
    """Run a query batch; returns (ids [nq, k] padded with -1, seconds of the device search).
    ``threads`` is accepted for signature compatibility (search.py:90-115)."""
    _check_graph(graph, dataset)
    sp.validate(graph.num_vertices)
    q = _check_query(dataset, np.asarray(queries))
    if q.ndim == 1:
        q = q.reshape(1, -1)
    entries = _entries_for(sp, graph.num_vertices, q.shape[0])
    dev = _device(device)
    with torch.cuda.device(dev):
        off, nb = _upload_graph(graph, dev)
        data_dev = upload(dataset.data, dev)
        qd = _upload_queries(q, dev)
        ent = torch.from_numpy(entries).to(dev)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        ids = search_device(off, nb, data_dev, dataset.dim, qd, sp.L, sp.k, ent)
        torch.cuda.synchronize(dev)
        elapsed = time.perf_counter() - t0
    return ids.cpu().numpy(), elapsed


def brute_force_knn(dataset: Dataset, query, k: int, *, device=None) -> np.ndarray:
    """Exact k nearest ids for one query, ties broken by ascending id (search.py:118-127)."""
    if k < 1 or k > dataset.num_points:
        raise ParamError("k must satisfy 1 <= k <= N")
    q = _check_query(dataset, np.asarray(query))
    out = brute_force_knn_batch(dataset, q.reshape(1, -1) if q.ndim == 1 else q, k, device=device)
    return out[0] if out.shape[0] == 1 and np.asarray(query).ndim == 1 else out


def brute_force_knn_batch(dataset: Dataset, queries, k: int, threads: int = 1, *, device=None) -> np.ndarray:
    """Ground-truth ids for a query batch (search.py:130-142)."""
    if k < 1 or k > dataset.num_points:
        raise ParamError("k must satisfy 1 <= k <= N")
    q = _check_query(dataset, np.asarray(queries))
    if q.ndim == 1:
        q = q.reshape(1, -1)
    dev = _device(device)
    with torch.cuda.device(dev):
        ids = brute_force_device(upload(dataset.data, dev), dataset.dim, _upload_queries(q, dev), k)
        return ids.cpu().numpy()


def recall_at_k(retrieved, truth) -> float:
    """|retrieved intersect truth| / k for two duplicate-free id lists (search.py:145-152)."""
    r = np.asarray(retrieved).ravel()
    t = np.asarray(truth).ravel()
    if r.shape[0] != t.shape[0]:
        raise LengthMismatch(f"length mismatch: {r.shape[0]} vs {t.shape[0]}")
    k = r.shape[0]
    return len(set(r.tolist()) & set(t.tolist())) / k


def mean_recall(retrieved: np.ndarray, truth: np.ndarray) -> float:
    """Average recall_at_k over the rows of two (nq, k) id matrices (search.py:155-159)."""
    return float(np.mean([recall_at_k(retrieved[i], truth[i]) for i in range(retrieved.shape[0])]))


def knn_graph_recall(graph: Graph, truth: np.ndarray, sample: np.ndarray) -> float:
    """k-NN-graph recall (not in the reference): the fraction of each sampled
    vertex's exact nearest neighbours ``truth[i]`` (itself excluded) found among its
    out-neighbours."""
    hits = 0
    for i, v in enumerate(np.asarray(sample)):
        nb = set(graph.neighbor_ids[graph.offsets[v]:graph.offsets[v + 1]].tolist())
        hits += len(nb & set(int(x) for x in truth[i]))
    return hits / float(truth.shape[0] * truth.shape[1])


__all__ = [
    "SearchParams", "brute_force_device", "brute_force_knn", "brute_force_knn_batch", "greedy_search",
    "knn_graph_recall", "mean_recall", "padded_ld", "recall_at_k", "search_batch", "search_device",
]
