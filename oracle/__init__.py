"""ctypes wrapper around the CPU oracle (grnnd_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs import this module.
The product package ``paper_2510_02774_b200`` never does.

The oracle restates the reference kernels of
/root/reference/pkg/src/grnnd/_numba_kernels.py and the round structure of
builder.py (see the per-function citations in grnnd_oracle.c).  Parity with
the reference is pinned by tests/test_oracle_golden.py against fixtures the
reference itself produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

STATS_FIELDS = (
    "kind", "messages", "redirects", "survivors", "reverse_attempts",
    "inserted", "duplicate", "replaced", "rejected",
)

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u64 = C.c_uint64
_i64 = C.c_int64
_i32 = C.c_int32


def build_oracle() -> Path:
    """Compile liboracle.so with the committed Makefile (needs gcc)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build_oracle()
    L = C.CDLL(str(_LIB_PATH))
    sig = {
        "orc_mix64": (_u64, [_u64]),
        "orc_hash4": (_u64, [_u64, _u64, _u64, _u64]),
        "orc_sqdist": (C.c_float, [_f32p, _f32p, _i32]),
        "orc_sqdist_batch": (None, [_f32p, _f32p, _i64, _i32, _f32p]),
        "orc_set_threads": (None, [_i32]),
        "orc_max_threads": (_i32, []),
        "orc_fill_perm": (None, [_i32p, _i32, _u64, _u64, _u64, _i32p, _f32p, _i32]),
        "orc_sample_initial": (_i32, [_i64, _i32, _u64, _i32p]),
        "orc_init_dists": (None, [_f32p, _i64, _i32, _i32p, _i32, _f32p]),
        "orc_gen_update_messages": (
            None,
            [_f32p, _i64, _i32, _i32p, _f32p, _i32p, _i32, _u64, _u64, _i32, _i32p, _i32p, _f32p, _i32p],
        ),
        "orc_gen_update_messages_lo": (
            None,
            [_f32p, _i64, _i64, _i32, _i32p, _f32p, _i32p, _i32, _u64, _u64, _i32, _i32p, _i32p, _f32p, _i32p],
        ),
        "orc_gen_reverse_messages_lo": (
            None, [_i32p, _f32p, _i32p, _i64, _i64, _i32, C.c_double, _i32p, _i32p, _f32p, _i32p]
        ),
        "orc_reverse_count": (_i32, [C.c_double, _i32]),
        "orc_gen_reverse_messages": (
            None, [_i32p, _f32p, _i32p, _i64, _i32, C.c_double, _i32p, _i32p, _f32p, _i32p]
        ),
        "orc_gen_merge_messages": (None, [_i32p, _f32p, _i32p, _i64, _i32, _i32p, _i32p, _f32p, _i32p]),
        "orc_build_flat": (
            _i64, [_i32p, _i32p, _f32p, _i32p, _i64, _i32, _i64p, _i32p, _i32p, _f32p, _i32p]
        ),
        "orc_group_by_target": (None, [_i32p, _i64, _i64, _i64p, _i64p]),
        "orc_apply_grouped": (
            None, [_i32p, _f32p, _i32p, _i64, _i32, _i32p, _f32p, _i64p, _i64p, _i64p]
        ),
        "orc_finalize": (None, [_i32p, _f32p, _i32p, _i64, _i32, _i64p, _i32p]),
        "orc_state_new": (C.c_void_p, [_f32p, _i64, _i32, _i32, _i32, _u64, C.POINTER(_i32)]),
        "orc_state_free": (None, [C.c_void_p]),
        "orc_state_update_round": (None, [C.c_void_p, _u64, _u64, _i32, _i64p]),
        "orc_state_reverse_round": (None, [C.c_void_p, C.c_double, _i64p]),
        "orc_state_export": (None, [C.c_void_p, _i32p, _f32p, _i32p]),
        "orc_state_import": (None, [C.c_void_p, _i32p, _f32p, _i32p]),
        "orc_state_finalize": (None, [C.c_void_p, _i64p, _i32p]),
        "orc_build": (
            _i32,
            [_f32p, _i64, _i32, _i32, _i32, _i32, _i32, C.c_double, _u64, _i32, _i64p, _i32p, C.c_void_p],
        ),
        "orc_normalize_rows": (None, [_f32p, _i64, _i32]),
        "orc_brute_force": (None, [_f32p, _i64, _i32, _f32p, _i64, _i32, _i32p]),
        "orc_greedy_search": (
            None, [_i64p, _i32p, _f32p, _i64, _i32, _f32p, _i64, _i32, _i32, _i64p, _i32p]
        ),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32a(a):
    return np.ascontiguousarray(a, dtype=np.int32)


M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    return int(lib().orc_mix64(int(x) & M64))


def hash4(seed: int, stream: int, v: int, i: int) -> int:
    return int(lib().orc_hash4(seed & M64, stream & M64, v & M64, i & M64))


def sqdist(a, b) -> np.float32:
    a, b = _f32(a), _f32(b)
    return np.float32(lib().orc_sqdist(a, b, a.shape[0]))


def sqdist_batch(a, b) -> np.ndarray:
    a, b = _f32(a), _f32(b)
    out = np.empty(a.shape[0], np.float32)
    lib().orc_sqdist_batch(a, b, a.shape[0], a.shape[1], out)
    return out


def fisher_yates_perm(k: int, seed: int, stream: int, v: int) -> np.ndarray:
    perm = np.empty(max(k, 1), np.int32)
    dummy_i = np.zeros(max(k, 1), np.int32)
    dummy_d = np.zeros(max(k, 1), np.float32)
    lib().orc_fill_perm(perm, k, seed & M64, stream & M64, v, dummy_i, dummy_d, 0)
    return perm[:k]


def sample_initial(n: int, count: int, seed: int) -> tuple[np.ndarray, int]:
    out = np.full((n, count), -1, np.int32)
    fail = lib().orc_sample_initial(n, count, seed & M64, out)
    return out, int(fail)


def init_dists(data, ids) -> np.ndarray:
    data, ids = _f32(data), _i32a(ids)
    out = np.empty(ids.shape, np.float32)
    lib().orc_init_dists(data, data.shape[0], data.shape[1], ids, ids.shape[1], out)
    return out


def gen_update_messages(data, read_ids, read_dists, read_count, seed, stream, order_code):
    """Returns (msg_tgt, msg_id, msg_dist, msg_cnt); mutates ``read_ids`` in place."""
    data = _f32(data)
    n, cap = read_ids.shape
    assert read_ids.dtype == np.int32 and read_ids.flags.c_contiguous
    mt = np.full(n * cap, -1, np.int32)
    mi = np.full(n * cap, -1, np.int32)
    md = np.zeros(n * cap, np.float32)
    mc = np.zeros(n, np.int32)
    lib().orc_gen_update_messages(
        data, n, data.shape[1], read_ids, _f32(read_dists), _i32a(read_count), cap,
        seed & M64, stream & M64, order_code, mt, mi, md, mc,
    )
    return mt, mi, md, mc


def gen_update_messages_lo(data, lo, read_ids, read_dists, read_count, seed, stream, order_code):
    """gen_update_messages on owned rows [lo, lo + n): returns slices; mutates read_ids."""
    data = _f32(data)
    n, cap = read_ids.shape
    mt = np.full(n * cap, -1, np.int32)
    mi = np.full(n * cap, -1, np.int32)
    md = np.zeros(n * cap, np.float32)
    mc = np.zeros(n, np.int32)
    lib().orc_gen_update_messages_lo(
        data, lo, n, data.shape[1], read_ids, _f32(read_dists), _i32a(read_count), cap,
        seed & M64, stream & M64, order_code, mt, mi, md, mc,
    )
    return mt, mi, md, mc


def gen_reverse_messages_lo(lo, read_ids, read_dists, read_count, rho):
    n, cap = read_ids.shape
    mt = np.full(n * cap, -1, np.int32)
    mi = np.full(n * cap, -1, np.int32)
    md = np.zeros(n * cap, np.float32)
    mc = np.zeros(n, np.int32)
    lib().orc_gen_reverse_messages_lo(
        _i32a(read_ids), _f32(read_dists), _i32a(read_count), lo, n, cap, float(rho), mt, mi, md, mc
    )
    return mt, mi, md, mc


def gen_reverse_messages(read_ids, read_dists, read_count, rho):
    n, cap = read_ids.shape
    mt = np.full(n * cap, -1, np.int32)
    mi = np.full(n * cap, -1, np.int32)
    md = np.zeros(n * cap, np.float32)
    mc = np.zeros(n, np.int32)
    lib().orc_gen_reverse_messages(
        _i32a(read_ids), _f32(read_dists), _i32a(read_count), n, cap, float(rho), mt, mi, md, mc
    )
    return mt, mi, md, mc


def gen_merge_messages(read_ids, read_dists, read_count):
    n, cap = read_ids.shape
    mt = np.full(n * cap, -1, np.int32)
    mi = np.full(n * cap, -1, np.int32)
    md = np.zeros(n * cap, np.float32)
    mc = np.zeros(n, np.int32)
    lib().orc_gen_merge_messages(_i32a(read_ids), _f32(read_dists), _i32a(read_count), n, cap, mt, mi, md, mc)
    return mt, mi, md, mc


def build_flat(mt, mi, md, mc, cap):
    n = mc.shape[0]
    total = int(mc.astype(np.int64).sum())
    offs = np.zeros(n + 1, np.int64)
    ft = np.empty(max(total, 1), np.int32)
    fi = np.empty(max(total, 1), np.int32)
    fd = np.empty(max(total, 1), np.float32)
    fs = np.empty(max(total, 1), np.int32)
    lib().orc_build_flat(_i32a(mt), _i32a(mi), _f32(md), _i32a(mc), n, cap, offs, ft, fi, fd, fs)
    return ft[:total], fi[:total], fd[:total], fs[:total]


def group_by_target(flat_tgt, n):
    flat_tgt = _i32a(flat_tgt)
    m = flat_tgt.shape[0]
    order = np.empty(max(m, 1), np.int64)
    starts = np.zeros(n + 1, np.int64)
    lib().orc_group_by_target(flat_tgt if m else np.zeros(1, np.int32), m, n, order, starts)
    return order[:m], starts


def apply_grouped_messages(write_ids, write_dists, write_count, flat_id, flat_dist, order, starts):
    n, cap = write_ids.shape
    out4 = np.zeros(4, np.int64)
    fi = _i32a(flat_id) if len(flat_id) else np.zeros(1, np.int32)
    fd = _f32(flat_dist) if len(flat_dist) else np.zeros(1, np.float32)
    od = np.ascontiguousarray(order, np.int64) if len(order) else np.zeros(1, np.int64)
    lib().orc_apply_grouped(
        write_ids, write_dists, write_count, n, cap, fi, fd, od, np.ascontiguousarray(starts, np.int64), out4
    )
    return tuple(int(x) for x in out4)


def finalize(read_ids, read_dists, read_count):
    n, cap = read_ids.shape
    offsets = np.zeros(n + 1, np.int64)
    total = int(np.asarray(read_count, np.int64).sum())
    nbrs = np.empty(max(total, 1), np.int32)
    lib().orc_finalize(_i32a(read_ids), _f32(read_dists), _i32a(read_count), n, cap, offsets, nbrs)
    return offsets, nbrs[:total]


def num_rounds(T1: int, T2: int) -> int:
    return T1 * T2 + (T1 - 1)


def build(data, S, R, T1, T2, rho, seed, order_code=0, with_stats=False):
    """Full reference build (params must already be clamped/validated).

    Returns (offsets int64[N+1], neighbor_ids int32[M]) and, if requested,
    an int64 [rounds, 9] stats matrix (columns: STATS_FIELDS).
    """
    data = _f32(data)
    n, dim = data.shape
    offsets = np.zeros(n + 1, np.int64)
    nbrs = np.empty(max(n * R, 1), np.int32)
    stats = np.zeros((num_rounds(T1, T2), len(STATS_FIELDS)), np.int64) if with_stats else None
    rc = lib().orc_build(
        data, n, dim, S, R, T1, T2, float(rho), seed & M64, order_code, offsets, nbrs,
        stats.ctypes.data_as(C.c_void_p) if stats is not None else None,
    )
    if rc == 1:
        raise RuntimeError("initial neighbor sampling did not converge")
    if rc != 0:
        raise MemoryError("oracle build: allocation failed")
    out = (offsets, nbrs[: offsets[-1]].copy())
    return out + (stats,) if with_stats else out


class State:
    """Oracle build state driven round by round (mirrors builder.BuildState)."""

    def __init__(self, data, S, R, seed):
        self.data = _f32(data)
        self.n, self.dim = self.data.shape
        self.R = R
        fail = _i32(0)
        self._p = lib().orc_state_new(self.data, self.n, self.dim, S, R, seed & M64, C.byref(fail))
        if not self._p:
            raise MemoryError("oracle state allocation failed")
        if fail.value:
            raise RuntimeError("initial neighbor sampling did not converge")

    def update_round(self, seed, stream, order_code=0):
        st = np.zeros(len(STATS_FIELDS), np.int64)
        lib().orc_state_update_round(self._p, seed & M64, stream & M64, order_code, st)
        return st

    def reverse_round(self, rho):
        st = np.zeros(len(STATS_FIELDS), np.int64)
        lib().orc_state_reverse_round(self._p, float(rho), st)
        return st

    def export(self):
        ids = np.empty((self.n, self.R), np.int32)
        d = np.empty((self.n, self.R), np.float32)
        c = np.empty(self.n, np.int32)
        lib().orc_state_export(self._p, ids, d, c)
        return ids, d, c

    def load(self, ids, dists, counts):
        lib().orc_state_import(self._p, _i32a(ids), _f32(dists), _i32a(counts))

    def finalize(self):
        _, _, c = self.export()
        offsets = np.zeros(self.n + 1, np.int64)
        nbrs = np.empty(max(int(c.astype(np.int64).sum()), 1), np.int32)
        lib().orc_state_finalize(self._p, offsets, nbrs)
        return offsets, nbrs[: offsets[-1]]

    def __del__(self):
        p = getattr(self, "_p", None)
        if p:
            lib().orc_state_free(p)
            self._p = None


def normalize_rows(data) -> np.ndarray:
    """IP metric: a copy of ``data`` with unit-norm rows (orc_normalize_rows)."""
    x = np.array(data, dtype=np.float32, order="C", copy=True)
    lib().orc_normalize_rows(x, x.shape[0], x.shape[1])
    return x


def brute_force_knn(data, queries, k):
    data, queries = _f32(data), _f32(queries)
    out = np.empty((queries.shape[0], k), np.int32)
    lib().orc_brute_force(data, data.shape[0], data.shape[1], queries, queries.shape[0], k, out)
    return out


def greedy_search(offsets, nbrs, data, queries, L, k, entry=0):
    data, queries = _f32(data), _f32(queries)
    nq = queries.shape[0]
    entries = np.full(nq, entry, np.int64) if np.isscalar(entry) else np.ascontiguousarray(entry, np.int64)
    out = np.empty((nq, k), np.int32)
    nb = _i32a(nbrs) if len(nbrs) else np.zeros(1, np.int32)
    lib().orc_greedy_search(
        np.ascontiguousarray(offsets, np.int64), nb, data, data.shape[0], data.shape[1],
        queries, nq, L, k, entries, out,
    )
    return out


def mean_recall(ids, truth) -> float:
    """search.mean_recall (search.py:145-159): |retrieved & truth| / k averaged."""
    k = truth.shape[1]
    return float(np.mean([len(set(ids[i].tolist()) & set(truth[i].tolist())) / k for i in range(ids.shape[0])]))


if os.environ.get("GRNND_ORACLE_THREADS"):
    set_threads(int(os.environ["GRNND_ORACLE_THREADS"]))
