"""ctypes binding of libgrnnd_b200.so (the C ABI in include/grnnd_b200.h).

There is deliberately no fallback: if the shared library is missing or cannot
be loaded, importing this module raises.  Build it with
``python __graft_entry__.py`` (or ``make -C paper_2510_02774_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import DeviceError, ParamError

LIB_PATH = Path(__file__).resolve().parent / "_build" / "libgrnnd_b200.so"
if os.environ.get("GRNND_B200_LIB"):  # A/B builds of the same sources (tools/variants.sh)
    LIB_PATH = Path(os.environ["GRNND_B200_LIB"]).resolve()

OK, EINVAL, ECUDA, EUNSUPPORTED, EWORKSPACE = 0, 1, 2, 3, 4
NSTATS = 20
ST_MESSAGES, ST_REDIRECTS, ST_SURVIVORS, ST_REVERSE_ATTEMPTS = 0, 1, 2, 3
ST_INSERTED, ST_DUPLICATE, ST_REPLACED, ST_REJECTED = 4, 5, 6, 7
ST_PAIRS, ST_PAIRS_REF, ST_CANDIDATES, ST_OVERFLOWS = 8, 9, 10, 11
ST_REDIRECTABLE, ST_LOST, ST_RECPOOLS, ST_ACTIVE_K = 12, 13, 14, 15
ST_TCV_CHECKED, ST_TCV_MAX_RATIO, ST_TCV_VIOLATIONS = 16, 17, 18
MSG_WORDS = 5
MAX_CAP = 256

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_dbl = C.c_double
_sz = C.c_size_t


class Pools(C.Structure):
    """grnnd_pools (include/grnnd_b200.h)."""

    _fields_ = [
        ("data", _vp),
        ("n_total", _i64),
        ("lo", _i64),
        ("hi", _i64),
        ("dim", _i32),
        ("ld", _i32),
        ("cap", _i32),
        ("read_ids", _vp),
        ("read_dists", _vp),
        ("read_count", _vp),
        ("write_ids", _vp),
        ("write_dists", _vp),
        ("write_count", _vp),
        ("workspace", _vp),
        ("workspace_bytes", _sz),
        ("msg_capacity", _i64),
        ("stats", _vp),
        ("norms", _vp),
        ("filter_split", _i32),
    ]


_SIGS = {
    "grnnd_last_error": (C.c_char_p, []),
    "grnnd_abi_version": (C.c_int, []),
    "grnnd_launch_count": (C.c_ulonglong, []),
    "grnnd_set_instrumentation": (C.c_int, [C.c_int]),
    "grnnd_update_emit": (C.c_int, [C.POINTER(Pools), _u64, _u64, _i32, _vp]),
    "grnnd_reverse_emit": (C.c_int, [C.POINTER(Pools), _dbl, _vp]),
    "grnnd_apply_emitted": (C.c_int, [C.POINTER(Pools), _i32, _vp]),
    "grnnd_hash4_batch": (C.c_int, [_u64, _u64, _vp, _vp, _i64, _vp, _vp]),
    "grnnd_sqdist_batch": (C.c_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "grnnd_sample_initial": (C.c_int, [_i64, _i32, _u64, _vp, _vp, _vp]),
    "grnnd_init_dists": (C.c_int, [_vp, _i64, _i32, _i32, _vp, _i32, _vp, _vp]),
    "grnnd_workspace_bytes": (_sz, [_i64, _i32, _i64]),
    "grnnd_gen_update_messages": (
        C.c_int,
        [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _i32, _u64, _u64, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp],
    ),
    "grnnd_gen_reverse_messages": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _dbl, _vp, _vp, _vp, _vp, _vp]),
    "grnnd_gen_merge_messages": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "grnnd_message_offsets": (C.c_int, [_vp, _i64, _vp, _vp, _sz, _vp]),
    "grnnd_compact_messages": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "grnnd_group_by_target": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "grnnd_apply_grouped_messages": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "grnnd_init_pools": (C.c_int, [C.POINTER(Pools), _i32, _u64, _vp, _vp]),
    "grnnd_update_round": (C.c_int, [C.POINTER(Pools), _u64, _u64, _i32, _vp]),
    "grnnd_reverse_round": (C.c_int, [C.POINTER(Pools), _dbl, _vp]),
    "grnnd_round_emit": (C.c_int, [C.POINTER(Pools), _i32, _u64, _u64, _i32, _dbl, _vp, _i32, _vp, _vp]),
    "grnnd_round_buffers": (C.c_int, [C.POINTER(Pools), C.POINTER(_vp), C.POINTER(_vp)]),
    "grnnd_round_apply": (C.c_int, [C.POINTER(Pools), _i32, _i64, _vp]),
    "grnnd_finalize": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "grnnd_sorted_rows": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "grnnd_finalize_pools": (C.c_int, [C.POINTER(Pools), _vp, _vp, _vp, _vp]),
    "grnnd_check_finite": (C.c_int, [_vp, _i64, _i32, _i32, _vp, _vp]),
    "grnnd_row_norms": (C.c_int, [_vp, _i64, _i32, _i32, _vp, _vp]),
    "grnnd_band_terms": (C.c_int, [C.POINTER(Pools), _vp, _vp]),
    "grnnd_brute_force_workspace_bytes": (_sz, [_i64, _i64, _i32]),
    "grnnd_brute_force": (C.c_int, [_vp, _i64, _i32, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "grnnd_search_visited_bytes": (_sz, [_i64, _i64]),
    "grnnd_greedy_search": (
        C.c_int, [_vp, _vp, _i64, _vp, _i32, _i32, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    ),
    "grnnd_normalize_rows": (C.c_int, [_vp, _i64, _i32, _i32, _vp]),
    "grnnd_refine_accept_loop": (C.c_int, [_vp, _i32, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: the B200 kernels are not built (run `python __graft_entry__.py`"
        " or `make -C paper_2510_02774_b200/csrc`); there is no CPU fallback"
    )

lib = C.CDLL(str(LIB_PATH))
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    msg = lib.grnnd_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map a C status code to the reference's exception types."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == EINVAL:
        raise ParamError(msg)
    raise DeviceError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)
