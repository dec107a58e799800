"""Fixtures for the sequential oracle from the reference itself:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_seq_golden.py

* refine_accept_loop on sorted candidate lists of a random corpus (_numba_kernels.py:354-381);
* two whole build_seq graphs (sequential.py:169-179).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import grnnd  # noqa: E402
from grnnd import BuildParams  # noqa: E402

grnnd.set_backend("numba")
k = grnnd.backend.get_kernels()
out = {}
rng = np.random.default_rng(5)
data = rng.standard_normal((300, 12)).astype(np.float32)
for t in range(6):
    kk = int(rng.integers(1, 60))
    ids = rng.choice(300, kk, replace=False).astype(np.int32)
    d = rng.random(kk).astype(np.float32) * 20
    if t == 5:
        d[:] = np.float32(7.0)  # ties: (dist, id) order
    o = np.lexsort((ids, d))
    ids, d = ids[o], d[o]
    a_i = np.empty(kk, np.int32); a_d = np.empty(kk, np.float32)
    r_t = np.empty(kk, np.int32); r_i = np.empty(kk, np.int32); r_d = np.empty(kk, np.float32)
    na, nr = k.refine_accept_loop(data, ids, d, a_i, a_d, r_t, r_i, r_d)
    out[f"ral{t}_in"] = np.stack([ids.view(np.int32), d.view(np.int32)])
    out[f"ral{t}_acc"] = np.stack([a_i[:na], a_d[:na].view(np.int32)])
    out[f"ral{t}_red"] = np.stack([r_t[:nr], r_i[:nr], r_d[:nr].view(np.int32)])
out["ral_data"] = data
for name, (n, dim, dist, p) in {
    "seqA": (1500, 8, "gaussian", BuildParams(S=8, R=16, T1=2, T2=3, seed=4)),
    "seqB": (800, 24, "clustered", BuildParams(S=6, R=12, T1=1, T2=2, seed=9)),
}.items():
    ds = grnnd.generate(n, dim, dist, seed=3)
    g = grnnd.build_seq(ds, p)
    out[f"{name}_data"] = ds.data
    out[f"{name}_offsets"] = g.offsets
    out[f"{name}_nbrs"] = g.neighbor_ids
    out[f"{name}_params"] = np.array([p.S, p.R, p.T1, p.T2, p.seed], np.int64)
np.savez_compressed(Path(__file__).resolve().parent / "seq.npz", **out)
print("wrote seq.npz", sorted(out))
