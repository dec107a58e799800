"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``grnnd`` (numba backend, the reference's
default) and records inputs/outputs of each build-path kernel and of whole
builds into tests/golden/*.npz.  The GPU box never reads /root/reference;
tests compare the oracle (CPU) and the CUDA path against these files.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import grnnd  # noqa: E402
from grnnd import BuildParams  # noqa: E402
from grnnd import _numba_kernels as nk  # noqa: E402
from grnnd import builder as rb  # noqa: E402
from grnnd import rng as rrng  # noqa: E402

grnnd.set_backend("numba")
OUT = Path(__file__).resolve().parent

# ------------------------------------------------------------------ RNG KATs
hash_cases = [(0, 0, 0, 0), (1, 2, 3, 4), (2**63, 5, 12345, 999), (2**64 - 1, 7, 1, 1),
              (123456789, 1, 42, 7), (1, 1, 999999, 95), (42, 61, 7, 2**22 + 3)]
hash_in = np.array(hash_cases, dtype=np.uint64)
hash_out = np.array([rrng.hash4(*c) for c in hash_cases], dtype=np.uint64)
perm_cases = [(16, 1, 2, 3), (20, 1, 1, 0), (96, 7, 33, 123456), (2, 5, 5, 5), (1, 0, 1, 0)]
perms = [rrng.fisher_yates_perm(*c) for c in perm_cases]
samp_cases = [(37, 5, 99), (5, 4, 3), (1000, 20, 1), (200, 8, 42)]
samples = []
for n, c, s in samp_cases:
    out = np.full((n, c), -1, np.int32)
    flag = np.zeros(1, np.int64)
    nk.sample_initial(n, c, np.uint64(s), out, flag)
    assert flag[0] == 0
    samples.append(out)
np.savez_compressed(
    OUT / "rng.npz",
    hash_in=hash_in, hash_out=hash_out,
    perm_cases=np.array(perm_cases, dtype=np.int64),
    perms=np.array([np.pad(p, (0, 96 - len(p)), constant_values=-1) for p in perms], dtype=np.int32),
    samp_cases=np.array(samp_cases, dtype=np.int64),
    **{f"sample_{i}": s for i, s in enumerate(samples)},
)

# ------------------------------------------------------------------ distances
g = np.random.default_rng(20240612)
dist = {}
for d in (1, 3, 16, 100, 128, 960):
    a = g.standard_normal((64, d)).astype(np.float32)
    b = g.standard_normal((64, d)).astype(np.float32)
    dist[f"a_{d}"] = a
    dist[f"b_{d}"] = b
    dist[f"out_{d}"] = np.array([nk.sqdist(a[i], b[i]) for i in range(64)], dtype=np.float32)
np.savez_compressed(OUT / "sqdist.npz", **dist)


# ------------------------------------------------------------------ per-stage kernels
def state_after(ds, params, n_updates, reverse_after=None):
    st = rb.init_neighbors(ds, params)
    for r in range(n_updates):
        rb.update_round(st)
        if reverse_after is not None and r == reverse_after:
            rb.reverse_edge_sampling(st)
    return st


stage = {}
cases = [
    ("gauss16", grnnd.generate(600, 16, "gaussian", seed=3), BuildParams(S=10, R=24, seed=5), 2, 0),
    ("int8", grnnd.Dataset(np.random.default_rng(7).integers(-8, 9, (500, 32)).astype(np.float32)),
     BuildParams(S=8, R=16, seed=9), 3, 1),
    ("clust4", grnnd.generate(400, 4, "clustered", seed=11, clusters=3), BuildParams(S=12, R=40, seed=2), 1, 0),
    ("gauss128", grnnd.generate(300, 128, "gaussian", seed=1), BuildParams(S=20, R=96, seed=1), 2, 0),
    ("asc_u8", grnnd.generate(300, 8, "uniform", seed=4), BuildParams(S=8, R=20, seed=4), 1, 1),
]
for name, ds, params, n_up, order in cases:
    st = state_after(ds, params, n_up)
    n, cap = st.read_ids.shape
    rid = st.read_ids.copy()
    rd = st.read_dists.copy()
    rc = st.read_count.copy()
    seed = params.seed
    stream = 1 + n_up
    mt = np.full(n * cap, -7, np.int32)
    mi = np.full(n * cap, -7, np.int32)
    md = np.full(n * cap, -7.0, np.float32)
    mc = np.zeros(n, np.int32)
    after = rid.copy()
    nk.gen_update_messages(ds.data, after, rd, rc, np.uint64(seed), np.uint64(stream), order, mt, mi, md, mc)
    stage[f"{name}_data"] = ds.data
    stage[f"{name}_rid"] = rid
    stage[f"{name}_rd"] = rd
    stage[f"{name}_rc"] = rc
    stage[f"{name}_args"] = np.array([seed, stream, order], dtype=np.int64)
    stage[f"{name}_mt"] = mt
    stage[f"{name}_mi"] = mi
    stage[f"{name}_md"] = md
    stage[f"{name}_mc"] = mc
    stage[f"{name}_after"] = after
    # the rest of that round through the reference: flat, group, apply
    ft, fi, fd, fs = nk.build_flat(mt, mi, md, mc, cap)
    order_, starts = nk.group_by_target(ft, n)
    wi = np.full((n, cap), -1, np.int32)
    wd = np.full((n, cap), np.inf, np.float32)
    wc = np.zeros(n, np.int32)
    oc = nk.apply_grouped_messages(wi, wd, wc, fi, fd, order_, starts)
    stage[f"{name}_order"] = order_
    stage[f"{name}_starts"] = starts
    stage[f"{name}_wi"] = wi
    stage[f"{name}_wd"] = wd
    stage[f"{name}_wc"] = wc
    stage[f"{name}_outcomes"] = np.array(oc, dtype=np.int64)
    # reverse messages on the post-round state
    st2 = state_after(ds, params, n_up + 1)
    for rho in (0.6, 0.7, 1.0):
        rmt = np.full(n * cap, -7, np.int32)
        rmi = np.full(n * cap, -7, np.int32)
        rmd = np.full(n * cap, -7.0, np.float32)
        rmc = np.zeros(n, np.int32)
        nk.gen_reverse_messages(st2.read_ids, st2.read_dists, st2.read_count, rho, rmt, rmi, rmd, rmc)
        tag = f"{name}_rev{int(rho * 10)}"
        stage[f"{tag}_mt"], stage[f"{tag}_mi"], stage[f"{tag}_md"], stage[f"{tag}_mc"] = rmt, rmi, rmd, rmc
    stage[f"{name}_rid2"] = st2.read_ids
    stage[f"{name}_rd2"] = st2.read_dists
    stage[f"{name}_rc2"] = st2.read_count
np.savez_compressed(OUT / "stages.npz", names=np.array([c[0] for c in cases]), **stage)

# random message streams for apply (test_insert.py:63-118 style) incl. hub contention
gen = np.random.default_rng(1234)
apply = {}
ntr = 0
for trial in range(12):
    n_pools = int(gen.integers(1, 8))
    cap = int(gen.integers(1, 9))
    m = int(gen.integers(0, 120))
    tgt = gen.integers(0, n_pools, m).astype(np.int32)
    mid = gen.integers(0, 1000, m).astype(np.int32)
    mid = np.where(mid == tgt, mid + 1000, mid).astype(np.int32)
    mdist = gen.uniform(0, 10, m).astype(np.float32)
    mdist[gen.random(m) < 0.2] = 5.0  # ties
    order_, starts = nk.group_by_target(tgt, n_pools)
    wi = np.full((n_pools, cap), -1, np.int32)
    wd = np.full((n_pools, cap), np.inf, np.float32)
    wc = np.zeros(n_pools, np.int32)
    oc = nk.apply_grouped_messages(wi, wd, wc, mid, mdist, order_, starts)
    for k, v in dict(tgt=tgt, id=mid, dist=mdist, order=order_, starts=starts, wi=wi, wd=wd, wc=wc,
                     oc=np.array(oc, np.int64), shape=np.array([n_pools, cap])).items():
        apply[f"t{trial}_{k}"] = v
    ntr += 1
hub_tgt = np.zeros(5000, np.int32)
hub_id = (1 + np.arange(5000)).astype(np.int32)
hub_d = (np.arange(5000) % 17).astype(np.float32)
order_, starts = nk.group_by_target(hub_tgt, 2)
wi = np.full((2, 8), -1, np.int32)
wd = np.full((2, 8), np.inf, np.float32)
wc = np.zeros(2, np.int32)
oc = nk.apply_grouped_messages(wi, wd, wc, hub_id, hub_d, order_, starts)
for k, v in dict(tgt=hub_tgt, id=hub_id, dist=hub_d, order=order_, starts=starts, wi=wi, wd=wd, wc=wc,
                 oc=np.array(oc, np.int64), shape=np.array([2, 8])).items():
    apply[f"t{ntr}_{k}"] = v
ntr += 1
np.savez_compressed(OUT / "apply.npz", ntrials=np.array(ntr), **apply)

# ------------------------------------------------------------------ whole builds
builds = {}
build_cases = [
    # (tag, n, dim, dist, seed, clusters, S, R, T1, T2, rho, bseed, order)
    ("u500", 500, 4, "uniform", 6, 5, 4, 8, 2, 2, 0.6, 13, "disordered"),
    ("g2000", 2000, 16, "gaussian", 1, 5, 8, 32, 3, 4, 0.6, 1, "disordered"),
    ("c3000", 3000, 32, "clustered", 7, 5, 10, 24, 2, 5, 0.6, 7, "disordered"),
    ("g1000x128", 1000, 128, "gaussian", 1, 5, 20, 96, 2, 3, 0.6, 1, "disordered"),
    ("asc300", 300, 4, "uniform", 2, 5, 4, 8, 2, 2, 0.5, 3, "ascending"),
    ("tiny5", 5, 2, "uniform", 1, 5, 8, 32, 1, 1, 0.6, 0, "disordered"),
    ("rho1", 800, 8, "gaussian", 5, 5, 6, 16, 3, 2, 1.0, 5, "disordered"),
    ("g600x960", 600, 960, "gaussian", 2, 5, 10, 32, 2, 2, 0.6, 2, "disordered"),
]
for tag, n, dim, distn, dseed, cl, S, R, T1, T2, rho, bseed, order in build_cases:
    ds = grnnd.generate(n, dim, distn, seed=dseed, clusters=cl)
    log: list = []
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        gph = grnnd.build(ds, BuildParams(S=S, R=R, T1=T1, T2=T2, rho=rho, seed=bseed, workers=8),
                          pair_order=order, report_stats=log)
    builds[f"{tag}_offsets"] = gph.offsets
    builds[f"{tag}_nbrs"] = gph.neighbor_ids
    builds[f"{tag}_stats"] = np.array(
        [[0 if s.kind == "update" else 1, s.messages, s.redirects, s.survivors, s.reverse_attempts,
          s.inserted, s.duplicate, s.replaced, s.rejected] for s in log], dtype=np.int64)
np.savez_compressed(
    OUT / "builds.npz",
    cases=np.array([[str(x) for x in c] for c in build_cases]),
    **builds,
)

# ------------------------------------------------------------------ acceptance corpus recall (criterion 03)
ds = grnnd.generate(10000, 16, "uniform", seed=1)
q = grnnd.generate(100, 16, "uniform", seed=2).data
truth = grnnd.brute_force_knn_batch(ds, q, 10, threads=8)
gph = grnnd.build(ds, BuildParams(S=8, R=32, T1=3, T2=6, rho=0.6, seed=1, workers=8))
ids, _ = grnnd.search_batch(gph, ds, q, grnnd.SearchParams(L=64, k=10), threads=8)
np.savez_compressed(OUT / "acceptance10k.npz", truth=truth, search_ids=ids,
                    recall=np.array(grnnd.mean_recall(ids, truth)),
                    offsets=gph.offsets, nbrs=gph.neighbor_ids)
print("golden fixtures written to", OUT)
