"""Pin a whole-build config against the REFERENCE itself: digest + stats + recall.

Run in the build container (where /root/reference exists), e.g. for C2:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reference_digest.py c2

It runs the reference's own numba build (`grnnd.build`, builder.py:365-390) on the
reference's `generate(N, D, "gaussian", seed=1)` corpus with S20 R96 T1=4 T2=15 rho=.6
seed=1, then:

* sha256 of the CSR `offsets` (int64) and `neighbor_ids` (int32) bytes;
* the per-round `RoundStats` rows (63 x 8);
* `brute_force_knn_batch` truth (k=10) for 1000 queries `generate(1000, D, "gaussian",
  seed=2)` (search.py:130-142) and `search_batch` ids + recall@10 at L in
  {32, 64, 96, 128, 256}, entry 0 (search.py:90-115, 155-159);
* k-NN-graph recall@10 over 1000 sampled vertices: the fraction of each
  sampled vertex's 10 exact nearest neighbours (excluding itself) that are among its
  out-neighbours.

Everything lands in tests/golden/<name>_reference.npz (small: digests, stats, ids); the
full graph goes to /tmp/<name>_ref_graph.npz for local oracle comparisons only.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import grnnd  # noqa: E402
from grnnd import BuildParams  # noqa: E402
from grnnd.search import SearchParams, brute_force_knn_batch, mean_recall, search_batch  # noqa: E402

CONFIGS = {
    "c1": (20_000, 128),
    "c2": (1_000_000, 128),
    "c3": (1_000_000, 960),
    "c2c": (1_000_000, 128),  # clustered(5), queries held out of the same draw
}
HELD_OUT = {"c2c"}
LS = (32, 64, 96, 128, 256)
NQ = 1000
NS = 1000  # sampled vertices for k-NN-graph recall


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def knn_graph_recall(graph, data, sample: np.ndarray, threads: int) -> tuple[float, np.ndarray]:
    # exact 11-NN of each sampled vertex (it finds itself at distance 0); drop the vertex
    truth = brute_force_knn_batch(grnnd.Dataset(data), data[sample], 11, threads=threads)
    hits = 0
    t10 = np.empty((sample.shape[0], 10), np.int32)
    for i, v in enumerate(sample):
        row = [int(x) for x in truth[i] if int(x) != int(v)][:10]
        t10[i] = row
        nb = set(graph.neighbor_ids[graph.offsets[v]:graph.offsets[v + 1]].tolist())
        hits += len(nb & set(row))
    return hits / (10.0 * sample.shape[0]), t10


def main() -> None:
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    n, d = CONFIGS[name]
    threads = os.cpu_count() or 1
    grnnd.set_backend("numba")
    k = grnnd.backend.get_kernels()
    k.warmup()
    # one throwaway small build so every JIT specialisation is compiled
    grnnd.build(grnnd.generate(2000, d, "gaussian", seed=3),
                BuildParams(S=20, R=96, T1=2, T2=2, rho=0.6, seed=1, workers=threads))

    if name in HELD_OUT:
        # one draw of n + NQ rows (a different seed would move the cluster centres, io.py:151-153);
        # the last NQ rows are the queries
        full = grnnd.generate(n + NQ, d, "clustered", seed=1).data
        ds = grnnd.Dataset(np.ascontiguousarray(full[:n]))
        held = np.ascontiguousarray(full[n:])
    else:
        ds = grnnd.generate(n, d, "gaussian", seed=1)
        held = None
    params = BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1, workers=threads)
    stats: list = []
    t0 = time.perf_counter()
    g = grnnd.build(ds, params, report_stats=stats)
    build_s = time.perf_counter() - t0
    print(f"{name}: build {build_s:.1f}s on {threads} threads, edges {g.offsets[-1]}", flush=True)
    fields = ("messages", "redirects", "survivors", "reverse_attempts", "inserted", "duplicate",
              "replaced", "rejected")
    stats_arr = np.array([[getattr(s, f) for f in fields] for s in stats], np.int64)
    np.savez(f"/tmp/{name}_ref_graph.npz", offsets=g.offsets, neighbor_ids=g.neighbor_ids)

    q = held if held is not None else grnnd.generate(NQ, d, "gaussian", seed=2).data
    t0 = time.perf_counter()
    truth = brute_force_knn_batch(ds, q, 10, threads=threads)
    bf_s = time.perf_counter() - t0
    ids_l, rec_l = [], []
    for L in LS:
        ids, _ = search_batch(g, ds, q, SearchParams(L=L, k=10), threads=threads)
        ids_l.append(ids)
        rec_l.append(mean_recall(ids, truth))
    print("recall@10", dict(zip(LS, rec_l)), flush=True)
    sample = np.random.default_rng(7).choice(n, NS, replace=False).astype(np.int64)
    sample.sort()
    kg, kg_truth = knn_graph_recall(g, ds.data, sample, threads)
    print(f"knn-graph recall@10 {kg:.4f}", flush=True)

    out = Path(__file__).resolve().parent / f"{name}_reference.npz"
    meta = {"n": n, "dim": d, "distribution": "clustered" if name in HELD_OUT else "gaussian",
            "queries": "held out (last 1000 rows of one draw)" if name in HELD_OUT else "generate(1000, D, seed=2)",
            "S": 20, "R": 96, "T1": 4, "T2": 15, "rho": 0.6, "seed": 1,
            "threads": threads, "build_seconds": build_s, "brute_force_seconds": bf_s,
            "numba": __import__("numba").__version__, "edges": int(g.offsets[-1]),
            "sha256_offsets": sha(g.offsets.astype(np.int64)),
            "sha256_neighbor_ids": sha(g.neighbor_ids.astype(np.int32)),
            "recall_at_10": dict(zip(map(str, LS), rec_l)), "knn_graph_recall_at_10": kg,
            "stats_fields": fields}
    np.savez_compressed(out, meta=np.array(json.dumps(meta)), stats=stats_arr, truth=truth,
                        Ls=np.array(LS, np.int32), search_ids=np.stack(ids_l),
                        recall=np.array(rec_l), knn_sample=sample, knn_truth=kg_truth,
                        knn_graph_recall=np.array(kg))
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
