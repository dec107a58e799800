"""Digest of the CPU oracle's build of a workload the reference cannot build here in
reasonable time (C4: 10M x 96 inner product, L2-normalised rows):

    python tests/golden/make_oracle_digest.py c4   -> profiles/oracle_digest_c4.json

The oracle (oracle/, the C restatement of the reference's numba kernels) is pinned to the
reference's own builds bit for bit at C1, C2 and C3 (profiles/oracle_digest_c{1,2}.json,
tests/test_oracle_golden.py), so its digest at C4 stands in for the reference's.  Data:
numpy default_rng(1).standard_normal (the reference's generate recipe), rows normalised in
float64 and rounded to fp32 (oracle.normalize_rows).  Test infrastructure; needs no GPU.
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

CONFIGS = {"c4": (10_000_000, 96, "ip"), "c2": (1_000_000, 128, "l2")}
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
n, d, metric = CONFIGS[name]
data = np.random.default_rng(1).standard_normal((n, d), dtype=np.float32)
if metric == "ip":
    data = oracle.normalize_rows(data)
t0 = time.perf_counter()
off, nb, st = oracle.build(data, 20, 96, 4, 15, 0.6, 1, with_stats=True)
secs = time.perf_counter() - t0
res = {"config": name, "n": n, "dim": d, "metric": metric, "oracle_seconds": secs, "threads": oracle.max_threads(),
       "sha256_offsets": hashlib.sha256(off.astype(np.int64).tobytes()).hexdigest(),
       "sha256_neighbor_ids": hashlib.sha256(nb.astype(np.int32).tobytes()).hexdigest(),
       "edges": int(off[-1]), "stats_fields": ["messages", "redirects", "survivors", "reverse_attempts", "inserted",
                                               "duplicate", "replaced", "rejected"],
       "stats": st[:, 1:9].tolist()}
(ROOT / "profiles" / f"oracle_digest_{name}.json").write_text(json.dumps(res, indent=1))
print(json.dumps({k: v for k, v in res.items() if k != "stats"}, indent=1))
