"""Pin the oracle at a whole-build config against the reference's committed digest.

    python tests/golden/check_oracle_digest.py c2  -> profiles/oracle_digest_c2.json

Runs the C oracle (oracle/, the restatement the GPU tests compare against) on the same
generate(N, D, "gaussian", seed=1) corpus and schedule as make_reference_digest.py and
compares sha256 digests of its CSR graph and its per-round stats with the reference's
(tests/golden/<cfg>_reference.npz).  Test infrastructure; needs no GPU.
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

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
ref = np.load(ROOT / "tests" / "golden" / f"{name}_reference.npz")
meta = json.loads(str(ref["meta"]))
data = np.random.default_rng(1).standard_normal((meta["n"], meta["dim"]), dtype=np.float32)
t0 = time.perf_counter()
off, nb, st = oracle.build(data, 20, 96, 4, 15, 0.6, 1, with_stats=True)
secs = time.perf_counter() - t0
so = hashlib.sha256(off.astype(np.int64).tobytes()).hexdigest()
sn = hashlib.sha256(nb.astype(np.int32).tobytes()).hexdigest()
stats_ok = bool(np.array_equal(st[:, 1:9], ref["stats"]))
res = {"config": name, "n": meta["n"], "dim": meta["dim"], "oracle_seconds": secs, "threads": oracle.max_threads(),
       "sha256_offsets": so, "sha256_neighbor_ids": sn, "edges": int(off[-1]),
       "digest_match": so == meta["sha256_offsets"] and sn == meta["sha256_neighbor_ids"],
       "stats_match": stats_ok, "reference_build_seconds": meta["build_seconds"],
       "reference_threads": meta["threads"]}
out = ROOT / "profiles" / f"oracle_digest_{name}.json"
out.write_text(json.dumps(res, indent=1))
print(json.dumps(res, indent=1))
