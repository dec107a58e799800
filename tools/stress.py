"""Run many C2-shape builds back to back on one engine (no host sync between them) and
count graphs that differ from the reference digest (debug aid).
    python tools/stress.py [builds] [n]"""
import hashlib, json, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200.builder import DeviceBuild, upload
builds = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
data = np.random.default_rng(1).standard_normal((n, 128), dtype=np.float32)
dd = upload(data, torch.device("cuda"))
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
eng = DeviceBuild(dd, 128, p)
ref = json.loads(str(np.load("tests/golden/c2_reference.npz")["meta"])) if n == 1_000_000 else None
keep, bad = [], 0
digests = {}
for b in range(builds):
    off, nb, _, _ = eng.run()
    keep.append((off.clone(), nb.clone(), eng.stats.clone()))
    if len(keep) == 10 or b == builds - 1:
        for o, nbr, st in keep:
            oh = o.cpu().numpy(); e = int(oh[-1])
            d = hashlib.sha256(oh.astype(np.int64).tobytes()).hexdigest()
            d2 = hashlib.sha256(nbr[:e].cpu().numpy().tobytes()).hexdigest()
            digests[(d, d2)] = digests.get((d, d2), 0) + 1
            if ref and (d != ref["sha256_offsets"] or d2 != ref["sha256_neighbor_ids"]):
                bad += 1
                s = st.cpu().numpy()
                print("mismatch: edges", e, "redirects per round", s[:, 1].tolist(), flush=True)
        keep = []
print(f"stress: {builds} builds, {bad} differ from the reference; distinct digests {len(digests)}", flush=True)
