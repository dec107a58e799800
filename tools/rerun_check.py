"""Digests of repeated runs of one DeviceBuild engine (debug aid)."""
import hashlib, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200.builder import DeviceBuild, upload
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
mc = int(sys.argv[2]) if len(sys.argv) > 2 else 0
data = np.random.default_rng(1).standard_normal((n, 128), dtype=np.float32)
dd = upload(data, torch.device("cuda"))
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
eng = DeviceBuild(dd, 128, p, msg_capacity=mc or None)
for r in range(4):
    ph = [] if r == 2 else None
    off, nb, bad, fail = eng.run(phase_events=ph)
    st = eng.round_stats()
    o = off.cpu().numpy(); e = int(o[-1])
    print(r, eng.pools.msg_capacity, hashlib.sha256(o.astype(np.int64).tobytes()).hexdigest()[:16],
          hashlib.sha256(nb[:e].cpu().numpy().tobytes()).hexdigest()[:16], e,
          "redirects", [s.redirects for s in st][:6], flush=True)
