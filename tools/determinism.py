"""Back-to-back C2 builds on one engine with no host sync between them (the bench's timed
loop); every run's graph is kept on the device and compared at the end (debug aid).
    python tools/determinism.py [n] [runs] [mode]   mode: nosync | sync"""
import hashlib, sys, threading, subprocess
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200.builder import DeviceBuild, upload
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 6
mode = sys.argv[3] if len(sys.argv) > 3 else "nosync"
data = np.random.default_rng(1).standard_normal((n, 128), dtype=np.float32)
dd = upload(data, torch.device("cuda"))
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
eng = DeviceBuild(dd, 128, p)
keep = []
for r in range(runs):
    off, nb, bad, fail = eng.run()
    keep.append((off.clone(), nb.clone(), eng.stats.clone()))
    if mode == "sync":
        torch.cuda.synchronize()
torch.cuda.synchronize()
for r, (off, nb, st) in enumerate(keep):
    o = off.cpu().numpy(); e = int(o[-1])
    s = st.cpu().numpy()
    print(r, hashlib.sha256(o.astype(np.int64).tobytes()).hexdigest()[:16],
          hashlib.sha256(nb[:e].cpu().numpy().tobytes()).hexdigest()[:16], e,
          "first differing round vs run 0:",
          next((i for i in range(len(s)) if not np.array_equal(s[i, :8], keep[0][2].cpu().numpy()[i, :8])), None),
          flush=True)
