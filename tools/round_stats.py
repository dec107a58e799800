"""Per-round counters of a C2-shape build (debug aid): entries, redirects, pairs computed,
pairs the reference evaluates, candidates, redirect-capable pairs, active entries."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200 import builder as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dist = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
ds = g.generate(n, dim, dist, seed=1)
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
st = g.init_neighbors(ds, p)
rows = torch.zeros((B.num_rounds(p), 20), dtype=torch.int64, device="cuda")
kinds = B.run_rounds(st, rows)
r = rows.cpu().numpy()
print("round kind   sum_k  redirects  pairs  pairs_ref  cand  redirectable  recpools  active_k")
for i, (k, x) in enumerate(zip(kinds, r)):
    print(f"{i+1:3d} {k[:3]} {x[0]/1e6:8.2f}M {x[1]/1e6:7.3f}M {x[8]/1e6:8.1f}M {x[9]/1e6:8.1f}M {x[10]/1e6:7.2f}M {x[12]/1e6:7.2f}M {x[14]/1e3:8.1f}K {x[15]/1e6:7.2f}M")
