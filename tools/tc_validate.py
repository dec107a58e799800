"""Run a C2-shape schedule with a GRNND_TC_VALIDATE build and report the tensor-core filter's
observed error against its bound (stats[13] pairs checked, [14] max err/bound ratio bits,
[15] violations)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200 import builder as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dist = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
T2 = int(sys.argv[4]) if len(sys.argv) > 4 else 15
ds = g.generate(n, dim, dist, seed=1)
params = g.BuildParams(S=20, R=96, T1=2, T2=T2, rho=0.6, seed=1)
st = g.init_neighbors(ds, params)
rows = torch.zeros((B.num_rounds(params), 16), dtype=torch.int64, device="cuda")
p = st.params
i = 0
for t1 in range(1, p.T1 + 1):
    for _ in range(p.T2):
        st.pools.update(p.seed, 1 + st.round_index, 0, rows[i]); st.round_index += 1; i += 1
    if t1 != p.T1:
        st.pools.reverse(p.rho, rows[i]); i += 1
torch.cuda.synchronize()
r = rows.cpu().numpy()
ratio = r[:, 14].astype(np.int64).astype(np.int32).view(np.float32)
print(f"{dist} n={n} dim={dim}: pairs checked {r[:,13].sum():.4e}, violations {r[:,15].sum()}, "
      f"max err/bound {ratio.max():.4f}, pairs {r[:,8].sum():.4e}")
