"""Per-round pool-size distribution of a C2-shape build (development aid): for selected
update rounds, the number of pools / rows / upper-bound pairs per tensor-core bin
(k <= 8, 16, 24, 32, 48, 96) and the number of 96-row groups each bin launches."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2510_02774_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 128
ds = g.generate(n, dim, "gaussian", seed=1)
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
st = g.init_neighbors(ds, p)
row = torch.zeros(16, dtype=torch.int64, device="cuda")
edges = [1, 8, 16, 24, 32, 48, 96]
gp = [12, 6, 4, 3, 2, 1]
show = {1, 2, 4, 8, 15, 16, 20, 30, 45, 60}
r = 0
for t1 in range(1, p.T1 + 1):
    for _ in range(p.T2):
        r += 1
        if r in show:
            k = st.pools.read_count.cpu().numpy().astype(np.int64)
            line = [f"round {r:2d}: sum_k {k.sum() / 1e6:6.2f}M mean {k.mean():5.1f} p50 {np.percentile(k, 50):.0f} "
                    f"p90 {np.percentile(k, 90):.0f} p99 {np.percentile(k, 99):.0f} max {k.max()}"]
            tot_g = 0
            for b in range(6):
                m = (k > edges[b]) & (k <= edges[b + 1])
                npool = int(m.sum())
                grp = (npool + gp[b] - 1) // gp[b]
                tot_g += grp
                line.append(f"   bin<= {edges[b + 1]:2d}: pools {npool:7d} rows {k[m].sum() / 1e6:6.2f}M "
                            f"pairs {(k[m] * (k[m] - 1) // 2).sum() / 1e6:7.1f}M groups {grp:7d} "
                            f"rows/group {k[m].sum() / max(grp, 1):5.1f}")
            line.append(f"   total groups {tot_g}")
            print("\n".join(line), flush=True)
        st.pools.update(p.seed, 1 + st.round_index, 0, row)
        st.round_index += 1
    if t1 != p.T1:
        st.pools.reverse(p.rho, row)
torch.cuda.synchronize()
