"""Quick device timing of a full build (development aid, not the bench)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200 import builder as B

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dist = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
ds = g.generate(n, dim, dist, seed=1)
params = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = g.init_neighbors(ds, params)
    rows = torch.zeros((B.num_rounds(params), 16), dtype=torch.int64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(B.num_rounds(params) + 2)]
    ev[0].record()
    p = st.params
    i = 0
    for t1 in range(1, p.T1 + 1):
        for _ in range(p.T2):
            st.pools.update(p.seed, 1 + st.round_index, 0, rows[i]); st.round_index += 1; i += 1
            ev[i].record()
        if t1 != p.T1:
            st.pools.reverse(p.rho, rows[i]); i += 1
            ev[i].record()
    off, nb, bad = B._finalize_device(st.pools)
    ev[i + 1].record()
    torch.cuda.synchronize()
    t1_ = time.perf_counter()
    per = [ev[j].elapsed_time(ev[j + 1]) for j in range(i + 1)]
    r = rows.cpu().numpy()
    print(f"rep {rep}: wall {t1_ - t0:.3f}s  rounds+finalize device {sum(per):.1f} ms")
    print("  per-round ms:", " ".join(f"{x:.1f}" for x in per))
    print("  pairs total %.3e  pairs_ref %.3e  sum_k %.3e  candidates %.3e (%.2f%%)  overflows %d" % (
        r[:, 8].sum(), r[:, 9].sum(), r[:, 0].sum(), r[:, 10].sum(), 100 * r[:, 10].sum() / max(r[:, 8].sum(), 1),
        r[:, 11].sum()))
    print("  redirect-capable pairs %.3e (%.3f%% of pairs)" % (r[:, 12].sum(), 100 * r[:, 12].sum() / max(r[:, 8].sum(), 1)))
    print("  per-round candidates %:", " ".join(f"{100 * a / max(b, 1):.2f}" for a, b in zip(r[:, 10], r[:, 8])))
