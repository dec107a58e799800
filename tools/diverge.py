"""Round-by-round comparison of the device build with the oracle State (development aid,
e.g. under compute-sanitizer): prints the first round whose pools differ and the rows.
    python tools/diverge.py [n] [reps]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import oracle
import paper_2510_02774_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ds = g.generate(n, 128, "gaussian", seed=1)
params = g.BuildParams(S=20, R=96, T1=2, T2=3, rho=0.6, seed=1)
bad = 0
for rep in range(reps):
    st = g.init_neighbors(ds, params)
    ost = oracle.State(ds.data, 20, 96, 1)
    r = 0
    ok = True
    for t1 in range(1, params.T1 + 1):
        for kind in ["u"] * params.T2 + (["r"] if t1 != params.T1 else []):
            r += 1
            if kind == "u":
                s = g.update_round(st)
                os_ = ost.update_round(1, st.round_index)
            else:
                s = g.reverse_edge_sampling(st)
                os_ = ost.reverse_round(0.6)
            ids, d, c = st.snapshot()
            oi, od, oc = ost.export()
            if not (np.array_equal(c, oc) and np.array_equal(ids, oi) and np.array_equal(d.view(np.uint32), od.view(np.uint32))):
                rows = np.flatnonzero((c != oc) | (ids != oi).any(1) | (d.view(np.uint32) != od.view(np.uint32)).any(1))
                print(f"rep {rep}: round {r} ({kind}) differs in {len(rows)} rows, first {rows[:8].tolist()}")
                v = int(rows[0])
                print("  gpu   ", c[v], ids[v, :c[v]].tolist())
                print("  oracle", oc[v], oi[v, :oc[v]].tolist())
                print("  stats gpu", [s.messages, s.redirects, s.inserted, s.duplicate, s.replaced, s.rejected],
                      "oracle", os_[[1, 2, 5, 6, 7, 8]].tolist())
                ost.load(ids, d, c)  # continue from the device state
                ok = False
    bad += 0 if ok else 1
print(f"diverge: {bad}/{reps} builds differed")
