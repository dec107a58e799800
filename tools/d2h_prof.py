"""Where the graph emission time goes (debug aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200 import builder as B
n = 1_000_000
ds = g.generate(n, 128, "gaussian", seed=1)
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
st = g.init_neighbors(ds, p)
B.run_rounds(st)
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    off, nb, bad = B._finalize_device(st.pools); torch.cuda.synchronize(); t.append(time.perf_counter())
    o = off.cpu().numpy(); t.append(time.perf_counter())
    e = int(o[-1]); ids = nb[:e].cpu().numpy(); t.append(time.perf_counter())
    f = int(bad.item()); t.append(time.perf_counter())
    po = torch.empty(off.shape, dtype=off.dtype, pin_memory=True); pn = torch.empty((e,), dtype=torch.int32, pin_memory=True); t.append(time.perf_counter())
    po.copy_(off, non_blocking=True); pn.copy_(nb[:e], non_blocking=True); torch.cuda.synchronize(); t.append(time.perf_counter())
    a1 = po.numpy(); a2 = pn.numpy(); x = np.empty_like(a2); x[:] = a2; t.append(time.perf_counter())
    names = ["finalize", "offsets.cpu", "nbrs.cpu", "bad.item", "pinned alloc", "pinned copy", "numpy copy of pinned"]
    print(" | ".join(f"{k} {1e3*(b-a):.1f}" for k, a, b in zip(names, t[:-1], t[1:])))
