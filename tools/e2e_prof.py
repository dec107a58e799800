"""Stage times of the public build() from pinned host memory (debug aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200 import builder as B

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
data = np.random.default_rng(1).standard_normal((n, 128), dtype=np.float32)
host = torch.from_numpy(data).pin_memory()
ds = g.Dataset(host.numpy())
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
g.build(ds, p)  # warm
torch.cuda.synchronize()
for rep in range(3):
    T = {}
    t0 = time.perf_counter()
    def mark(k):
        torch.cuda.synchronize()
        T[k] = time.perf_counter()
    dev = torch.device("cuda")
    d = B.upload(ds.data, dev); mark("h2d")
    B.check_finite_device(d, 128); mark("finite")
    pools = B._DevicePools(d, 128, 96, msg_capacity=B.optimistic_msg_capacity(n, 96)); mark("alloc+norms")
    pools.init(p.S, p.seed); mark("init")
    st = B.BuildState(ds, p, pools)
    rows = torch.zeros((B.num_rounds(p), 20), dtype=torch.int64, device=dev)
    B.run_rounds(st, rows); mark("rounds")
    hr = rows.cpu().numpy(); mark("stats")
    graph = B.finalize_graph(st); mark("finalize+d2h")
    t1 = time.perf_counter()
    prev = t0
    print(f"rep {rep}: total {1e3*(t1-t0):.1f} ms: " + " ".join(f"{k} {1e3*(v-prev):.1f}" for k, v in T.items() if not (prev := prev) or True) )
    prev = t0
    out = []
    for k, v in T.items():
        out.append(f"{k} {1e3*(v-prev):.1f}")
        prev = v
    print("   ", " | ".join(out))
    t0 = time.perf_counter(); gg = g.build(ds, p); t1 = time.perf_counter()
    print(f"    build() {1e3*(t1-t0):.1f} ms")
