"""One-time calibration: the full CPU oracle build of the bench workload, round by round,
on all host threads -> profiles/c2_cpu_rounds.json (per-round CPU seconds).  bench.py uses
the per-round shape to extrapolate its bounded CPU sample.  Run on the GPU box's host."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle
from paper_2510_02774_b200.core import generate

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
out = Path(sys.argv[2]) if len(sys.argv) > 2 else Path("profiles/c2_cpu_rounds.json")
S, R, T1, T2, rho, seed = 20, 96, 4, 15, 0.6, 1
data = generate(n, 128, "gaussian", seed=1).data
t0 = time.perf_counter(); st = oracle.State(data, S, R, seed); t_init = time.perf_counter() - t0
rounds = []
ri = 0
for t1 in range(1, T1 + 1):
    for _ in range(T2):
        t0 = time.perf_counter(); s = st.update_round(seed, 1 + ri, 0); dt = time.perf_counter() - t0
        rounds.append({"kind": "update", "seconds": dt, "messages": int(s[1]), "redirects": int(s[2])}); ri += 1
        print(ri, f"{dt:.2f}s", flush=True)
    if t1 != T1:
        t0 = time.perf_counter(); s = st.reverse_round(rho); dt = time.perf_counter() - t0
        rounds.append({"kind": "reverse", "seconds": dt, "messages": int(s[1])})
t0 = time.perf_counter(); off, nb = st.finalize(); t_fin = time.perf_counter() - t0
total = t_init + sum(r["seconds"] for r in rounds) + t_fin
res = {"n": n, "dim": 128, "threads": oracle.max_threads(), "init_s": t_init, "finalize_s": t_fin,
       "total_s": total, "rounds": rounds, "edges": int(off[-1])}
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps(res, indent=1))
print("total", total)
