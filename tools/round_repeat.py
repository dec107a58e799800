"""Repeat one update round's emit many times from the same state and diff (debug aid).
    python tools/round_repeat.py [round] [reps] [n]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200.builder import STREAM_ROUND_BASE, upload
from paper_2510_02774_b200.sharded import ShardPools

rnd = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
dev = torch.device("cuda")
data = np.random.default_rng(1).standard_normal((n, 128), dtype=np.float32)
dd = upload(data, dev)
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
pools = ShardPools(dd, 128, 96, 0, n, n, 1)
bounds = torch.tensor([0, n], dtype=torch.int64, device=dev)
pools.compute_norms()
pools.init(p.S, p.seed)
stats = torch.zeros(32, dtype=torch.int64, device=dev)
for ri in range(rnd - 1):  # plain rounds up to the one under test
    pools.update(p.seed, STREAM_ROUND_BASE + ri, 0, stats)
snap = [t.clone() for t in (pools.read_ids, pools.read_dists, pools.read_count)]


def run():
    for dst, src in zip((pools.read_ids, pools.read_dists, pools.read_count), snap):
        dst.copy_(src)
    pools.write_count.zero_()
    stats.zero_()
    pools.emit(0, p.seed, STREAM_ROUND_BASE + rnd - 1, 0, p.rho, bounds, stats)
    c = int(pools.send_counts[0].item())
    m = pools.out[:c].clone()
    key = (m[:, 0].to(torch.int64) & 0xFFFFFFFF) | (m[:, 1].to(torch.int64) << 32)
    o = torch.argsort(key)
    return c, m[o], key[o], pools.read_ids.clone(), stats.clone()


c0, m0, k0, t0, s0 = run()
print(f"round {rnd}: {c0} messages; stats {s0[:16].tolist()}", flush=True)
bad = 0
for r in range(reps):
    c, m, k, t, s = run()
    if c == c0 and torch.equal(m, m0) and torch.equal(t, t0):
        continue
    bad += 1
    rows = torch.nonzero((t != t0).any(1)).flatten()
    srcs = set((k0 // 96).tolist()) ^ set((k // 96).tolist())
    print(f"rep {r}: count {c} vs {c0}; stats {s[:16].tolist()}", flush=True)
    print(f"   tombstone rows differ: {rows[:10].tolist()} (of {len(rows)})", flush=True)
    for v in rows[:3].tolist():
        kv = int(snap[2][v])
        print(f"   v={v} k={kv} ids={snap[0][v, :kv].tolist()}", flush=True)
        print(f"      ref tomb {(t0[v, :kv] == -1).nonzero().flatten().tolist()}", flush=True)
        print(f"      bad tomb {(t[v, :kv] == -1).nonzero().flatten().tolist()}", flush=True)
        sel0 = (k0 // 96) == v
        sel = (k // 96) == v
        print(f"      ref msgs {m0[sel0][:, 2:].tolist()}", flush=True)
        print(f"      bad msgs {m[sel][:, 2:].tolist()}", flush=True)
    if bad >= 3:
        break
print(f"round_repeat: {bad} of {reps} reps differ", flush=True)
