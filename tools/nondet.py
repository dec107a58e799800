"""Nondeterminism hunt (debug aid): a C2-shape build driven round by round through the
one-rank sharded round API; every update round's emit is run twice from the same pool
state and the packed message lists (sorted by key) and tombstoned rows compared, then the
apply is run twice from the same state and the new pools compared.
    python tools/nondet.py [n] [reps_per_round]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200.builder import STREAM_ROUND_BASE, upload
from paper_2510_02774_b200.sharded import ShardPools

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda")
data = np.random.default_rng(1).standard_normal((n, 128), dtype=np.float32)
dd = upload(data, dev)
p = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
pools = ShardPools(dd, 128, 96, 0, n, n, 1)
bounds = torch.tensor([0, n], dtype=torch.int64, device=dev)
pools.compute_norms()
pools.init(p.S, p.seed)
stats = torch.zeros(32, dtype=torch.int64, device=dev)


def sorted_msgs(c):
    m = pools.out[:c].clone()
    key = (m[:, 0].to(torch.int64) & 0xFFFFFFFF) | (m[:, 1].to(torch.int64) << 32)
    return m[torch.argsort(key)]


def state():
    return [t.clone() for t in (pools.read_ids, pools.read_dists, pools.read_count, pools.write_ids,
                                pools.write_dists, pools.write_count)]


def restore(s):
    for dst, src in zip((pools.read_ids, pools.read_dists, pools.read_count, pools.write_ids, pools.write_dists,
                         pools.write_count), s):
        dst.copy_(src)


bad = 0
ri = 0
for t1 in range(1, p.T1 + 1):
    for kind in [0] * p.T2 + ([1] if t1 != p.T1 else []):
        s0 = state()
        outs = []
        for r in range(reps):
            restore(s0)
            stats.zero_()
            pools.emit(kind, p.seed, STREAM_ROUND_BASE + ri, 0, p.rho, bounds, stats)
            c = int(pools.send_counts[0].item())
            outs.append((c, sorted_msgs(c), pools.read_ids.clone()))
        for r in range(1, reps):
            same = outs[r][0] == outs[0][0] and torch.equal(outs[r][1], outs[0][1]) and torch.equal(outs[r][2], outs[0][2])
            if not same:
                bad += 1
                c0, m0, t0 = outs[0]
                c1, m1, t1_ = outs[r]
                rows = torch.nonzero((t0 != t1_).any(1)).flatten()[:5].tolist()
                print(f"round {ri + 1 if kind == 0 else 'rev'} kind {kind}: EMIT differs (rep {r}): counts {c0} vs {c1}, "
                      f"tombstone rows differ {int((t0 != t1_).any(1).sum())} e.g. {rows}", flush=True)
                if c0 == c1:
                    d = torch.nonzero((m0 != m1).any(1)).flatten()[:5]
                    print("   first differing messages:", m0[d].tolist(), m1[d].tolist(), flush=True)
        # apply twice from the same emitted state
        s1 = state()
        c = outs[-1][0]
        saved = pools.out[:c].clone()  # the send buffer doubles as sort scratch during apply
        app = []
        for r in range(reps):
            restore(s1)
            pools.inb[:c].copy_(saved)
            stats.zero_()
            p_ = pools.struct(stats)
            import ctypes as C
            from paper_2510_02774_b200 import _lib
            from paper_2510_02774_b200.builder import _stream
            _lib.call("grnnd_round_apply", C.byref(p_), kind, int(c), _stream(dev))
            app.append((pools.write_ids.clone(), pools.write_dists.clone(), pools.write_count.clone()))
        for r in range(1, reps):
            if not all(torch.equal(a, b) for a, b in zip(app[r], app[0])):
                bad += 1
                rows = torch.nonzero(app[r][2] != app[0][2]).flatten()[:5].tolist()
                print(f"round {ri + 1} kind {kind}: APPLY differs (rep {r}); count rows {rows}", flush=True)
        pools.swap()
        if kind == 0:
            ri += 1
torch.cuda.synchronize()
print(f"nondet: {bad} differing phases", flush=True)
