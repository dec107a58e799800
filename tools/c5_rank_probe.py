"""C5 (100M x 96, P = 8) one-rank probe on ONE B200: does a rank's share fit, and how long
do its first rounds take?

This run has one GPU, so the 8-rank build cannot execute.  What can: rank 0's complete
device footprint -- the replicated 100M x 96 vectors generated on the device (38.4 GB),
the row norms, the pools of its 12.5M owned rows, the workspace at the optimistic message
capacity, and the CSR buffers of the final emission -- and its round-1 work, which is
exactly what rank 0 of a real 8-GPU run does in round 1 (init and the round-1 pair phase
depend only on the rank's own rows).  Round 1's apply here receives only rank 0's own
messages (the other ranks' 7/8 are missing), so later rounds are not representative and
are not timed.

    python tools/c5_rank_probe.py [--n 100000000] [--dim 96] [--world 8] [--metric l2|ip]

Prints one JSON line: planned vs measured peak bytes, init / round-1 emit / apply times.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2510_02774_b200 as g  # noqa: E402
from paper_2510_02774_b200.sharded import ShardedBuild, generate_device, memory_plan  # noqa: E402
from paper_2510_02774_b200.builder import _finalize_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--metric", default="l2")
    a = ap.parse_args()
    params = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
    plan = memory_plan(a.n, a.dim, params.R, a.world, a.metric, normalize_in_place=True)
    torch.cuda.reset_peak_memory_stats()
    t0 = time.perf_counter()
    data = generate_device(a.n, a.dim, seed=1, device="cuda:0")
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    sb = ShardedBuild(data, a.dim, params, a.rank, a.world, metric=a.metric, normalize_in_place=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    phase = []
    gen = sb.rounds(phase)
    ev[0].record()
    next(gen)  # init + norms + round-1 emit
    ev[1].record()
    torch.cuda.synchronize()
    pools = sb.pools
    counts = [int(x) for x in pools.send_counts.cpu().tolist()]
    own = counts[a.rank]
    start = sum(counts[: a.rank])
    pools.inb[:own].copy_(pools.out[start:start + own])  # rank 0's own messages only
    ev[2].record()
    gen.send(own)  # round-1 apply, then round-2 emit
    ev[3].record()
    torch.cuda.synchronize()
    offsets, nbrs, bad = _finalize_device(pools)  # the CSR buffers of the final emission
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated()
    free, total = torch.cuda.mem_get_info()
    e1 = phase[0]
    line = {
        "probe": f"C5 rank {a.rank} of {a.world}: {a.n} x {a.dim} {a.metric}, rows {pools.rows}",
        "planned_bytes": plan,
        "peak_allocated_bytes": int(peak),
        "device_total_bytes": int(total),
        "fits": bool(peak < total),
        "generate_s": round(gen_s, 3),
        "init_plus_round1_emit_ms": round(ev[0].elapsed_time(ev[1]), 2),
        "round1_emit_ms": round(e1[0].elapsed_time(e1[1]), 2),
        "round1_messages_out": sum(counts),
        "round1_messages_to_self": own,
        "round1_apply_plus_round2_emit_ms (own messages only)": round(ev[2].elapsed_time(ev[3]), 2),
        "note": "round-1 emit is the real rank-0 work of an 8-GPU run; the apply sees only rank 0's own "
                "messages (one GPU), so nothing after it is representative",
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
