"""Multi-GPU path.

* CPU (gloo, world_size 2): the sharded round structure -- owned ID ranges, rank
  bucketing, exchange_all_to_all (the same host function the NCCL path uses), keyed
  regrouping with the own-entry splice -- driven with oracle compute, must reproduce the
  single-process reference build bit for bit.
* GPU: build_virtual_shards (P ranks' kernels on one GPU, exchange by concatenation)
  must equal build() and the oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2510_02774_b200.core import generate
from paper_2510_02774_b200.sharded import MSG_WORDS, exchange_all_to_all, pack_messages, shard_bounds, unpack_messages


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _apply_ordered(rows, R, lo, kind, incoming, own_ids, own_d, own_cnt):
    """Per owned target: incoming sorted by key, own entries spliced at src == tgt
    (update) or after everything (reverse); three-stage insert via the oracle."""
    key, tgt, mid, md = incoming
    flat_id, flat_d, starts = [], [], [0]
    for r in range(rows):
        t = lo + r
        sel = np.flatnonzero(tgt == t)
        sel = sel[np.argsort(key[sel], kind="stable")]
        split = np.searchsorted(key[sel], t * R) if kind == 0 else len(sel)
        own = [(own_ids[r, s], own_d[r, s]) for s in range(own_cnt[r]) if own_ids[r, s] != -1]
        seq = [(mid[i], md[i]) for i in sel[:split]] + own + [(mid[i], md[i]) for i in sel[split:]]
        flat_id += [x for x, _ in seq]
        flat_d += [d for _, d in seq]
        starts.append(len(flat_id))
    wi = np.full((rows, R), -1, np.int32)
    wd = np.full((rows, R), np.inf, np.float32)
    wc = np.zeros(rows, np.int32)
    n = len(flat_id)
    oracle.apply_grouped_messages(wi, wd, wc, np.array(flat_id, np.int32), np.array(flat_d, np.float32),
                                  np.arange(n, dtype=np.int64), np.array(starts, np.int64))
    return wi, wd, wc


def _worker(rank, world, port, cfg, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, dim, S, R, T1, T2, rho, seed = cfg
        data = generate(n, dim, "gaussian", seed=seed).data
        b = shard_bounds(n, world)
        lo, hi = b[rank], b[rank + 1]
        rows = hi - lo
        ids_all, _ = oracle.sample_initial(n, S, seed)
        d_all = oracle.init_dists(data, ids_all)
        rid = np.full((rows, R), -1, np.int32)
        rd = np.full((rows, R), np.inf, np.float32)
        rc = np.full(rows, S, np.int32)
        rid[:, :S] = ids_all[lo:hi]
        rd[:, :S] = d_all[lo:hi]
        ri = 0
        for t1 in range(1, T1 + 1):
            for kind in [0] * T2 + ([1] if t1 != T1 else []):
                if kind == 0:
                    mt, mi, md, mc = oracle.gen_update_messages_lo(data, lo, rid, rd, rc, seed, 1 + ri, 0)
                    ri += 1
                else:
                    mt, mi, md, mc = oracle.gen_reverse_messages_lo(lo, rid, rd, rc, rho)
                # outgoing = redirects / reverse edges; survivors stay home (not sent)
                msgs = []
                for v in range(rows):
                    for j in range(mc[v]):
                        t = mt[v * R + j]
                        if kind == 1 or t != lo + v:
                            msgs.append(((lo + v) * R + j, t, mi[v * R + j], md[v * R + j]))
                owner = np.searchsorted(np.array(b[1:]), [m[1] for m in msgs], side="right") if msgs else []
                order = np.argsort(owner, kind="stable") if msgs else []
                msgs = [msgs[i] for i in order]
                send_counts = [int(np.sum(np.asarray(owner) == r)) for r in range(world)]
                # the packed payload (one all-to-all per round), as rank_scatter_kernel lays it out
                out = pack_messages(torch.tensor([m[0] for m in msgs], dtype=torch.int64),
                                    torch.tensor([m[1] for m in msgs], dtype=torch.int32),
                                    torch.tensor([m[2] for m in msgs], dtype=torch.int32),
                                    torch.tensor([m[3] for m in msgs], dtype=torch.float32))
                inb = torch.zeros((n * R, MSG_WORDS), dtype=torch.int32)
                n_in = exchange_all_to_all(out, send_counts, inb)
                incoming = tuple(x.numpy() for x in unpack_messages(inb[:n_in]))
                rid, rd, rc = _apply_ordered(rows, R, lo, kind, incoming, rid, rd, rc)
        off, nb = oracle.finalize(rid, rd, rc)
        parts = [None] * world
        dist.all_gather_object(parts, (off, nb))
        if rank == 0:
            out_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_exchange_cpu_gloo_bit_exact(world):
    cfg = (600, 8, 8, 16, 2, 3, 0.6, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    base, offs, nbrs = 0, [], []
    for off, nb in parts:
        offs.append(off[:-1] + base)
        nbrs.append(nb)
        base += int(off[-1])
    offsets = np.concatenate(offs + [np.array([base])])
    n, dim, S, R, T1, T2, rho, seed = cfg
    want_off, want_nb = oracle.build(generate(n, dim, "gaussian", seed=seed).data, S, R, T1, T2, rho, seed)
    assert np.array_equal(offsets, want_off)
    assert np.array_equal(np.concatenate(nbrs), want_nb)


def test_pack_roundtrip():
    key = torch.tensor([0, 1, 2**40 + 5, 9_600_000_000, 2**31 - 1, 2**32 + 7], dtype=torch.int64)
    tgt = torch.arange(6, dtype=torch.int32)
    mid = torch.arange(6, dtype=torch.int32) * 3
    d = torch.tensor([0.0, 1.5, float("inf"), 3e-38, 7.25, -0.0], dtype=torch.float32)
    k2, t2, i2, d2 = unpack_messages(pack_messages(key, tgt, mid, d))
    assert torch.equal(k2, key) and torch.equal(t2, tgt) and torch.equal(i2, mid)
    assert torch.equal(d2.view(torch.int32), d.view(torch.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4])
def test_virtual_shards_bit_exact(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_02774_b200 as g
    from paper_2510_02774_b200.sharded import build_virtual_shards

    ds = generate(5000, 32, "gaussian", seed=4)
    params = g.BuildParams(S=12, R=32, T1=3, T2=3, rho=0.6, seed=4)
    log1, logp = [], []
    one = g.build(ds, params, report_stats=log1)
    shard = build_virtual_shards(ds, params, world, report_stats=logp)
    assert np.array_equal(shard.offsets, one.offsets)
    assert np.array_equal(shard.neighbor_ids, one.neighbor_ids)
    assert [s.inserted for s in logp] == [s.inserted for s in log1]
    off, nb = oracle.build(ds.data, 12, 32, 3, 3, 0.6, 4)
    assert np.array_equal(shard.neighbor_ids, nb)


@pytest.mark.gpu
def test_virtual_shards_hub_and_ip():
    """A hub (many vertices near one point: segments above the bitonic cap, the heavy sort
    that uses the send buffer as scratch) and the IP metric through the sharded driver."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_02774_b200 as g
    from paper_2510_02774_b200.sharded import build_virtual_shards

    r = np.random.default_rng(11)
    x = np.concatenate([r.standard_normal((200, 16)) * 0.001, r.standard_normal((9800, 16))]).astype(np.float32)
    ds = g.Dataset(x)
    params = g.BuildParams(S=16, R=64, T1=2, T2=3, rho=1.0, seed=2)
    one = g.build(ds, params)
    for world in (2, 4):
        sh = build_virtual_shards(ds, params, world)
        assert np.array_equal(sh.offsets, one.offsets) and np.array_equal(sh.neighbor_ids, one.neighbor_ids)
    ip1 = g.build(ds, params, metric="ip")
    ip2 = build_virtual_shards(ds, params, 3, metric="ip")
    assert np.array_equal(ip1.offsets, ip2.offsets) and np.array_equal(ip1.neighbor_ids, ip2.neighbor_ids)
    off, nb = oracle.build(oracle.normalize_rows(x), 16, 64, 2, 3, 1.0, 2)
    assert np.array_equal(ip1.offsets, off) and np.array_equal(ip1.neighbor_ids, nb)


@pytest.mark.gpu
def test_message_overflow_is_reported():
    """A message capacity below what a round emits is reported (DeviceError), never a
    silently wrong graph."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_02774_b200 as g
    from paper_2510_02774_b200.sharded import build_virtual_shards

    ds = generate(3000, 16, "gaussian", seed=1)
    with pytest.raises(g.DeviceError):
        build_virtual_shards(ds, g.BuildParams(S=16, R=32, T1=2, T2=2, seed=1), 2, msg_capacity=2000)


def _gpu_worker(rank, world, port, cfg, out_q, small_capacity=False, backend="gloo"):
    """One rank of a real multi-process sharded build on the GPU (ranks share cuda:0 over
    gloo: NCCL refuses two ranks on one device); the public build_sharded API."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_02774_b200 as g
        from paper_2510_02774_b200.sharded import build_sharded

        if small_capacity:  # every rank starts with 1024 message slots: forces the collective retry
            import paper_2510_02774_b200.sharded as sh

            sh.optimistic_msg_capacity = lambda rows, cap: 64
        n, dim, dist_name, S, R, T1, T2, seed = cfg
        ds = generate(n, dim, dist_name, seed=seed)
        log = []
        graph = build_sharded(ds, g.BuildParams(S=S, R=R, T1=T1, T2=T2, rho=0.6, seed=seed), report_stats=log)
        if rank == 0:
            out_q.put((graph.offsets, graph.neighbor_ids, [s.redirects for s in log]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,cfg,small", [(2, (6000, 64, "gaussian", 16, 48, 2, 5, 3), False),
                                             (3, (4000, 32, "clustered", 12, 24, 2, 4, 5), False),
                                             (2, (5000, 32, "gaussian", 16, 32, 2, 3, 7), True)])
def test_multi_process_sharded_build_gpu_bit_exact(world, cfg, small):
    """build_sharded in `world` separate processes (the exchange, the sharded pair phase and
    apply, the graph gather): the oracle's graph and per-round redirect counts.  small: the
    optimistic message capacity is overrun (emission and inbox), every rank redoes the
    build at the worst-case capacity together, and the result is still exact."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, cfg, q, small)) for r in range(world)]
    for p in procs:
        p.start()
    off, nb, red = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, dim, dist_name, S, R, T1, T2, seed = cfg
    want_off, want_nb, st = oracle.build(generate(n, dim, dist_name, seed=seed).data, S, R, T1, T2, 0.6, seed,
                                         with_stats=True)
    assert np.array_equal(off, want_off) and np.array_equal(nb, want_nb)
    assert red == st[:, 2].tolist()


def test_c5_per_rank_memory_plan_fits_one_b200():
    """SURVEY 8(d) C5 (100M x 96 over 8 B200, vectors replicated): a rank's device bytes --
    vectors, norms, its pools, the workspace at the optimistic message capacity and the
    final CSR -- fit in 180 GB (L2, and IP normalised in place); the worst-case message
    capacity (the retry path) is what would not."""
    from paper_2510_02774_b200.sharded import memory_plan

    hbm = 180e9
    for metric in ("l2", "ip"):
        p = memory_plan(100_000_000, 96, 96, 8, metric, normalize_in_place=True)
        assert p["rows"] == 12_500_000 and p["vectors"] == 100_000_000 * 96 * 4
        assert p["total"] < hbm, (metric, p["total"])
    worst = memory_plan(100_000_000, 96, 96, 8, msg_per_row=96)
    assert worst["workspace"] > memory_plan(100_000_000, 96, 96, 8)["workspace"]
    # C4 on one GPU (the bench config) and at P = 8
    assert memory_plan(10_000_000, 96, 96, 1, "ip")["total"] < hbm
    assert memory_plan(10_000_000, 96, 96, 8, "ip")["total"] < memory_plan(10_000_000, 96, 96, 1, "ip")["total"]


@pytest.mark.gpu
@pytest.mark.parametrize("small", [False, True])
def test_nccl_exchange_single_rank_gpu_bit_exact(small):
    """The NCCL code path of build_sharded (all_gather_into_tensor of the counts, all_to_all_single
    of the packed payload, device buffers) in a one-rank NCCL group on cuda:0 -- the collectives
    the 8-GPU build issues; small: through the collective capacity retry."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = (5000, 48, "gaussian", 16, 40, 2, 4, 11)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_gpu_worker, args=(0, 1, _free_port(), cfg, q, small, "nccl"))
    p.start()
    off, nb, red = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    n, dim, dist_name, S, R, T1, T2, seed = cfg
    want_off, want_nb, st = oracle.build(generate(n, dim, dist_name, seed=seed).data, S, R, T1, T2, 0.6, seed,
                                         with_stats=True)
    assert np.array_equal(off, want_off) and np.array_equal(nb, want_nb)
    assert red == st[:, 2].tolist()


@pytest.mark.gpu
def test_memory_plan_matches_device_allocation():
    """sharded.memory_plan against what a rank actually allocates (the C5 probe's accounting
    at a size one test can afford): device-generated corpus, one rank of four, init + the
    round-1 pair phase + the final CSR buffers.  Peak within 2% of the plan."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_02774_b200 as g
    from paper_2510_02774_b200.builder import _finalize_device
    from paper_2510_02774_b200.sharded import ShardedBuild, generate_device, memory_plan

    n, dim, world = 400_000, 96, 4
    params = g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    data = generate_device(n, dim, seed=1, device="cuda:0")
    again = generate_device(1000, dim, seed=1, device="cuda:0")
    assert torch.equal(again, generate_device(1000, dim, seed=1, device="cuda:0"))  # seeded
    del again
    sb = ShardedBuild(data, dim, params, 1, world, metric="ip", normalize_in_place=True)
    gen = sb.rounds()
    next(gen)  # init + round-1 emit
    offsets, nbrs, bad = _finalize_device(sb.pools)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    plan = memory_plan(n, dim, params.R, world, "ip", normalize_in_place=True)
    assert abs(peak - plan["total"]) <= 0.02 * plan["total"], (peak, plan)
    norms = data[:, :dim].norm(dim=1)
    assert torch.allclose(norms, torch.ones_like(norms), atol=1e-5)  # IP rows normalised in place
