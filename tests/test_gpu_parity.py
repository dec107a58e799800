"""GPU parity: the sm_100a kernels (through libgrnnd_b200.so) against the reference.

Bar: bit-exact.  Distances use the reference's exact fp32 arithmetic, so every
message, tombstone, pool entry, outcome counter and final graph must equal the
reference's (numba backend) bit for bit -- checked against the golden fixtures the
reference produced and against the pinned CPU oracle on larger seeded inputs.
"""

import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402

from paper_2510_02774_b200.core import generate  # noqa: E402


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_02774_b200 as pkg

    return pkg


@pytest.fixture(scope="module")
def K(g):
    from paper_2510_02774_b200 import kernels

    return kernels


def _prefix(a, cnt, cap):
    mask = (np.arange(cap)[None, :] < cnt[:, None]).ravel()
    return a[mask]


# ------------------------------------------------------------------ kernel-module surface
def test_hash_and_sqdist_bit_exact(K, golden):
    r = golden("rng")
    for (s, st, v, i), want in zip(r["hash_in"].tolist(), r["hash_out"].tolist()):
        assert int(K.hash4_u64(s, st, v, i)) == want
    d = golden("sqdist")
    for dim in (1, 3, 16, 100, 128, 960):
        a, b, want = d[f"a_{dim}"], d[f"b_{dim}"], d[f"out_{dim}"]
        for i in range(0, 64, 7):
            assert np.float32(K.sqdist(a[i], b[i])).view(np.uint32) == want[i].view(np.uint32)


def test_sample_initial_bit_exact(K, golden):
    r = golden("rng")
    for i, (n, c, s) in enumerate(r["samp_cases"].tolist()):
        out = np.full((n, c), -1, np.int32)
        flag = np.zeros(1, np.int64)
        K.sample_initial(n, c, s, out, flag)
        assert flag[0] == 0
        assert np.array_equal(out, r[f"sample_{i}"])


@pytest.mark.parametrize("name", ["gauss16", "int8", "clust4", "gauss128", "asc_u8"])
def test_gen_update_messages_bit_exact(K, golden, name):
    s = golden("stages")
    rid = s[f"{name}_rid"].copy()
    n, cap = rid.shape
    seed, stream, order = s[f"{name}_args"].tolist()
    mt = np.full(n * cap, -7, np.int32)
    mi = np.full(n * cap, -7, np.int32)
    md = np.full(n * cap, -7.0, np.float32)
    mc = np.zeros(n, np.int32)
    K.gen_update_messages(s[f"{name}_data"], rid, s[f"{name}_rd"], s[f"{name}_rc"], seed, stream, order,
                          mt, mi, md, mc)
    assert np.array_equal(mc, s[f"{name}_mc"])
    assert np.array_equal(rid, s[f"{name}_after"])  # tombstones
    assert np.array_equal(mt, s[f"{name}_mt"])  # untouched tails stay untouched too
    assert np.array_equal(mi, s[f"{name}_mi"])
    assert np.array_equal(md.view(np.uint32), s[f"{name}_md"].view(np.uint32))


@pytest.mark.parametrize("name", ["gauss16", "int8", "clust4", "gauss128", "asc_u8"])
def test_flat_group_apply_bit_exact(K, golden, name):
    s = golden("stages")
    n, cap = s[f"{name}_rid"].shape
    ft, fi, fd, fs = K.build_flat(s[f"{name}_mt"], s[f"{name}_mi"], s[f"{name}_md"], s[f"{name}_mc"], cap)
    order, starts = K.group_by_target(ft, n)
    assert np.array_equal(order, s[f"{name}_order"]) and np.array_equal(starts, s[f"{name}_starts"])
    wi = np.full((n, cap), -1, np.int32)
    wd = np.full((n, cap), np.inf, np.float32)
    wc = np.zeros(n, np.int32)
    oc = K.apply_grouped_messages(wi, wd, wc, fi, fd, order, starts)
    assert oc == tuple(s[f"{name}_outcomes"].tolist())
    assert np.array_equal(wi, s[f"{name}_wi"]) and np.array_equal(wc, s[f"{name}_wc"])
    assert np.array_equal(wd.view(np.uint32), s[f"{name}_wd"].view(np.uint32))


@pytest.mark.parametrize("name", ["gauss16", "int8", "gauss128"])
@pytest.mark.parametrize("rho", [0.6, 0.7, 1.0])
def test_reverse_messages_bit_exact(K, golden, name, rho):
    s = golden("stages")
    rid2 = s[f"{name}_rid2"]
    n, cap = rid2.shape
    mt = np.full(n * cap, -7, np.int32)
    mi = np.full(n * cap, -7, np.int32)
    md = np.full(n * cap, -7.0, np.float32)
    mc = np.zeros(n, np.int32)
    K.gen_reverse_messages(rid2, s[f"{name}_rd2"], s[f"{name}_rc2"], rho, mt, mi, md, mc)
    tag = f"{name}_rev{int(rho * 10)}"
    assert np.array_equal(mc, s[f"{tag}_mc"])
    assert np.array_equal(mt, s[f"{tag}_mt"]) and np.array_equal(mi, s[f"{tag}_mi"])
    assert np.array_equal(md, s[f"{tag}_md"])


def test_apply_trials_and_hub_bit_exact(K, golden):
    a = golden("apply")
    for t in range(int(a["ntrials"])):
        n_pools, cap = a[f"t{t}_shape"].tolist()
        order, starts = K.group_by_target(a[f"t{t}_tgt"], n_pools)
        assert np.array_equal(order, a[f"t{t}_order"])
        wi = np.full((n_pools, cap), -1, np.int32)
        wd = np.full((n_pools, cap), np.inf, np.float32)
        wc = np.zeros(n_pools, np.int32)
        oc = K.apply_grouped_messages(wi, wd, wc, a[f"t{t}_id"], a[f"t{t}_dist"], order, starts)
        assert oc == tuple(a[f"t{t}_oc"].tolist())
        assert np.array_equal(wi, a[f"t{t}_wi"]) and np.array_equal(wc, a[f"t{t}_wc"])


@pytest.mark.parametrize("m,hub_share", [(3000, 0.0), (50_000, 0.5), (40_000, 0.9)])
def test_group_by_target_stable_with_hubs(K, m, hub_share):
    """Segments of every size: register sort (<=32), smem bitonic (<=8192) and the
    counting fallback (>8192) must all give the stable counting-sort order."""
    r = np.random.default_rng(m)
    n = 700
    tgt = r.integers(0, n, m).astype(np.int32)
    tgt[r.random(m) < hub_share] = 3
    order, starts = K.group_by_target(tgt, n)
    want_o, want_s = oracle.group_by_target(tgt, n)
    assert np.array_equal(starts, want_s)
    assert np.array_equal(order, want_o)


# ------------------------------------------------------------------ fused path: whole builds
def _golden_cases(golden):
    b = golden("builds")
    return b, [list(c) for c in b["cases"]]


def test_whole_builds_bit_exact_vs_reference(g, golden):
    from test_oracle_golden import build_case_data

    b, cases = _golden_cases(golden)
    for case in cases:
        tag, n = case[0], int(case[1])
        S, R, T1, T2 = (int(x) for x in case[6:10])
        rho, seed, order = float(case[10]), int(case[11]), case[12]
        ds = g.Dataset(build_case_data(case))
        log = []
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            graph = g.build(ds, g.BuildParams(S=S, R=R, T1=T1, T2=T2, rho=rho, seed=seed), pair_order=order,
                            report_stats=log)
        assert np.array_equal(graph.offsets, b[f"{tag}_offsets"]), tag
        assert np.array_equal(graph.neighbor_ids, b[f"{tag}_nbrs"]), tag
        st = np.array([[0 if s.kind == "update" else 1, s.messages, s.redirects, s.survivors, s.reverse_attempts,
                        s.inserted, s.duplicate, s.replaced, s.rejected] for s in log], dtype=np.int64)
        assert np.array_equal(st, b[f"{tag}_stats"]), tag
        graph.validate(R)


@pytest.mark.parametrize(
    "n,dim,dist,S,R,T1,T2,seed",
    [
        (20000, 128, "gaussian", 20, 96, 2, 4, 1),   # config C1 shape, shortened schedule
        (6000, 3, "uniform", 8, 33, 2, 3, 4),        # ld padding (dim % 4 != 0), RPL=2 with a ragged row
        (3000, 24, "clustered", 16, 130, 2, 3, 9),   # R > 128: propagate bin 5, apply RPL 5
        (4000, 200, "gaussian", 12, 40, 2, 2, 3),    # two 128-dim chunks
        (2000, 1, "uniform", 4, 8, 2, 3, 2),         # D = 1, many exact ties
        (20000, 128, "gaussian", 20, 128, 4, 15, 1), # R = 128: the 96 < R <= 128 tensor-core path, full schedule
        (12000, 128, "gaussian", 20, 100, 2, 8, 6),  # R = 100
        (8000, 96, "clustered", 20, 112, 2, 6, 7),   # R = 112, D = 96
    ],
)
def test_build_bit_exact_vs_oracle(g, n, dim, dist, S, R, T1, T2, seed):
    ds = generate(n, dim, dist, seed=seed)
    graph = g.build(ds, g.BuildParams(S=S, R=R, T1=T1, T2=T2, rho=0.6, seed=seed))
    off, nb = oracle.build(ds.data, S, R, T1, T2, 0.6, seed)
    assert np.array_equal(graph.offsets, off)
    assert np.array_equal(graph.neighbor_ids, nb)


def test_integer_valued_build_bit_exact(g):
    x = np.random.default_rng(5).integers(-8, 9, (5000, 32)).astype(np.float32)
    graph = g.build(g.Dataset(x), g.BuildParams(S=10, R=32, T1=3, T2=4, seed=8))
    off, nb = oracle.build(x, 10, 32, 3, 4, 0.6, 8)
    assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)


def test_config1_full_schedule_bit_exact(g):
    """BASELINE config 1: 20K x 128 gaussian, S=20 R=96 T1=4 T2=15 rho=.6 seed 1."""
    ds = generate(20000, 128, "gaussian", seed=1)
    log = []
    graph = g.build(ds, g.BuildParams(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1), report_stats=log)
    off, nb, st = oracle.build(ds.data, 20, 96, 4, 15, 0.6, 1, with_stats=True)
    assert np.array_equal(graph.offsets, off)
    assert np.array_equal(graph.neighbor_ids, nb)
    mine = np.array([[s.messages, s.redirects, s.inserted, s.duplicate, s.replaced, s.rejected] for s in log])
    assert np.array_equal(mine, st[:, [1, 2, 5, 6, 7, 8]])


# ------------------------------------------------------------------ stepwise API (reference tests)
def test_stepwise_boundaries_and_accounting(g):
    ds = generate(2000, 8, "clustered", seed=3, clusters=3)
    params = g.BuildParams(S=16, R=16, T1=2, T2=4, rho=0.6, seed=3)
    st = g.init_neighbors(ds, params)
    ost = oracle.State(ds.data, 16, 16, 3)
    g.validate_state(st)
    for t1 in range(1, params.T1 + 1):
        for _ in range(params.T2):
            k_total = int(st.read_count.sum())
            s = g.update_round(st)
            os_ = ost.update_round(3, st.round_index)
            assert s.messages == k_total
            assert s.redirects + s.survivors == s.messages
            assert s.inserted + s.duplicate + s.replaced + s.rejected == s.messages
            assert int(st.read_count.sum()) == s.inserted
            assert [s.messages, s.redirects, s.inserted, s.duplicate, s.replaced, s.rejected] == \
                os_[[1, 2, 5, 6, 7, 8]].tolist()
            g.validate_state(st)
            ids, d, c = st.snapshot()
            oi, od, oc = ost.export()
            assert np.array_equal(c, oc) and np.array_equal(ids, oi) and np.array_equal(d, od)
        if t1 != params.T1:
            s = g.reverse_edge_sampling(st)
            ost.reverse_round(0.6)
            g.validate_state(st)
            assert s.messages == s.reverse_attempts + s.survivors
    graph = g.finalize_graph(st)
    off, nb = ost.finalize()
    assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)


def test_manual_state_traces(g):
    """test_builder.py:101-121: lone neighbour and the collinear hand trace."""
    def manual(data, read, cap):
        n = data.shape[0]
        ri = np.full((n, cap), -1, np.int32)
        rd = np.full((n, cap), np.inf, np.float32)
        rc = np.zeros(n, np.int32)
        for v, nbrs in read.items():
            for s, j in enumerate(nbrs):
                ri[v, s] = j
                dd = data[v].astype(np.float64) - data[j].astype(np.float64)
                rd[v, s] = np.float32((dd * dd).sum())
            rc[v] = len(nbrs)
        return g.BuildState.from_arrays(data, g.BuildParams(S=1, R=cap, seed=0), ri, rd, rc)

    st = manual(np.array([[0.0], [1.0], [5.0]], np.float32), {0: [1]}, 2)
    s = g.update_round(st)
    assert s.messages == 1 and s.redirects == 0
    assert st.read_ids[0, 0] == 1 and st.read_count.tolist() == [1, 0, 0]

    st = manual(np.array([[0.0], [1.0], [2.0]], np.float32), {0: [1, 2], 1: [0, 2], 2: [0, 1]}, 2)
    s = g.update_round(st)
    assert s.redirects == 2
    ri, _, rc = st.snapshot()
    assert ri[0, : rc[0]].tolist() == [1]
    assert sorted(ri[1, : rc[1]].tolist()) == [0, 2]
    assert ri[2, : rc[2]].tolist() == [1]
    g.validate_state(st)

    # reverse count guard: ceil(0.7 * 10) == 7 (test_builder.py:154-163)
    data = np.arange(24, dtype=np.float32).reshape(12, 2)
    read = {v: [(v + 1 + i) % 12 for i in range(10)] for v in range(12)}
    st = manual(data, read, 12)
    st.params = g.BuildParams(S=1, R=12, rho=0.7, seed=0)
    assert g.reverse_edge_sampling(st).reverse_attempts == 12 * 7


def test_fixed_degree_view(g):
    ds = generate(3000, 16, "gaussian", seed=2)
    params = g.BuildParams(S=8, R=24, T1=2, T2=3, seed=2)
    fixed = g.build_fixed_degree(ds, params)
    graph = g.build(ds, params)
    assert fixed.shape == (3000, 24)
    for v in range(0, 3000, 97):
        row = fixed[v]
        assert np.array_equal(row[row >= 0], graph.neighbors(v))
        assert np.all(row[len(graph.neighbors(v)):] == -1)


def test_nonfinite_rejected_on_device(g):
    x = generate(100, 4, "uniform", seed=1).data.copy()
    x[7, 2] = np.inf
    with pytest.raises(g.ParamError, match="non-finite"):
        g.build(g.Dataset(x), g.BuildParams(S=4, R=8, T1=1, T2=1))


def test_recall_parity_acceptance_corpus(g, golden):
    """criterion 03 corpus: the GPU graph equals the reference graph, hence the
    reference's recall@10 = 0.9770 at L=64 (test_output.txt:201)."""
    a = golden("acceptance10k")
    ds = generate(10000, 16, "uniform", seed=1)
    graph = g.build(ds, g.BuildParams(S=8, R=32, T1=3, T2=6, rho=0.6, seed=1))
    assert np.array_equal(graph.offsets, a["offsets"]) and np.array_equal(graph.neighbor_ids, a["nbrs"])
    q = generate(100, 16, "uniform", seed=2).data
    ids = oracle.greedy_search(graph.offsets, graph.neighbor_ids, ds.data, q, 64, 10)
    assert oracle.mean_recall(ids, a["truth"]) == pytest.approx(0.9770, abs=1e-12)


# ------------------------------------------------------------------ filtered vs exact pair phase
@pytest.mark.parametrize(
    "n,dim,dist,S,R,T1,T2,seed",
    [
        (20000, 128, "gaussian", 20, 96, 2, 3, 1),
        (4000, 200, "gaussian", 12, 40, 2, 2, 3),    # D > 128: candidates re-evaluated from global rows
        (3000, 24, "clustered", 16, 130, 2, 3, 9),
    ],
)
def test_exact_only_pair_phase_bit_exact(g, monkeypatch, n, dim, dist, S, R, T1, T2, seed):
    """The exact-only pair phase (no norms: every pair in the reference's arithmetic)
    and the default filtered phase build the same graph as the oracle."""
    ds = generate(n, dim, dist, seed=seed)
    params = g.BuildParams(S=S, R=R, T1=T1, T2=T2, rho=0.6, seed=seed)
    monkeypatch.setenv("GRNND_EXACT_PAIRS", "1")
    exact = g.build(ds, params)
    monkeypatch.delenv("GRNND_EXACT_PAIRS")
    filt = g.build(ds, params)
    off, nb = oracle.build(ds.data, S, R, T1, T2, 0.6, seed)
    assert np.array_equal(exact.offsets, off) and np.array_equal(exact.neighbor_ids, nb)
    assert np.array_equal(filt.offsets, off) and np.array_equal(filt.neighbor_ids, nb)


@pytest.mark.parametrize("force", ["1", "0"])
@pytest.mark.parametrize("dim", [16, 128, 160])
def test_filter_degenerate_ties_and_large_norms(g, monkeypatch, dim, force):
    """Filter stress: exact duplicates (d = 0 = hi, every pair a candidate: the candidate
    queue overflows into the exact sweep) and rows far from the origin (|a|^2 >> d, so the
    error band is wide) -- with the filter forced on, and with the band check (which keeps
    the exact pair phase for such data)."""
    monkeypatch.setenv("GRNND_FORCE_FILTER", force)
    r = np.random.default_rng(dim)
    base = r.standard_normal((60, dim)).astype(np.float32)
    dup = base[r.integers(0, 60, 3000)]
    far = (r.standard_normal((3000, dim)) * 0.05 + 300.0).astype(np.float32)
    for x in (dup, far):
        graph = g.build(g.Dataset(x), g.BuildParams(S=16, R=96, T1=2, T2=3, rho=0.6, seed=4))
        off, nb = oracle.build(x, 16, 96, 2, 3, 0.6, 4)
        assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)


def test_filtered_phase_from_the_first_round(g, monkeypatch):
    """Filtered pair phase from round 1 (random pools: most pairs are candidates, the
    tensor-core path's candidate queues overflow into exact sweeps) -- same graph."""
    monkeypatch.setenv("GRNND_EXACT_FIRST_ROUNDS", "0")
    for n, dim, dist, R, seed in [(20000, 128, "gaussian", 96, 1), (6000, 100, "clustered", 64, 2),
                                  (5000, 128, "gaussian", 40, 3)]:
        ds = generate(n, dim, dist, seed=seed)
        graph = g.build(ds, g.BuildParams(S=20 if R > 20 else 16, R=R, T1=2, T2=4, rho=0.6, seed=seed))
        off, nb = oracle.build(ds.data, 20 if R > 20 else 16, R, 2, 4, 0.6, seed)
        assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb), (n, dim, dist, R)


# ------------------------------------------------------------------ direct fixture tests (reference outputs)
def test_init_dists_and_merge_messages_bit_exact(K, golden):
    """kernels.init_dists (_numba_kernels.py:118-122) and gen_merge_messages (:236-250) on
    the reference's own stage fixtures."""
    s = golden("stages")
    for name in ("gauss16", "int8", "clust4", "gauss128"):
        data, rid, rd, rc = s[f"{name}_data"], s[f"{name}_rid"], s[f"{name}_rd"], s[f"{name}_rc"]
        n, cap = rid.shape
        live = np.arange(cap)[None, :] < rc[:, None]
        ids = np.where(live, rid, (np.arange(n, dtype=np.int32)[:, None] + 1) % n).astype(np.int32)
        out = np.zeros((n, cap), np.float32)
        K.init_dists(data, ids, out)
        # the reference's pools store its own _sqdist of (v, id): equal bits on the live prefix
        assert np.array_equal(out[live].view(np.uint32), rd[live].view(np.uint32)), name
        assert np.array_equal(out.view(np.uint32), oracle.init_dists(data, ids).view(np.uint32))
        mt = np.full(n * cap, -7, np.int32)
        mi = np.full(n * cap, -7, np.int32)
        md = np.full(n * cap, -7.0, np.float32)
        mc = np.zeros(n, np.int32)
        K.gen_merge_messages(rid, rd, rc, mt, mi, md, mc)
        wt, wi, wd, wc = oracle.gen_merge_messages(rid, rd, rc)
        assert np.array_equal(mc, wc), name
        m = (np.arange(cap)[None, :] < mc[:, None]).ravel()
        assert np.array_equal(mt[m], wt[m]) and np.array_equal(mi[m], wi[m]) and np.array_equal(md[m], wd[m])
        assert np.all(mt[~m] == -7)  # untouched tails


def test_message_capacity_overflow_rebuilds_exactly(g, monkeypatch):
    """build() starts with an optimistic message capacity; a round that outgrows it is
    detected on the device (GRNND_ST_LOST) and the build is redone at the worst-case
    capacity -- the graph is still the oracle's."""
    from paper_2510_02774_b200 import builder as B

    calls = []

    def tiny(rows, cap):
        calls.append(rows)
        return 300

    monkeypatch.setattr(B, "optimistic_msg_capacity", tiny)
    ds = generate(3000, 32, "gaussian", seed=4)
    graph = g.build(ds, g.BuildParams(S=12, R=24, T1=2, T2=3, rho=0.6, seed=4))
    off, nb = oracle.build(ds.data, 12, 24, 2, 3, 0.6, 4)
    assert calls and np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)


@pytest.mark.parametrize("dim,R", [(960, 96), (300, 48), (129, 24)])
def test_tensor_core_multichunk_bit_exact(g, monkeypatch, dim, R):
    """D > 128 on the tensor cores (tc3 MULTI: 128-dim chunks accumulated in TMEM, exact
    chains from global rows), from round 1 (queue overflows -> exact sweeps) and after the
    exact first rounds: the oracle's graph bit for bit."""
    ds = generate(3000, dim, "gaussian", seed=dim)
    off, nb = oracle.build(ds.data, 16, R, 2, 4, 0.6, 5)
    for first in ("0", "3"):
        monkeypatch.setenv("GRNND_EXACT_FIRST_ROUNDS", first)
        graph = g.build(ds, g.BuildParams(S=16, R=R, T1=2, T2=4, rho=0.6, seed=5))
        assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb), (dim, R, first)


def test_band_check_picks_the_pair_phase(g):
    """The plain TF32 filter is kept for data whose band is narrow (gaussian: band /
    distance ~1%); data far from the origin relative to its neighbour distances (clustered,
    shifted) keep the exact pair phase: the pools report the measured ratio; every graph
    equals the oracle's."""
    from paper_2510_02774_b200 import builder as B

    for dist, shift, want in (("gaussian", 0.0, 1), ("clustered", 0.0, 0), ("gaussian", 50.0, 0)):
        ds = generate(6000, 64, dist, seed=2)
        x = (ds.data + np.float32(shift)).astype(np.float32)
        st = g.init_neighbors(g.Dataset(x), g.BuildParams(S=16, R=48, T1=2, T2=5, rho=0.6, seed=2))
        B.run_rounds(st)
        assert st.pools._filter_ok == want, (dist, shift, st.pools.band_ratio)
        graph = g.finalize_graph(st)
        off, nb = oracle.build(x, 16, 48, 2, 5, 0.6, 2)
        assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb), (dist, shift)


@pytest.mark.parametrize("mode", ["2", "0"])
@pytest.mark.parametrize("dist,shift,R", [("clustered", 0.0, 96), ("gaussian", 300.0, 40), ("gaussian", 0.0, 24),
                                          ("uniform", 0.0, 64)])
def test_split_tf32_filter_bit_exact(g, monkeypatch, dist, shift, R, mode):
    """The split-TF32 Gram (hi*hi + hi*lo + lo*hi, band 2^-15 (|a|^2 + |b|^2)) and the exact
    pair phase forced on near- and far-from-origin data: the oracle's graph bit for bit."""
    monkeypatch.setenv("GRNND_FORCE_FILTER", mode)
    ds = generate(5000, 128, dist, seed=7)
    x = (ds.data + np.float32(shift)).astype(np.float32)
    graph = g.build(g.Dataset(x), g.BuildParams(S=16, R=R, T1=2, T2=5, rho=0.6, seed=7))
    off, nb = oracle.build(x, 16, R, 2, 5, 0.6, 7)
    assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)


def _tied_pools(n, cap, seed):
    """Duplicate-free pools with heavily tied distances (four values), random counts."""
    rng = np.random.default_rng(seed)
    ids = np.full((n, cap), -1, np.int32)
    dists = np.zeros((n, cap), np.float32)
    counts = rng.integers(0, cap + 1, n).astype(np.int32)
    counts[:4] = [0, 1, cap, cap]
    for v in range(n):
        k = int(counts[v])
        cand = rng.permutation(np.setdiff1d(np.arange(n), [v]))[:k]
        ids[v, :k] = cand
        dists[v, :k] = rng.integers(0, 4, k).astype(np.float32) * np.float32(0.25)
    return ids, dists, counts


@pytest.mark.parametrize("cap", [8, 33, 96, 130, 256])
def test_reverse_selection_and_finalize_with_ties(K, g, cap):
    """The warp bitonic (dist, id) sort of gen_reverse_messages (_numba_kernels.py:195-233)
    and finalize_graph (builder.py:342-362) against the oracle on tie-heavy rows, every
    keys-per-lane width (cap 8 ... 256)."""
    n = 300
    ids, dists, counts = _tied_pools(n, cap, cap)
    for rho in (0.6, 1.0):
        mt = np.full(n * cap, -7, np.int32)
        mi = np.full(n * cap, -7, np.int32)
        md = np.full(n * cap, -7.0, np.float32)
        mc = np.zeros(n, np.int32)
        K.gen_reverse_messages(ids, dists, counts, rho, mt, mi, md, mc)
        wt, wi, wd, wc = oracle.gen_reverse_messages(ids, dists, counts, rho)
        assert np.array_equal(mc, wc)
        m = (np.arange(cap)[None, :] < mc[:, None]).ravel()
        assert np.array_equal(mt[m], wt[m]) and np.array_equal(mi[m], wi[m])
        assert np.array_equal(md[m].view(np.uint32), wd[m].view(np.uint32))
    data = generate(n, 4, "gaussian", seed=1).data
    st = g.BuildState.from_arrays(data, g.BuildParams(S=1, R=cap, T1=1, T2=1), ids, dists, counts)
    graph = g.finalize_graph(st)
    off, nb = oracle.finalize(ids, dists, counts)
    assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)


@pytest.mark.parametrize("defect,msg", [("dup", "duplicate"), ("self", "self-loop"), ("range", "out of range")])
def test_finalize_flags_invalid_rows_on_device(g, defect, msg):
    """Graph.validate's checks (core.py:171-201) run inside the finalize kernel."""
    n, cap = 200, 40
    ids, dists, counts = _tied_pools(n, cap, 5)
    v = 17
    counts[v] = 30
    ids[v, :30] = np.setdiff1d(np.arange(n), [v])[:30]
    if defect == "dup":
        ids[v, 29] = ids[v, 3]
    elif defect == "self":
        ids[v, 12] = v
    else:
        ids[v, 5] = n + 3
    data = generate(n, 4, "gaussian", seed=1).data
    st = g.BuildState.from_arrays(data, g.BuildParams(S=1, R=cap, T1=1, T2=1), ids, dists, counts)
    with pytest.raises(g.ParamError, match=msg):
        g.finalize_graph(st)


@pytest.mark.parametrize("dim,cap", [(3, 40), (100, 96), (128, 130), (960, 33)])
def test_init_dists_wide_rows_bit_exact(K, dim, cap):
    """init_dists (_numba_kernels.py:118-122) with more than 32 neighbours per row (several
    row groups) and partial 128-dim chunks."""
    n = 500
    data = generate(n, dim, "gaussian", seed=dim).data
    rng = np.random.default_rng(cap)
    ids = rng.integers(0, n, (n, cap)).astype(np.int32)
    out = np.zeros((n, cap), np.float32)
    K.init_dists(data, ids, out)
    assert np.array_equal(out.view(np.uint32), oracle.init_dists(data, ids).view(np.uint32))
