"""Pin the CPU oracle to the reference: every check compares oracle/ (C restatement)
with fixtures the reference itself produced (tests/golden/make_golden.py), plus the
known-answer values of SURVEY.md A.1 and pkg/test_output.txt.  CPU only."""

import numpy as np
import pytest

import oracle

from paper_2510_02774_b200.core import generate

M64 = (1 << 64) - 1


def test_hash4_known_answers(golden):
    g = golden("rng")
    for (s, st, v, i), want in zip(g["hash_in"].tolist(), g["hash_out"].tolist()):
        assert oracle.hash4(s, st, v, i) == want
    # SURVEY.md A.1 (computed from rng.py)
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF
    assert oracle.hash4(0, 0, 0, 0) == 0x2130748AAAC80268
    assert oracle.hash4(1, 2, 3, 4) == 0xD55CCD4AEB3CCAFB
    assert oracle.hash4(M64, 7, 1, 1) == 0xE6A51E8A5F992D77
    assert oracle.hash4(123456789, 1, 42, 7) == 0xD7E73A70B6644C82


def test_fisher_yates_known_answers(golden):
    g = golden("rng")
    for (k, seed, stream, v), row in zip(g["perm_cases"].tolist(), g["perms"]):
        assert np.array_equal(oracle.fisher_yates_perm(k, seed, stream, v), row[:k])
    assert oracle.fisher_yates_perm(16, 1, 2, 3).tolist() == [0, 4, 9, 12, 13, 11, 8, 14, 3, 1, 2, 15, 7, 5, 6, 10]


def test_sample_initial_matches_reference(golden):
    g = golden("rng")
    for i, (n, c, s) in enumerate(g["samp_cases"].tolist()):
        out, fail = oracle.sample_initial(n, c, s)
        assert fail == 0
        assert np.array_equal(out, g[f"sample_{i}"])
    out, _ = oracle.sample_initial(1_000_000, 20, 1)
    assert out[0].tolist() == [971414, 154915, 429959, 215320, 322067, 343532, 73341, 957420, 592606, 168853,
                               195043, 800193, 240050, 868530, 493393, 527743, 818969, 337031, 502118, 137681]


def test_sqdist_bit_exact(golden):
    g = golden("sqdist")
    for d in (1, 3, 16, 100, 128, 960):
        got = oracle.sqdist_batch(g[f"a_{d}"], g[f"b_{d}"])
        assert np.array_equal(got.view(np.uint32), g[f"out_{d}"].view(np.uint32)), d


def test_golden_distance_constant():
    # test_metric.py:12-13: GOLDEN_SQ from default_rng(20240612) uniform(-1, 1), 128-d
    r = np.random.default_rng(20240612)
    a = r.uniform(-1.0, 1.0, 128).astype(np.float32)
    b = r.uniform(-1.0, 1.0, 128).astype(np.float32)
    assert float(oracle.sqdist(a, b)) == pytest.approx(70.45210050999715, rel=1e-5)


def _prefix_equal(a, b, cnt, cap):
    mask = (np.arange(cap)[None, :] < cnt[:, None]).ravel()
    return np.array_equal(a[mask], b[mask])


@pytest.fixture(scope="module")
def stages(golden):
    return golden("stages")


@pytest.mark.parametrize("name", ["gauss16", "int8", "clust4", "gauss128", "asc_u8"])
def test_update_messages_match_reference(stages, name):
    g = stages
    rid = g[f"{name}_rid"].copy()
    seed, stream, order = g[f"{name}_args"].tolist()
    mt, mi, md, mc = oracle.gen_update_messages(g[f"{name}_data"], rid, g[f"{name}_rd"], g[f"{name}_rc"],
                                                seed, stream, order)
    cap = rid.shape[1]
    assert np.array_equal(mc, g[f"{name}_mc"])
    assert np.array_equal(rid, g[f"{name}_after"])
    assert _prefix_equal(mt, g[f"{name}_mt"], mc, cap)
    assert _prefix_equal(mi, g[f"{name}_mi"], mc, cap)
    assert _prefix_equal(md.view(np.uint32), g[f"{name}_md"].view(np.uint32), mc, cap)


@pytest.mark.parametrize("name", ["gauss16", "int8", "clust4", "gauss128", "asc_u8"])
def test_flat_group_apply_match_reference(stages, name):
    g = stages
    n, cap = g[f"{name}_rid"].shape
    ft, fi, fd, fs = oracle.build_flat(g[f"{name}_mt"], g[f"{name}_mi"], g[f"{name}_md"], g[f"{name}_mc"], cap)
    order, starts = oracle.group_by_target(ft, n)
    assert np.array_equal(order, g[f"{name}_order"])
    assert np.array_equal(starts, g[f"{name}_starts"])
    wi = np.full((n, cap), -1, np.int32)
    wd = np.full((n, cap), np.inf, np.float32)
    wc = np.zeros(n, np.int32)
    oc = oracle.apply_grouped_messages(wi, wd, wc, fi, fd, order, starts)
    assert oc == tuple(g[f"{name}_outcomes"].tolist())
    assert np.array_equal(wi, g[f"{name}_wi"])
    assert np.array_equal(wc, g[f"{name}_wc"])
    assert np.array_equal(wd.view(np.uint32), g[f"{name}_wd"].view(np.uint32))


@pytest.mark.parametrize("name", ["gauss16", "int8", "clust4", "gauss128", "asc_u8"])
@pytest.mark.parametrize("rho", [0.6, 0.7, 1.0])
def test_reverse_messages_match_reference(stages, name, rho):
    g = stages
    cap = g[f"{name}_rid2"].shape[1]
    mt, mi, md, mc = oracle.gen_reverse_messages(g[f"{name}_rid2"], g[f"{name}_rd2"], g[f"{name}_rc2"], rho)
    tag = f"{name}_rev{int(rho * 10)}"
    assert np.array_equal(mc, g[f"{tag}_mc"])
    assert _prefix_equal(mt, g[f"{tag}_mt"], mc, cap)
    assert _prefix_equal(mi, g[f"{tag}_mi"], mc, cap)
    assert _prefix_equal(md, g[f"{tag}_md"], mc, cap)


def test_apply_trials_match_reference(golden):
    g = golden("apply")
    for t in range(int(g["ntrials"])):
        n_pools, cap = g[f"t{t}_shape"].tolist()
        order, starts = oracle.group_by_target(g[f"t{t}_tgt"], n_pools)
        assert np.array_equal(order, g[f"t{t}_order"])
        wi = np.full((n_pools, cap), -1, np.int32)
        wd = np.full((n_pools, cap), np.inf, np.float32)
        wc = np.zeros(n_pools, np.int32)
        oc = oracle.apply_grouped_messages(wi, wd, wc, g[f"t{t}_id"], g[f"t{t}_dist"], order, starts)
        assert oc == tuple(g[f"t{t}_oc"].tolist())
        assert np.array_equal(wi, g[f"t{t}_wi"]) and np.array_equal(wc, g[f"t{t}_wc"])


def build_case_data(case):
    tag, n, dim, distn, dseed, cl = case[:6]
    return generate(int(n), int(dim), distn, seed=int(dseed), clusters=int(cl)).data


def build_case_params(case):
    S, R, T1, T2 = (int(x) for x in case[6:10])
    rho, bseed, order = float(case[10]), int(case[11]), case[12]
    n = int(case[1])
    if S > n - 1 or R > n - 1:  # effective_params clamp (builder.py:209-218)
        R = min(R, n - 1)
        S = min(S, R)
    return S, R, T1, T2, rho, bseed, 0 if order == "disordered" else 1


def test_whole_builds_match_reference(golden):
    g = golden("builds")
    for case in g["cases"]:
        tag = case[0]
        data = build_case_data(case)
        S, R, T1, T2, rho, seed, order = build_case_params(case)
        off, nb, st = oracle.build(data, S, R, T1, T2, rho, seed, order, with_stats=True)
        assert np.array_equal(off, g[f"{tag}_offsets"]), tag
        assert np.array_equal(nb, g[f"{tag}_nbrs"]), tag
        assert np.array_equal(st, g[f"{tag}_stats"]), tag


def test_acceptance_recall_matches_reference(golden):
    """criterion 03 corpus (test_acceptance.py:68-73, test_output.txt:201): recall 0.9770."""
    g = golden("acceptance10k")
    data = generate(10000, 16, "uniform", seed=1).data
    q = generate(100, 16, "uniform", seed=2).data
    truth = oracle.brute_force_knn(data, q, 10)
    assert np.array_equal(truth, g["truth"])
    off, nb = oracle.build(data, 8, 32, 3, 6, 0.6, 1)
    assert np.array_equal(off, g["offsets"]) and np.array_equal(nb, g["nbrs"])
    ids = oracle.greedy_search(off, nb, data, q, 64, 10)
    assert np.array_equal(ids, g["search_ids"])
    assert oracle.mean_recall(ids, truth) == pytest.approx(0.9770, abs=1e-12)
