"""File formats (fvecs / ivecs / GRND v1) and the CLI.

Format tests run on CPU: byte-exact layouts (the reference's hand-computed golden bytes,
test_io.py:28-34, 108-121), round trips, malformed-file rejection.  The CLI's build /
search / bench commands and the device graph writer need the GPU (-m gpu).
"""

import struct

import numpy as np
import pytest

from paper_2510_02774_b200.core import Dataset, Graph, generate
from paper_2510_02774_b200.errors import FormatError, ParamError
from paper_2510_02774_b200.io import read_fvecs, read_graph, read_ivecs, write_fvecs, write_graph, write_ivecs

# the reference's hand-computed 3-vertex path graph 0-1, 1-2 with R=2 (test_io.py:28-34)
GOLDEN_PATH_GRAPH = bytes.fromhex(
    "47524e4401000000030000000000000002000000"
    "00000000000000000100000000000000030000000000000004000000000000000"
    "1000000"
    "00000000020000000"
    "1000000"
)


def test_fvecs_bit_layout(tmp_path):
    raw = bytes.fromhex("02000000" "0000803f" "00000040")  # [dim=2][1.0f][2.0f]
    p = tmp_path / "one.fvecs"
    p.write_bytes(raw)
    ds = read_fvecs(p)
    assert ds.num_points == 1 and ds.dim == 2 and ds.data.tolist() == [[1.0, 2.0]]
    out = tmp_path / "copy.fvecs"
    write_fvecs(ds, out)
    assert out.read_bytes() == raw


def test_round_trips(tmp_path):
    r = np.random.default_rng(3)
    for n, d in [(1, 1), (7, 3), (100, 128)]:
        x = r.standard_normal((n, d)).astype(np.float32)
        write_fvecs(x, tmp_path / "a.fvecs")
        assert np.array_equal(read_fvecs(tmp_path / "a.fvecs").data, x)
        ids = r.integers(0, 1 << 30, (n, d)).astype(np.int32)
        write_ivecs(ids, tmp_path / "a.ivecs")
        assert np.array_equal(read_ivecs(tmp_path / "a.ivecs"), ids)
    (tmp_path / "e.fvecs").write_bytes(b"")
    assert read_fvecs(tmp_path / "e.fvecs").num_points == 0
    assert read_ivecs(tmp_path / "e.fvecs").shape == (0, 0)


@pytest.mark.parametrize("raw,msg", [
    (b"\x02\x00", "truncated dim"),
    (struct.pack("<i", 0), "non-positive dim"),
    (struct.pack("<i", -3) + b"\x00" * 12, "non-positive dim"),
    (struct.pack("<iff", 2, 1.0, 2.0) + b"\x00", "truncated record or trailing"),
    (struct.pack("<iffiff", 2, 1.0, 2.0, 3, 1.0, 2.0), "inconsistent dim"),
    (struct.pack("<iffif", 2, 1.0, 2.0, 1, 1.0), "truncated record or trailing"),
    (struct.pack("<iff", 2, 1.0, float("nan")), "non-finite"),
    (struct.pack("<iff", 2, float("inf"), 0.0), "non-finite"),
])
def test_malformed_fvecs(tmp_path, raw, msg):
    p = tmp_path / "bad.fvecs"
    p.write_bytes(raw)
    with pytest.raises(FormatError, match=msg):
        read_fvecs(p)


def test_golden_path_graph_bytes(tmp_path):
    g = Graph(num_vertices=3, offsets=np.array([0, 1, 3, 4]), neighbor_ids=np.array([1, 0, 2, 1]),
              max_degree_bound=2)
    p = tmp_path / "path.grnd"
    write_graph(g, p)
    assert p.read_bytes() == GOLDEN_PATH_GRAPH
    back = read_graph(p)
    assert back.num_vertices == 3 and back.neighbors(1).tolist() == [0, 2] and back.max_degree_bound == 2
    e = Graph(num_vertices=0, offsets=np.zeros(1), neighbor_ids=np.zeros(0))
    write_graph(e, tmp_path / "e.grnd")
    assert (tmp_path / "e.grnd").stat().st_size == 20 + 8
    assert read_graph(tmp_path / "e.grnd").num_vertices == 0


def test_graph_bytes_equal_reference_acceptance(tmp_path, golden):
    """A full reference-built graph (acceptance corpus) written and re-read."""
    a = golden("acceptance10k")
    g = Graph(10000, a["offsets"], a["nbrs"], 32)
    write_graph(g, tmp_path / "acc.grnd")
    raw = (tmp_path / "acc.grnd").read_bytes()
    assert raw[:20] == struct.pack("<4sIQI", b"GRND", 1, 10000, 32)
    assert raw[20:20 + 8 * 10001] == a["offsets"].astype("<u8").tobytes()
    assert raw[20 + 8 * 10001:] == a["nbrs"].astype("<u4").tobytes()
    back = read_graph(tmp_path / "acc.grnd")
    assert np.array_equal(back.offsets, a["offsets"]) and np.array_equal(back.neighbor_ids, a["nbrs"])


def test_malformed_graphs(tmp_path):
    p = tmp_path / "g.grnd"
    good = GOLDEN_PATH_GRAPH
    cases = [(good[:10], "truncated header"), (b"XXXX" + good[4:], "bad magic"),
             (good[:4] + struct.pack("<I", 2) + good[8:], "unsupported version"),
             (good[:30], "truncated offsets"), (good + b"\x00", "payload size"),
             (good[:-4] + struct.pack("<I", 7), "out of range")]
    for raw, msg in cases:
        p.write_bytes(raw)
        with pytest.raises(FormatError, match=msg):
            read_graph(p)
    # self loop -> validate fails -> FormatError
    bad = good[:-4] + struct.pack("<I", 2)
    p.write_bytes(bad)
    with pytest.raises(FormatError):
        read_graph(p)


def test_cli_gen_and_usage(tmp_path, capsys):
    from paper_2510_02774_b200.cli import main

    out = tmp_path / "g.fvecs"
    assert main(["gen", "--n", "50", "--dim", "8", "--dist", "gaussian", "--seed", "4", "--output", str(out)]) == 0
    assert np.array_equal(read_fvecs(out).data, generate(50, 8, "gaussian", seed=4).data)
    assert "seed=4" in capsys.readouterr().err
    with pytest.raises(SystemExit) as e:
        main(["build"])  # missing required flags: usage error, exit 1
    assert e.value.code == 1
    assert main(["search", "--graph", str(tmp_path / "missing.grnd"), "--base", str(out),
                 "--queries", str(out)]) == 2


# ------------------------------------------------------------------ GPU: CLI build/search, device writer
@pytest.mark.gpu
def test_cli_build_search_bench(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle
    from paper_2510_02774_b200.cli import main

    base, q = tmp_path / "b.fvecs", tmp_path / "q.fvecs"
    write_fvecs(generate(3000, 16, "uniform", seed=1), base)
    write_fvecs(generate(50, 16, "uniform", seed=2), q)
    capsys.readouterr()
    assert main(["build", "--input", str(base), "--output", str(tmp_path / "g.grnd"), "--S", "8", "--R", "16",
                 "--T1", "2", "--T2", "3", "--seed", "5"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "algo,n,dim,build_seconds,mean_degree,max_degree,rejected_inserts,seed"
    assert lines[1].startswith("grnnd,3000,16,") and lines[1].endswith(",5")
    g = read_graph(tmp_path / "g.grnd")
    off, nb = oracle.build(read_fvecs(base).data, 8, 16, 2, 3, 0.6, 5)
    assert np.array_equal(g.offsets, off) and np.array_equal(g.neighbor_ids, nb)
    assert main(["search", "--graph", str(tmp_path / "g.grnd"), "--base", str(base), "--queries", str(q),
                 "--L", "16", "--L", "32"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "L,recall@k,QPS" and [r.split(",")[0] for r in rows[1:]] == ["16", "32"]
    assert main(["bench", "--n", "2000", "--T1", "1", "2", "--queries", "20"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "T1,T2,rho,build_seconds,recall@10,QPS" and len(rows) == 3
    assert main(["build", "--input", str(base), "--output", str(tmp_path / "s.grnd"), "--algo", "seq"]) == 1


@pytest.mark.gpu
def test_device_graph_writer_streams_identical_bytes(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_02774_b200 as gpkg
    from paper_2510_02774_b200 import io as gio
    from paper_2510_02774_b200.builder import DeviceBuild, upload

    ds = generate(5000, 32, "gaussian", seed=3)
    params = gpkg.BuildParams(S=12, R=24, T1=2, T2=2, seed=3)
    eng = DeviceBuild(upload(ds.data, torch.device("cuda", 0)), 32, params)
    offsets, nbrs, bad, fail = eng.run()
    old = gio._CHUNK
    gio._CHUNK = 4096  # many chunks
    try:
        gio.write_graph_device(offsets, nbrs, 5000, 24, tmp_path / "d.grnd")
    finally:
        gio._CHUNK = old
    host = gpkg.build(ds, params)
    write_graph(host, tmp_path / "h.grnd")
    assert (tmp_path / "d.grnd").read_bytes() == (tmp_path / "h.grnd").read_bytes()
    with pytest.raises(ParamError):
        gio.write_graph_device(offsets[:-1], nbrs, 5000, 24, tmp_path / "x.grnd")
    assert Dataset(ds.data).num_points == 5000
