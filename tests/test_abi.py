"""CPU checks of the boundary: libgrnnd_b200.so loads, exports every function
include/grnnd_b200.h declares, the ctypes signatures cover them, and the host-side
API mirrors the reference's (params, errors, scalar specs).  No kernel launches."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "grnnd_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*|unsigned long long)\s*(grnnd_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2510_02774_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED, f"{name} has no ctypes signature"


def test_library_is_sm100a_only():
    import subprocess

    from paper_2510_02774_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_workspace_size_is_monotone():
    from paper_2510_02774_b200 import _lib

    a = _lib.lib.grnnd_workspace_bytes(1000, 32, 1000 * 32)
    b = _lib.lib.grnnd_workspace_bytes(2000, 32, 2000 * 32)
    assert 0 < a < b


def test_device_required_without_cuda():
    import torch

    import paper_2510_02774_b200 as g

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    ds = g.generate(50, 4, "uniform", seed=1)
    with pytest.raises(g.DeviceError):
        g.build(ds, g.BuildParams(S=4, R=8, T1=1, T2=1))


def test_params_bounds_match_reference_messages():
    from paper_2510_02774_b200 import BuildParams, ParamError, validate_params

    validate_params(BuildParams(S=8, R=32, T1=3, T2=6, rho=0.6), 10000)
    for kw, msg in [(dict(S=40, R=32), "S <= R"), (dict(rho=0.0), "rho"), (dict(rho=1.5), "rho"),
                    (dict(S=0), "S >= 1"), (dict(T1=0), "T1 >= 1"), (dict(T2=0), "T2 >= 1"),
                    (dict(workers=0), "workers >= 1")]:
        with pytest.raises(ParamError, match=re.escape(msg)):
            validate_params(BuildParams(**kw), 10000)
    with pytest.raises(ParamError, match="R <= N-1"):
        validate_params(BuildParams(S=8, R=32), 20)


def test_dataset_validation():
    from paper_2510_02774_b200 import Dataset, ParamError

    Dataset(np.zeros((4, 3), np.float32)).validate()
    with pytest.raises(ParamError):
        Dataset(np.zeros(12, np.float32))
    bad = np.zeros((4, 3), np.float32)
    bad[1, 2] = np.nan
    with pytest.raises(ParamError, match="non-finite"):
        Dataset(bad).validate()
    with pytest.raises(ParamError, match="N >= 2"):
        Dataset(np.zeros((1, 3), np.float32)).validate()
    assert Dataset(np.arange(6, dtype=np.float64).reshape(2, 3)).data.dtype == np.float32


def test_scalar_specs():
    from paper_2510_02774_b200 import SelfInsert, cooperative_insert, rng_redirect_check

    assert tuple(rng_redirect_check(1.0, 2.0, 1.5)) == (1, 0)
    assert rng_redirect_check(1.0, 2.0, 2.0) is None
    assert rng_redirect_check(1.0, 1.0, 1.0) is None
    assert tuple(rng_redirect_check(2.0, 2.0, 1.0)) == (1, 0)
    assert tuple(rng_redirect_check(3.0, 2.0, 1.0)) == (0, 1)
    ids = np.full(3, -1, np.int32)
    d = np.full(3, np.inf, np.float32)
    c = 0
    for nid, dd in [(1, 7.0), (2, 7.0), (3, 1.0)]:
        _, c = cooperative_insert(0, ids, d, c, nid, dd)
    st, _ = cooperative_insert(0, ids, d, c, 4, 2.0)
    assert st == "replaced" and ids.tolist() == [4, 2, 3]
    with pytest.raises(SelfInsert):
        cooperative_insert(5, ids, d, c, 5, 1.0)


def test_effective_params_clamps():
    import warnings

    from paper_2510_02774_b200 import BuildParams, effective_params

    with pytest.warns(UserWarning, match="clamping"):
        p = effective_params(BuildParams(S=8, R=32), 5)
    assert (p.S, p.R) == (4, 4)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        q = effective_params(BuildParams(S=4, R=4), 5)
    assert (q.S, q.R) == (4, 4)


def test_graph_validate():
    from paper_2510_02774_b200 import Graph, ParamError

    Graph(3, np.array([0, 1, 2, 3]), np.array([1, 2, 0])).validate(1)
    with pytest.raises(ParamError, match="self-loop"):
        Graph(2, np.array([0, 1, 1]), np.array([0])).validate()
    with pytest.raises(ParamError, match="duplicate"):
        Graph(3, np.array([0, 2, 2, 2]), np.array([1, 1])).validate()
    with pytest.raises(ParamError, match="degree"):
        Graph(3, np.array([0, 2, 2, 2]), np.array([1, 2])).validate(1)


def test_generate_matches_reference_recipe():
    from paper_2510_02774_b200 import generate

    a = generate(100, 8, "gaussian", seed=1).data
    assert np.array_equal(a, np.random.default_rng(1).standard_normal((100, 8), dtype=np.float32))
