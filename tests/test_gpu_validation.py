"""Validation-library runs (-m gpu): the tensor-core pre-screen's error bound, checked on
every screened pair of whole builds (libgrnnd_b200_tcv.so, built with -DGRNND_TC_VALIDATE
by the same Makefile), and the graphs of those builds against the oracle.

DESIGN.md 2 derives the bound |d~ - d| <= TC_EPS (|a|^2 + |b|^2) from TF32 truncation and
fp32 accumulation; the tensor core's internal accumulation order is not documented, so
this is the empirical check that the hardware meets it (expected: 0 violations).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402

from paper_2510_02774_b200.core import generate  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
TCV = ROOT / "paper_2510_02774_b200" / "_build" / "libgrnnd_b200_tcv.so"


def run_tcv(*args, force="1"):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    assert TCV.exists(), "validation library missing: build() compiles it"
    env = dict(os.environ, GRNND_B200_LIB=str(TCV), GRNND_FORCE_FILTER=force)  # the filter even where its band is wide
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "tcv_run.py"), *map(str, args)], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("n,dim,R,T1,T2,dist", [
    (20000, 128, 96, 4, 15, "gaussian"),   # BASELINE config 1, full schedule (tc3 path)
    (20000, 128, 128, 2, 6, "gaussian"),   # 96 < R <= 128: the tc_pairs path
    (8000, 100, 112, 2, 5, "clustered"),
    (6000, 64, 40, 2, 5, "uniform"),
    (4000, 960, 96, 2, 5, "gaussian"),     # D > 128: chunked Gram accumulated over K = 960
])
def test_tensor_core_bound_holds_and_graph_exact(n, dim, R, T1, T2, dist):
    r = run_tcv(n, dim, R, T1, T2, dist)
    assert r["lib"].endswith("libgrnnd_b200_tcv.so")
    assert r["checked"] > 0
    assert r["violations"] == 0, r
    assert r["max_ratio"] < 1.0
    off, nb = oracle.build(generate(n, dim, dist, seed=1).data, 20, R, T1, T2, 0.6, 1)
    assert np.array_equal(np.array(r["offsets"]), off) and np.array_equal(np.array(r["nbrs"]), nb)


@pytest.mark.parametrize("n,dim,R,T1,T2,dist", [
    (8000, 128, 96, 2, 6, "clustered"),   # far from the origin: the split-TF32 Gram's case
    (6000, 64, 40, 2, 5, "gaussian"),
])
def test_split_tf32_bound_holds_and_graph_exact(n, dim, R, T1, T2, dist):
    """The split-TF32 Gram's error against its band 2^-15 (|a|^2 + |b|^2), on every screened
    pair: 0 violations, the largest error well inside the band."""
    r = run_tcv(n, dim, R, T1, T2, dist, force="2")
    assert r["checked"] > 0
    assert r["violations"] == 0, r
    assert r["max_ratio"] < 1.0
    off, nb = oracle.build(generate(n, dim, dist, seed=1).data, 20, R, T1, T2, 0.6, 1)
    assert np.array_equal(np.array(r["offsets"]), off) and np.array_equal(np.array(r["nbrs"]), nb)
