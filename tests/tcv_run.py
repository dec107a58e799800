"""Subprocess body of tests/test_gpu_validation.py (run with GRNND_B200_LIB pointing at the
validation library): a build with per-round stats; prints one JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_02774_b200 as g  # noqa: E402
from paper_2510_02774_b200 import _lib  # noqa: E402
from paper_2510_02774_b200.builder import DeviceBuild, upload  # noqa: E402

n, dim, R, T1, T2 = (int(x) for x in sys.argv[1:6])
dist = sys.argv[6]
ds = g.generate(n, dim, dist, seed=1)
eng = DeviceBuild(upload(ds.data, torch.device("cuda", 0)), dim, g.BuildParams(S=20, R=R, T1=T1, T2=T2, rho=0.6, seed=1))
offsets, nbrs, bad, fail = eng.run()
torch.cuda.synchronize()
st = eng.stats.cpu().numpy()
off = offsets.cpu().numpy()
ratio = st[:, _lib.ST_TCV_MAX_RATIO].astype(np.int32).view(np.float32)
out = {"lib": str(_lib.LIB_PATH), "checked": int(st[:, _lib.ST_TCV_CHECKED].sum()),
       "violations": int(st[:, _lib.ST_TCV_VIOLATIONS].sum()), "max_ratio": float(ratio.max()),
       "offsets": off.tolist() if n <= 20000 else None,
       "nbrs": nbrs[: int(off[-1])].cpu().numpy().tolist() if n <= 20000 else None}
print(json.dumps(out))
