import os, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2510_02774_b200 as g
from paper_2510_02774_b200.core import generate
ds = generate(20000, 128, "gaussian", seed=1)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 128
off, nb = oracle.build(ds.data, 20, R, 2, 6, 0.6, 1)
for env in ("0", "3", "60"):
    os.environ["GRNND_EXACT_FIRST_ROUNDS"] = env
    gr = g.build(ds, g.BuildParams(S=20, R=R, T1=2, T2=6, rho=0.6, seed=1))
    print("R", R, "exact first rounds", env, "equal", np.array_equal(gr.offsets, off) and np.array_equal(gr.neighbor_ids, nb), flush=True)
