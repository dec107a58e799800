import sys; sys.path.insert(0, ".")
import paper_2510_02774_b200 as g, torch
ds = g.generate(1000000, 128, "clustered", seed=1)
g.build(ds, g.BuildParams(S=20, R=96, T1=1, T2=15, rho=0.6, seed=1)); torch.cuda.synchronize()
