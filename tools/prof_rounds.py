"""Run a short build schedule for ncu launch lists (development aid)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2510_02774_b200 as g
n = int(sys.argv[1]); dim = int(sys.argv[2]); T1 = int(sys.argv[3]); T2 = int(sys.argv[4])
ds = g.generate(n, dim, "gaussian", seed=1)
graph = g.build(ds, g.BuildParams(S=20, R=96, T1=T1, T2=T2, rho=0.6, seed=1))
torch.cuda.synchronize()
print("edges", len(graph.neighbor_ids))
