"""Small build for compute-sanitizer (memcheck / racecheck / synccheck): 4000 x 128 gaussian,
S20 R96 T1=2 T2=3 with the tensor-core pair phase from round 1, checked against the oracle,
then a device search + brute force."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import oracle
import paper_2510_02774_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
ds = g.generate(n, 128, "gaussian", seed=1)
graph = g.build(ds, g.BuildParams(S=20, R=96, T1=2, T2=3, rho=0.6, seed=1))
off, nb = oracle.build(ds.data, 20, 96, 2, 3, 0.6, 1)
assert np.array_equal(graph.offsets, off) and np.array_equal(graph.neighbor_ids, nb)
q = g.generate(16, 128, "gaussian", seed=2).data
ids, _ = g.search_batch(graph, ds, q, g.SearchParams(L=32, k=10))
truth = g.brute_force_knn_batch(ds, q, 10)
torch.cuda.synchronize()
print("sanitize build ok", len(graph.neighbor_ids), "edges; recall", g.mean_recall(ids, truth))
