"""Role timers + CTA-0 event trace of tc3_pairs_kernel (GRNND_T3_PROF build), one mid-build round."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2510_02774_b200 as g
from paper_2510_02774_b200 import _lib
lib = _lib.lib
lib.grnnd_debug_counters.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
lib.grnnd_debug_trace.argtypes = [C.POINTER(C.c_longlong)]
ds = g.generate(1_000_000, 128, "gaussian", seed=1)
p = g.BuildParams(S=20, R=96, T1=2, T2=15, rho=0.6, seed=1)
st = g.init_neighbors(ds, p)
row = torch.zeros(16, dtype=torch.int64, device="cuda")
buf = (C.c_ulonglong * 256)()
# slot, name, number of timed warps (lane 0 of each)
rows = [(0, "meta wait mempty", 1), (1, "meta total", 1), (2, "mma wait full", 1), (3, "mma wait acce", 1),
        (17, "mma total", 1), (20, "mma fence", 1), (21, "mma commit", 1), (4, "filt wait mfull", 3), (5, "filt bar1", 3), (6, "filt wait qemp", 3),
        (7, "filt wait accf", 3), (22, "filt ab terms", 3), (23, "filt scan", 3), (24, "filt one LDS", 3), (8, "filt total", 3), (9, "exact wait qrdy", 3), (10, "exact bar2", 3),
        (11, "exact total", 6), (18, "exact chains", 3), (19, "exact write-out", 3), (15, "rows wait mfull", 9), (16, "rows wait empty", 9), (14, "rows total", 9)]
for r in range(25):
    st.pools.update(p.seed, 1 + st.round_index, 0, row); st.round_index += 1
    torch.cuda.synchronize()
    lib.grnnd_debug_counters(buf, 256)
    if r in (3, 16, 24):
        allv = list(buf)
        for b in range(1, 7):
            v = allv[32 * b: 32 * b + 32]
            if not v[12]:
                continue
            print(f"round {r + 1} bin {b} (slot {96 // (12, 6, 4, 3, 2, 1)[b - 1]}): groups {v[12]}, "
                  f"CTA-cycles/group {v[1] / max(v[12], 1):.0f}")
            for slot, name, w in rows:
                print(f"   {name:22s} {v[slot] / max(v[12], 1) / w:10.0f} cycles/group")
tr = (C.c_longlong * 640)()
lib.grnnd_debug_trace(tr)
t = np.array(list(tr)).reshape(64, 10)
t0 = t[0, 0]
print("events (K cycles; CTA 0 of the last bin kernel): 0 meta issued, 1 rows issued (warp 0), 2 rows issued (last warp), 3 mma issued, 4 filter start, 5 filter done, 6 exact start, 7 exact done, 8 exact chains done, 9 exact write-out done")
for gi in range(0, 24):
    print(gi, " ".join(f"{(x - t0) / 1000:8.1f}" for x in t[gi]))
