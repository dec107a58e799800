"""Per-round kernel-time table from an ncu launch list (rounds start at bin_kernel)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
seq = [(r[ki], float(r[vi]) / 1e6) for r in data if r[mi] == "gpu__time_duration.sum"]
cls = [("pairs", ("pairs_kernel", "tc3_pairs", "tc_pairs", "tc_stage")), ("decide", ("decide_kernel",)),
       ("apply", ("apply_round",)), ("sort", ("segsort",)), ("bin", ("bin_kernel",)), ("scatter", ("scatter_kernel",))]
rounds, cur = [], None
for n, v in seq:
    if n.startswith("grnnd::bin_kernel"):
        cur = collections.Counter(); rounds.append(cur)
    if cur is None:
        continue
    c = next((c for c, keys in cls if any(k in n for k in keys)), "other")
    cur[c] += v
    cur["total"] += v
maxr = int(sys.argv[2]) if len(sys.argv) > 2 else 64
print("round " + " ".join(f"{c:>7s}" for c, _ in cls) + "   other   total (ms, serialized)")
for i, r in enumerate(rounds[:maxr]):
    print(f"{i + 1:5d} " + " ".join(f"{r[c]:7.2f}" for c, _ in cls) + f" {r['other']:7.2f} {r['total']:7.2f}")
