import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
d = defaultdict(dict)
for r in rows[h + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(r[ui], 1e-9)
        d[(r[hdr.index("ID")], r[ki][:44])][r[mi]] = v
tot_t = tot_fp = 0
for (i, k), m in d.items():
    t = m["gpu__time_duration.sum"]
    fp = sum(m.get(f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum", 0) * (2 if o == "ffma" else 1) for o in ("fadd", "fmul"))
    fp += m.get("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", 0)
    tot_t += t; tot_fp += fp
    print(f"{k:44s} t={t*1e3:6.3f}ms fp={fp/1e9:7.2f}G eff={fp/t/37.2e12:6.1%} lanes={m.get('smsp__thread_inst_executed_per_inst_executed.ratio',0):5.1f} "
          f"warps={m.get('sm__warps_active.avg.pct_of_peak_sustained_active',0):5.1f}% issue={m.get('smsp__issue_active.avg.pct_of_peak_sustained_active',0):5.1f}% inst={m.get('smsp__inst_executed.sum',0)/1e9:.2f}G")
print(f"total t={tot_t*1e3:.3f} ms fp={tot_fp/1e9:.1f}G eff={tot_fp/tot_t/37.2e12:.1%}")
