"""Summarise an ncu --set full report of one update round's pair-phase kernels into JSON
(profiles/): per-kernel duration, DRAM bytes, L2 hit rate, issue activity; and the sums
bench.py reports as roofline.traffic."""
import csv, io, json, subprocess, sys
rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
def val(d, name, scale=1.0):
    i = hdr.index(name)
    v = float(d[i].replace(",", "") or 0)
    u = units[i]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
            "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)
    return v * mult * scale
ks = []
for d in data:
    ks.append({
        "kernel": d[hdr.index("Kernel Name")].split("(")[0],
        "duration_ms": round(val(d, "gpu__time_duration.sum"), 4),
        "dram_read_bytes": int(val(d, "dram__bytes_read.sum")),
        "dram_write_bytes": int(val(d, "dram__bytes_write.sum")),
        "l2_hit_pct": round(val(d, "lts__t_sector_hit_rate.pct"), 2),
        "issue_active_pct": round(val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
        "warps_active_pct": round(val(d, "sm__warps_active.avg.pct_of_peak_sustained_active"), 2),
        "registers": int(val(d, "launch__registers_per_thread")),
    })
tot_ms = sum(k["duration_ms"] for k in ks)
dram = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in ks)
json.dump({"capture": note, "report": rep, "kernels": ks, "duration_ms_serialized": round(tot_ms, 4),
           "dram_bytes_per_round": dram, "dram_gbs_serialized": round(dram / (tot_ms * 1e-3) / 1e9, 1)},
          open(out, "w"), indent=1)
print(json.dumps({"duration_ms": tot_ms, "dram_bytes": dram}))
