"""Key metrics per kernel from an ncu report (ncu -i X --page raw --csv)."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__grid_size"]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for d in data:
    print("==", d[hdr.index("Kernel Name")][:90])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:70s} {d[i]} {units[i]}")
    st = sorted(((float(d[hdr.index(h)] or 0), h) for h in stalls), reverse=True)[:7]
    print("   stalls:", ", ".join(f"{h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}" for v, h in st))
