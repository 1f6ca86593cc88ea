"""Key metrics of an ncu --set full report (one kernel): time, DRAM traffic /
throughput, SM / issue activity, occupancy, L2 hit rate, top stall reasons."""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    print("kernel:", d.get("Kernel Name", "?")[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__shared_mem_per_block_dynamic", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
    st = [(float(d[k].replace(',', '') or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
          for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
    tot = sum(v for v, _ in st) or 1.0
    print("  stall samples (share):", ", ".join(f"{n} {v / tot:.2f}" for v, n in sorted(st, reverse=True)[:8]))
