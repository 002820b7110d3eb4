"""Print the key metrics of an ncu raw CSV (scripts/ncu_capture.sh output)."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
for i, h in enumerate(hdr):
    stall = "warps_issue_stalled" in h and "per_issue_active" in h
    if h in KEYS or stall:
        try:
            if stall and float(vals[i]) < 0.1:
                continue
        except ValueError:
            pass
        print(f"{h:75s} {units[i]:12s} {vals[i]}")
