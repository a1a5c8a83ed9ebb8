"""Summarise an ncu --set full capture (raw csv) into profiles/: per kernel the
duration, DRAM/L2 bytes and the main throughput / stall metrics."""
import csv, sys
src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
units = rows[1]
with open(dst, "w") as f:
    w = csv.writer(f)
    w.writerow(want)
    w.writerow([units[hdr.index(k)] if k in hdr else "" for k in want])
    for r in rows[2:]:
        w.writerow([r[hdr.index(k)] if k in hdr else "" for k in want])
print(open(dst).read())
