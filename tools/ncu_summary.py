import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "lts__t_bytes.sum", "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
for row in r[2:]:
    name = row[hdr.index("Kernel Name")][:40]
    print("==", name)
    for k in keys:
        if k in hdr:
            print("   %-60s %s %s" % (k, row[hdr.index(k)], r[1][hdr.index(k)]))
    st = [(h, float(v)) for h, v in zip(hdr, row) if "average_warps_issue_stalled" in h and "per_issue_active" in h and v.replace('.', '', 1).isdigit()]
    for h, v in sorted(st, key=lambda x: -x[1])[:6]:
        print("   stall %-50s %.2f" % (h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v))
