"""Key metrics per kernel launch from an ncu report (raw page)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__average_warp_latency_per_inst_issued.ratio", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__shared_mem_per_block_dynamic"]


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    res = []
    for r in rows[2:]:
        d = {"kernel": r[ki][:60]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    for d in metrics(sys.argv[1]):
        print(d["kernel"])
        for k, v in d.items():
            if k != "kernel":
                print(f"   {k:58s} {v}")
