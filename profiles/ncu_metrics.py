"""Summarise an ncu report: key throughput metrics + warp stall breakdown.
usage: python profiles/ncu_metrics.py <report.ncu-rep> [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (vals[i], units[i])
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               h.startswith("smsp__pcsamp_warps_issue_stalled_"):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v > 0:
                    stalls[h] = v
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:12]
        d["top_stalls"] = top
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        d["kernel"] = name
        out.append(d)
    for d in out:
        print(d["kernel"][:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k][0]:>16s} {d[k][1]}")
        print("  top stalls:")
        for k, v in d["top_stalls"]:
            print(f"    {k:70s} {v:12.2f}")
    if "--json" in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
