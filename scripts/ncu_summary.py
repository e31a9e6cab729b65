"""Summarise one k_solve capture (ncu --set full) into profiles/: the metric
block DESIGN.md and bench.py's roofline.traffic cite.

usage: python scripts/ncu_summary.py <report.ncu-rep> <out.txt> [config] [command description]
Also updates profiles/solve_traffic.json[config] (DRAM bytes per launch)."""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__block_size",
           "launch__grid_size", "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active"] + [
    f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio"
    for k in ("barrier", "lg_throttle", "long_scoreboard", "membar", "short_scoreboard", "wait")]


def main():
    rep, out = sys.argv[1:3]
    cfg = sys.argv[3] if len(sys.argv) > 3 else "2"
    desc = sys.argv[4] if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    lines = ["ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 "
             "python scripts/profile_solve.py " + (desc or "--solves 1"),
             f"(config {cfg}, min objective; one k_solve<exact> launch = one full "
             "solve; ncu flushes caches before the replayed launch)", ""]
    dram = 0.0
    for i, c in enumerate(hdr):
        if "__" in c:
            lines.append(f"{c} [{units[i]}]: {vals[i]}")
            if c.startswith("dram__bytes"):
                scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[units[i]]
                dram += float(vals[i]) * scale
    lines.append(f"dram bytes per launch: {dram:.4e}")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(os.path.abspath(out)).split("/profiles")[0], "profiles",
                         "solve_traffic.json")
    t = json.load(open(tpath)) if os.path.exists(tpath) else {}
    t[cfg] = {"kernel": "k_solve<exact,1>", "dram_bytes_per_launch": dram, "objective": "min",
              "source": os.path.relpath(os.path.abspath(out), os.path.dirname(os.path.dirname(tpath)))}
    with open(tpath, "w") as f:
        json.dump(t, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
