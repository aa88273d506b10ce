"""Key metrics + top stall reasons per launch of an ncu --set full report, as CSV.

usage: python tools/ncu_summary.py <report.ncu-rep> > profiles/<name>.csv
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    w = csv.writer(sys.stdout)
    w.writerow(["launch", "kernel"] + [f"{k} [{units[hdr.index(k)]}]" for k in KEYS if k in hdr]
               + ["top stalls (cycles per issued instruction)"])
    for i, r in enumerate(data):
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        st = sorted(((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
                      float(r[hdr.index(h)])) for h in stall if r[hdr.index(h)] not in ("", "n/a")),
                    key=lambda x: -x[1])[:6]
        w.writerow([i, name] + [r[hdr.index(k)] for k in KEYS if k in hdr]
                   + ["; ".join(f"{a}={b:.2f}" for a, b in st)])


if __name__ == "__main__":
    main(sys.argv[1])
