"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches, total, share and average duration."""
import csv
import sys
from collections import defaultdict


def main(path, skip_prefix=("k_dist_rows",)):
    rows = list(csv.reader(line for line in open(path) if not line.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("bm::dev::", "")
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[ui]]
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total us':>10s} {'share':>7s} {'avg us':>8s}")
    for name in sorted(tot, key=lambda n: -tot[n]):
        print(f"{name:28s} {cnt[name]:8d} {tot[name]:10.1f} {100 * tot[name] / allt:6.1f}% {tot[name] / cnt[name]:8.2f}")
    print(f"{'total':28s} {sum(cnt.values()):8d} {allt:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
