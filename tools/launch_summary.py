"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name.

Usage: python tools/launch_summary.py launches.csv "command line that produced it" > summary.txt
Per-launch times from ncu are cold-cache and serialised: the SHARES are what compare with the
bench's CUDA-event phase times, not the absolute sums.
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    t = {}
    name = {}
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            t[r[ii]] = float(r[vi].replace(",", ""))
            name[r[ii]] = r[ki]
    unit = 1e6  # ns -> ms
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for i, v in t.items():
        k = re.sub(r"^void ", "", name[i])
        k = re.sub(r"\(.*$", "", k).replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none --csv, command: {cmd}")
    print("Per-launch times are cold-cache and serialised: compare SHARES.")
    print(f"total {total / unit:.1f} ms over {len(t)} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / unit:10.2f} ms {cnt[k]:6d} launches {100 * v / total:5.1f}%  {k}")


if __name__ == "__main__":
    main()
