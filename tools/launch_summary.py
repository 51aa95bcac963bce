"""Per-kernel launch counts and mean durations of an ncu --metrics gpu__time_duration.sum CSV.

    python tools/launch_summary.py file.csv [--skip-setup]
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    return [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]


def main():
    data = load(sys.argv[1])
    agg = collections.OrderedDict()
    for _, k, v in data:
        kk = k.split("(")[0][:80]
        a = agg.setdefault(kk, [0, 0.0])
        a[0] += 1
        a[1] += v
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:5d} {t / 1e3:10.1f}us {t / n / 1e3:8.2f}us/launch  {k}")


if __name__ == "__main__":
    main()
