"""Per-kernel launch counts and mean durations of an ncu --metrics CSV
(gpu__time_duration.sum, plus dram__bytes_read.sum / dram__bytes_write.sum when
captured: mean bytes per launch and the achieved DRAM GB/s).

    python tools/launch_summary.py file.csv
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ii, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID"), h.index("Metric Name")
    out = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        out[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki]
    return [(i, names[i], m) for i, m in sorted(out.items())]


def main():
    data = load(sys.argv[1])
    agg = collections.OrderedDict()
    for _, k, m in data:
        kk = k.split("(")[0][:80]
        a = agg.setdefault(kk, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        extra = f"  {b / n / 1e6:8.2f} MB/launch {b / t:7.1f} GB/s" if b else ""
        print(f"{n:5d} {t / 1e3:10.1f}us {t / n / 1e3:8.2f}us/launch{extra}  {k}")


if __name__ == "__main__":
    main()
