"""Top SASS instructions by warp-stall samples from `ncu -i rep --page source --csv
--print-source sass` output, with the dominant stall columns.

    python tools/sass_hotspots.py sass.csv [N]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hi = [i for i, x in enumerate(rows) if "Source" in x and "Address" in x][0]
    h = rows[hi]
    idx = {k: i for i, k in enumerate(h)}
    stall_cols = [k for k in h if k.startswith("stall_")]
    body = [x for x in rows[hi + 1:] if len(x) == len(h)]
    key = idx["Warp Stall Sampling (All Samples)"]
    tot = sum(float(x[key] or 0) for x in body)
    body.sort(key=lambda x: -float(x[key] or 0))
    print(f"total samples {tot:.0f}")
    for x in body[:n]:
        st = sorted(((float(x[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"{x[idx['Address']][-5:]} {float(x[key]):6.0f} {100 * float(x[key]) / tot:5.1f}%  "
              f"{x[idx['Source']].strip()[:60]:60s} {' '.join(f'{c}:{v:.0f}' for v, c in st if v)}")


if __name__ == "__main__":
    main()
