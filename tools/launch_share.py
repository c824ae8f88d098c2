"""Per-kernel share of device time from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict


def shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6}.get(r[ui], 1)
        tot[r[ki][:90]] += v
        cnt[r[ki][:90]] += 1
    T = sum(tot.values())
    return [(k, v / 1e3, 100 * v / T, cnt[k]) for k, v in sorted(tot.items(), key=lambda x: -x[1])]


if __name__ == "__main__":
    for k, us, pct, n in shares(sys.argv[1]):
        print(f"{us:10.1f} us {pct:5.1f}% x{n:3d} {k}")
