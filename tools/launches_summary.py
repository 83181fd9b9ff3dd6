"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hdr + 1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        out.append((r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", ""), v * scale))
    return out


if __name__ == "__main__":
    data = load(sys.argv[1])
    agg = collections.OrderedDict()
    tot = sum(v for _, v in data)
    for n, v in data:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
    print(f"total {tot:.1f} us over {len(data)} launches (cold-cache, serialised)")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} us {100 * t / tot:5.1f}%  {c:4d}x {t / c:8.2f} us/launch  {n}")
