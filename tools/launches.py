"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import csv
import sys
from collections import OrderedDict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        us = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(u, v / 1e3)
        name = r[ki].split("(")[0].replace("ps::<unnamed>::", "").replace("void ", "")[:60]
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + us)
    tot = sum(t for _, t in agg.values())
    for name, (c, t) in agg.items():
        print(f"{t:10.1f} us  {100 * t / tot:5.1f}%  x{c:<3d} {name}")
    print(f"{tot:10.1f} us total")


if __name__ == "__main__":
    main()
