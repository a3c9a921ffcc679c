"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count / mean / share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
        unit = r[ui]
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v):12.1f} {unit} share={sum(v)/tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
