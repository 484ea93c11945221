"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    mi = h.index("Metric Name") if "Metric Name" in h else None
    tot, cnt = collections.defaultdict(float), collections.Counter()
    unit = "?"
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
        unit = r[ui] if ui is not None else unit
    T = sum(tot.values())
    out = []
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append((k, cnt[k], v, v / T, v / cnt[k]))
    return out, unit


if __name__ == "__main__":
    res, unit = shares(sys.argv[1])
    for k, n, v, sh, per in res:
        print(f"{k[:60]:60s} n={n:5d} total={v:14.1f} {unit} share={sh:.3f} per_launch={per:.1f}")
