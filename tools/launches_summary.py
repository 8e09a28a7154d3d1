"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: count, total, share."""
import collections
import csv
import re
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    tot, cnt = collections.defaultdict(float), collections.Counter()
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("void ", "").replace("(anonymous namespace)::", "")
        name = re.split(r"\(", name, 1)[0]
        if gi is not None:
            name += "  grid" + r[gi]
        unit = r[ui]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    T = sum(tot.values())
    lines = [f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} {cnt[k]:8d} {v * scale:10.3f} {100 * v / T:6.1f}%")
    lines.append(f"{'TOTAL':70s} {sum(cnt.values()):8d} {T * scale:10.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
