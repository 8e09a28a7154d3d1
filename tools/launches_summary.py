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
    mi = h.index("Metric Name") if "Metric Name" in h else None
    for r in rows[hdr + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        name = r[ki].replace("void ", "").replace("(anonymous namespace)::", "")
        name = re.split(r"\(", name, 1)[0]
        if gi is not None:
            name += "  grid" + r[gi]
        # every row carries its own unit (ncu switches between ns / us / ms per launch)
        sc = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(r[ui], 1e-6)
        tot[name] += float(r[vi].replace(",", "")) * sc / 1e-6
        cnt[name] += 1
    scale = 1e-6
    T = sum(tot.values())
    lines = [f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} {cnt[k]:8d} {v * scale:10.3f} {100 * v / T:6.1f}%")
    lines.append(f"{'TOTAL':70s} {sum(cnt.values()):8d} {T * scale:10.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
