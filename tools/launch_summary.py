"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summarize(path, top=12, by_grid=False):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        name = r[ki]
        base = name.split("(")[0]
        if "<" in base:
            base = base.split("<")[0] + "<" + base.split("<", 1)[1][:60]
        if by_grid:
            base += " grid" + r[gi]
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        v *= scale.get(r[ui], 1.0)
        agg[base][0] += 1
        agg[base][1] += v
    tot = sum(t for _, t in agg.values())
    out = [f"{path}: {sum(n for n, _ in agg.values())} launches, {tot:.1f} us total (ncu, serialised)"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"  {100 * t / tot:5.1f}%  {t:11.1f} us  n={n:6d}  avg={t / n:9.2f} us  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    grid = "--grid" in sys.argv
    for p in sys.argv[1:]:
        if p != "--grid":
            print(summarize(p, top=20 if grid else 12, by_grid=grid))
