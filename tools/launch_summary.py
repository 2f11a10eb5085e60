"""Per-kernel totals and shares of an ncu launch list (dev tool).

    python tools/launch_summary.py launches.csv "<header line>" > profiles/<name>.txt
"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        us = float(r[mi].replace(",", "")) * SCALE[r[ui]]
        n = r[ki][5:] if r[ki].startswith("void ") else r[ki]
        n = n.split("(")[0]
        tot[n][0] += 1
        tot[n][1] += us
    S = sum(v[1] for v in tot.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{n[:56]:56s} n={c:4d} total={t / 1e3:9.3f} ms mean={t / c:9.1f} us share={100 * t / S:5.1f}%")


if __name__ == "__main__":
    main()
