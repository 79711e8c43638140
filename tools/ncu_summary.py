"""Summarise an ncu launch list (gpu__time_duration per kernel) into shares."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'share':>7} {'launches':>8} {'mean us':>9}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v) / tot * 100:6.2f}% {len(v):8d} {sum(v) / len(v):9.2f}  {k}")
    print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches (cold-cache, serialised)")


if __name__ == "__main__":
    main(sys.argv[1])
