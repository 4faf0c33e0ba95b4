"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

usage: python profiles/summarize_launches.py launches.csv > summary.txt
Per-launch times from ncu are cold-cache and serialised: compare SHARES.
"""
import collections
import csv
import sys


def main(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:90]
        ns = float(r["Metric Value"].replace(",", ""))
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':92s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for k, (cnt, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:92s} {cnt:8d} {ns / 1e3:12.1f} {ns / 1e3 / cnt:10.2f} {100 * ns / total:6.1f}%")
    print(f"total {total / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
