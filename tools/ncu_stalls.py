"""Per-instruction-class stall breakdown from `ncu --page source --csv --print-source sass`.

usage: ncu -i rep --page source --csv --print-source sass > src.csv
       python tools/ncu_stalls.py src.csv [top]
"""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_op = collections.defaultdict(lambda: collections.Counter())
    total = collections.Counter()
    for r in data:
        src = r[col["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        for h in stalls:
            v = r[col[h]]
            if v and v != "0":
                by_op[op][h] += int(v)
                total[h] += int(v)
    print("total by reason:", ", ".join(f"{k[6:]}={v}" for k, v in total.most_common(10)))
    ranked = sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:int(top)]
    for op, c in ranked:
        print(f"{op:12s} {sum(c.values()):8d}  " + ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(4)))


if __name__ == "__main__":
    main(*sys.argv[1:])
