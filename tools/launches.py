"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel launches and ms."""
import csv
import sys
from collections import defaultdict


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        d = dict(zip(rows[hdr], r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:48]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", "")) / 1e6  # ns -> ms
    return agg


if __name__ == "__main__":
    agg = summarize(sys.argv[1])
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:50s} {n:5d} {t:10.3f} ms {100 * t / tot:5.1f}%")
    print(f"{'total':50s} {sum(n for n, _ in agg.values()):5d} {tot:10.3f} ms")
