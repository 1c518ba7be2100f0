"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = d["Kernel Name"].split("(")[0][-60:] + " " + d["Grid Size"]
    v = float(d["Metric Value"].replace(",", ""))
    v = v / 1e3 if d["Metric Unit"] == "ns" else (v * 1e3 if d["Metric Unit"] == "ms" else v)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'total ms':>10} {'share':>6} {'launches':>8} {'avg us':>10}  kernel grid")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1]/1e3:10.3f} {100*v[1]/tot:5.1f}% {v[0]:8d} {v[1]/v[0]:10.1f}  {k}")
print(f"sum of kernel time: {tot/1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
