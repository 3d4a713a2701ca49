"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:72s} n={len(v):4d} mean={sum(v)/len(v)/1000:9.2f}us share={sum(v)/tot:6.1%}")
