"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel: count, avg, last (us)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v = v / 1000 if d["Metric Unit"] in ("nsecond", "ns") else v * 1000 if d["Metric Unit"] == "msecond" else v
    agg.setdefault(d["Kernel Name"][:64], []).append(v)
for k, v in agg.items():
    print(f"{k:64s} n={len(v):3d} avg={sum(v) / len(v):9.2f} us  last={v[-1]:9.2f}")
