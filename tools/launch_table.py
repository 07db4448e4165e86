"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt, mx = defaultdict(float), defaultdict(int), defaultdict(float)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)  # -> us
    tot[name] += v
    cnt[name] += 1
    mx[name] = max(mx[name], v)
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:6d} launches {tot[k] / 1e3:9.2f} ms  avg {tot[k] / cnt[k]:9.1f} us  max {mx[k]:9.1f} us")
