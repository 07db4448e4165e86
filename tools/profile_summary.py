"""Summarise a GPU round's ncu output into profiles/ (tracked).

    python tools/profile_summary.py r01   # reads gpurun_out/{launches.csv,prof_*.ncu-rep}
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PROF, exist_ok=True)

# launch list: per-kernel share of device time
rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
hdr = None
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    tot[name] += float(d["Metric Value"]) / 1e6
    cnt[name] += 1
T = sum(tot.values())
with open(os.path.join(PROF, f"{tag}_launches.txt"), "w") as fh:
    fh.write("ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ python bench.py --steps 1 "
             "--warmup 0 --no-e2e --no-cpu --no-full-trace --points 10000 --lines 1024\n"
             "(cold-cache, serialised launches: compare SHARES, not absolutes)\n\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        fh.write(f"{k:50s} {cnt[k]:6d} launches {v:10.2f} ms {v / T * 100:6.2f}%\n")
    fh.write(f"total {T:.2f} ms\n")

# full-set captures
traffic = {}
for fn in sorted(os.listdir(OUT)):
    if not (fn.startswith("prof_") and fn.endswith(".ncu-rep")):
        continue
    rep = os.path.join(OUT, fn)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                         text=True)
    k = fn[len("prof_"):-len(".ncu-rep")]
    skip_file = os.path.join(OUT, f"prof_{k}.skip")
    skip = open(skip_file).read().split()[-1] if os.path.exists(skip_file) else "?"
    with open(os.path.join(PROF, f"{tag}_ncu_{k}.txt"), "w") as fh:
        fh.write(f"ncu --set full --clock-control none --import-source on -k regex:{k} -s {skip} -c 1 (one launch) "
                 f"of python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-full-trace --points 10000 "
                 f"--lines 1024\n\n")
        fh.write(res.stdout)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        d = dict(zip(rr[0], rr[2]))
        units = dict(zip(rr[0], rr[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}

        def val(key):
            v = d.get(key)
            return None if v in (None, "") else float(v.replace(",", "")) * scale.get(units.get(key, "byte"), 1)

        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        traffic[k] = {"dram_read_bytes": rd, "dram_write_bytes": wr,
                      "bytes_per_launch": (rd or 0) + (wr or 0),
                      "time_ns": val("gpu__time_duration.sum")}
json.dump(traffic, open(os.path.join(PROF, f"{tag}_ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(PROF, f"{tag}_launches.txt")).read())
print(json.dumps(traffic, indent=1))
