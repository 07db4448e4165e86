"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iS] or 0) for r in data)
agg = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in reasons}
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]}={v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
mode = sys.argv[3] if len(sys.argv) > 3 else "top"
if mode == "top":
    idx = sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))[:top]
    idx.sort()
else:
    idx = range(len(data))
for i in idx:
    r = data[i]
    s = float(r[iS] or 0)
    det = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:3]
    print(f"{r[0]:>6} {s / tot * 100:5.2f}% ex={float(r[iE] or 0):.3g} {r[1][:60]:60s} " +
          " ".join(f"{n}={v / max(s, 1) * 100:.0f}%" for v, n in det if v))
