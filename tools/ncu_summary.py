"""Summarise an ncu report of one kernel: time, pipes, stalls, instruction mix."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = {k: float(v) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
print("stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
h = srows[1]; data = srows[2:]
i_e = h.index("Instructions Executed")
ex = Counter()
for r in data:
    t = r[1].strip().split()
    if not t: continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ex[op] += float(r[i_e] or 0)
tot = sum(ex.values())
fp = sum(ex[k] for k in ("DFMA", "DMUL", "DADD", "DSETP"))
print(f"instructions {tot:.3g}, FP64 share {fp / tot * 100:.1f}%")
print("mix:", ", ".join(f"{k}={v / tot * 100:.1f}%" for k, v in ex.most_common(14)))
