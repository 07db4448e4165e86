# Dev: run the bench with per-step spans while nvidia-smi samples clocks,
# power, temperatures and throttle reasons every 50 ms (gpurun_out/smi.csv).
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/smi.csv 2>&1 &
SMI=$!
HVB_BENCH_SPANS=1 timeout 1500 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --no-full-trace --uniform-points 0 > gpurun_out/bs.json 2> gpurun_out/bs.err
kill $SMI
grep "^step" gpurun_out/bs.err
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/smi.csv")) if len(r) >= 7]
sm = collections.Counter(r[1].strip() for r in rows); mem = collections.Counter(r[2].strip() for r in rows)
rs = collections.Counter(r[6].strip() for r in rows)
print("sm", sm.most_common(6)); print("mem", mem.most_common(4)); print("reasons", rs.most_common(6))
print("temp gpu max", max(r[4] for r in rows), "mem temp max", max(r[5] for r in rows), "power max", max(float(r[3].split()[0]) for r in rows if r[3].strip()[0].isdigit()))
PY
