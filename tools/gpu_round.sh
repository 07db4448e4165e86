#!/bin/bash
# One GPU session (dev tool): tests, bench line, ncu launch list of OUR kernels
# and full-set captures of the top kernels.  Every step has its own timeout;
# gpurun_out/ must stay under 64 MiB (the reports are summarised to text on
# the box and only the small ones are kept).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --points 10000 --lines 1024 > gpurun_out/ncu_launch.log 2>&1
for k in k_assemble_row4 k_gemv k_field_dyn k_surface_distance k_trace_near; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k \
      python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --points 10000 --lines 8192 > gpurun_out/ncu_$k.log 2>&1
done
timeout 900 python tools/trace_probe.py 1.0 100000 > gpurun_out/cfg5_full.log 2>&1
du -sh gpurun_out/* | sort -h | tail -8
# keep the copy-back under the limit: drop the largest reports if needed
while [ "$(du -sm gpurun_out | cut -f1)" -gt 60 ]; do
  big=$(ls -S gpurun_out/*.ncu-rep 2>/dev/null | head -1); [ -z "$big" ] && break
  python tools/ncu_summary.py "$big" > "${big%.ncu-rep}.summary.txt" 2>&1; rm -f "$big"; echo "summarised+dropped $big"
done
ls -la gpurun_out
