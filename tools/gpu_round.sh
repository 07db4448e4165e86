#!/bin/bash
# One GPU session (dev tool): tests, bench line, ncu launch list of OUR kernels
# and full-set captures of the top kernels.  Every step has its own timeout.
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
ls -la gpurun_out
