#!/bin/bash
# One GPU session: tests, bench line, ncu launch list and full-set captures (dev tool).
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --points 10000 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assemble_dual -c 2 -o gpurun_out/prof_dual_full \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --points 10000 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemv -c 1 -o gpurun_out/prof_gemv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --points 10000 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_field -c 1 -o gpurun_out/prof_field \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --points 100000 > /dev/null 2>&1
ls -la gpurun_out
