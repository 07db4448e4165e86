#!/bin/bash
# Dev loop on the GPU box: build, -m gpu tests (minus the slow at-scale file
# unless FULL=1), a short bench line, and optionally an ncu capture of one
# kernel (NCU=<regex>).  Everything lands in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ "${FULL:-0}" = "1" ]; then sel=""; else sel="--deselect tests/test_gpu_scale_parity.py"; fi
if [ "${TESTS:-1}" = "1" ]; then timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q -x $sel 2>&1 | tail -30 > gpurun_out/gpu_tests.log; fi
[ -f gpurun_out/gpu_tests.log ] && tail -3 gpurun_out/gpu_tests.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu --lines ${LINES:-1024} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print('value', d['value'], 'phases', d['phases_s']); print('roofline', d['roofline'])" || tail -20 gpurun_out/bench_quick.err
fi
if [ -n "${NCU:-}" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU} -s ${NCU_SKIP:-0} -c 1 -o gpurun_out/prof_${NCU} \
      python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --points 1000 --lines 0 > gpurun_out/ncu_${NCU}.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_${NCU}.ncu-rep > gpurun_out/prof_${NCU}.txt 2>&1
  cat gpurun_out/prof_${NCU}.txt
fi
