#!/bin/bash
# One GPU session (dev tool) producing the round's evidence in gpurun_out/:
# the default bench line, the reference-arm line, the ncu launch list of our
# kernels and full-set captures of the top kernels (summarised to text on the
# box; reports dropped if the copy-back would exceed the limit).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
SMALL="--steps 1 --warmup 0 --no-e2e --no-cpu --no-full-trace --uniform-points 0 --points 10000 --lines 1024"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/launches.csv python bench.py $SMALL > gpurun_out/ncu_launch.log 2>&1
# kernel:skip -- which launch to capture (k_surface_distance -s 0 = the seed
# pick of the step's trace phase, a non-empty launch)
for ks in k_sweep:0 k_gemv_f64_v4:5 k_field:0 k_field_dyn:60 k_surface_distance:0 k_trace_near:60 k_mgs_cluster:20; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k$" -s $s -c 1 -o gpurun_out/prof_$k \
      python bench.py $SMALL > gpurun_out/ncu_$k.log 2>&1
  echo "$k -s $s" > gpurun_out/prof_$k.skip
done
du -sh gpurun_out/* | sort -h | tail -8
while [ "$(du -sm gpurun_out | cut -f1)" -gt 60 ]; do
  big=$(ls -S gpurun_out/*.ncu-rep 2>/dev/null | head -1); [ -z "$big" ] && break
  python tools/ncu_summary.py "$big" > "${big%.ncu-rep}.summary.txt" 2>&1; rm -f "$big"; echo "summarised+dropped $big"
done
ls -la gpurun_out
