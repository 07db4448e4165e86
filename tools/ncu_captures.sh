mkdir -p gpurun_out; rm -f gpurun_out/prof_*.ncu-rep
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SMALL="--steps 1 --warmup 0 --no-e2e --no-cpu --no-full-trace --uniform-points 0 --points 10000 --lines 1024"
for ks in k_sweep:0 k_gemv_f64_v4:5 k_field:0 k_field_dyn:60 k_surface_distance:0 k_trace_near:60 k_mgs_cluster:20; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s $s -c 1 -o gpurun_out/prof_$k \
      python bench.py $SMALL > gpurun_out/ncu_$k.log 2>&1
  echo "$k -s $s" > gpurun_out/prof_$k.skip
done
timeout 600 python tools/trace_rounds.py 1.0 8192 > gpurun_out/trace_rounds.txt 2>&1
du -sh gpurun_out/*.ncu-rep
