python -c "import __graft_entry__ as g; g.build()" >/dev/null
REPS=1 NOHOST=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_field_dyn|k_trace_near|k_surface|k_field_reduce_dyn|k_trace_ctrl" --csv --log-file gpurun_out/trace2k_launches.csv python tools/trace_tail_probe.py 2048 > gpurun_out/trace2k.log 2>&1
tail -2 gpurun_out/trace2k.log
