# Per-kernel device time of the tracer's rounds (ncu launch list, cold
# cache): LINES lines of cfg4 (tools/trace_tail_probe.py), kernels matched
# after SKIP launches of the trace kernels (SKIP > 0 looks at the tail).
python -c "import __graft_entry__ as g; g.build()" >/dev/null
REPS=1 NOHOST=1 timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_field_dyn|k_trace|k_surface|k_field_reduce_dyn" -s ${SKIP:-0} --csv \
    --log-file gpurun_out/trace_launches.csv python tools/trace_tail_probe.py ${LINES:-2048} > gpurun_out/trace_ncu.log 2>&1
tail -2 gpurun_out/trace_ncu.log
