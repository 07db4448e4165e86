#!/bin/bash
# A/B the assembly configuration on the bench workload (dev tool):
#   tools/ab.sh "QUAD=0" "QUAD=1 WIN=96" ...   (keys become HVB_ASM_<KEY>)
for cfg in "$@"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/HVB_ASM_\1=/g') timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
      --points 10000 --lines 0 > /tmp/ab.json 2> /tmp/ab.err || { echo "$cfg FAILED"; tail -5 /tmp/ab.err; continue; }
  python -c "import json,sys; d=json.loads(open('/tmp/ab.json').readline()); print('$cfg', round(d['value']/1e9,3), 'Gent/s', {k: round(v,4) for k,v in d['phases_s'].items()}, 'frac', round(d['roofline']['frac'],4))"
done
