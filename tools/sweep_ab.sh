#!/bin/bash
# Dev A/B of regular-sweep build variants on the GPU box: each argument is a
# set of -D flags; prints the probe line per variant.
for v in "$@"; do
  rm -f paper_2003_12663_b200/libhvb.so
  HVB_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"; grep -A4 "k_sweepILi12ELi0ELb0" paper_2003_12663_b200/csrc/build.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '; echo
  timeout 300 python tools/sweep_probe.py
done
rm -f paper_2003_12663_b200/libhvb.so
