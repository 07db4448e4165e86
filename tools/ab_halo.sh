# A/B of regular-sweep builds on the GPU box: optional sweep/parity/
# distributed GPU tests (TESTS=1), then the config-4 sweep time
# (tools/sweep_probe.py) for each HVB_NVCC_EXTRA variant in VARIANTS
# ('#' separates flags within one variant).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "${TESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests/test_distributed.py tests/test_gpu_edge.py tests/test_gpu_parity.py -m gpu -x -q \
      > gpurun_out/ab_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/ab_tests.log
fi
for v in ${VARIANTS:-"-DHVB_NONE"}; do
  rm -f paper_2003_12663_b200/libhvb.so
  HVB_NVCC_EXTRA="${v//#/ }" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "$v: $(timeout 600 python tools/sweep_probe.py 2>&1 | tail -1)"
done
