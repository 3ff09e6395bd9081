# shear-form deferred phases (complex128): parity, then A/B timing
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "c128" 2>&1 | tail -3 > gpurun_out/shear_tests.log
for v in 1 0 1 0; do
  echo "== HQ_SHEAR_FLUSH=$v"; HQ_SHEAR_FLUSH=$v timeout 300 python tools/pass_probe.py cfg4 1024 c128 2>&1 | tail -1
done > gpurun_out/shear_timing.log 2>&1
cat gpurun_out/shear_tests.log gpurun_out/shear_timing.log
