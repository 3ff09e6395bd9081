# ping-pong backward kernels: parity first (bounded by timeouts), then timing
export HQ_PINGPONG=1
timeout 300 python tools/pass_probe.py cfg4 128 c128 > gpurun_out/pp_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/pp_smoke.log
tail -2 gpurun_out/pp_smoke.log
if grep -q "smoke rc=0" gpurun_out/pp_smoke.log; then
  timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or random_layers or folded or natural or streaming or cfg2 or cfg3 or reupload or qae or deferred or trailing" 2>&1 | tail -5 > gpurun_out/pp_tests.log
  for pr in c128 c64; do
    for v in 0 1; do
      echo "== $pr HQ_PINGPONG=$v"; HQ_PINGPONG=$v timeout 300 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -1
    done
  done > gpurun_out/pp_timing.log 2>&1
fi
cat gpurun_out/pp_tests.log gpurun_out/pp_timing.log 2>/dev/null
