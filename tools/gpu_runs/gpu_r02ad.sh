# new transition-barrier parity test; forward time at 4 register bits (c128)
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "window_transition" > gpurun_out/pytest_ad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ad.log
for v in "HQ_REG_BITS=3" "HQ_REG_BITS=4" "HQ_REG_BITS=4 HQ_FWD_MINB=2" "HQ_REG_BITS=4 HQ_FWD_MINB=4"; do
  echo "== c128 $v" >> gpurun_out/probe_ad.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c128 >> gpurun_out/probe_ad.log 2>&1
done
