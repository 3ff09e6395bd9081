# complex64 batched dot partials per warp (4 default / 2), alternating processes; c128 default now 2
for rep in 1 2; do for v in "HQ_DOT_GROUP=4" "HQ_DOT_GROUP=2"; do
  echo "== c64 $v" >> gpurun_out/probe_aw.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c64 2>&1 | grep onchip >> gpurun_out/probe_aw.log
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_aw.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_aw.log
