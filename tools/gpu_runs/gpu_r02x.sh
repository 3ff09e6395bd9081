# group barriers for partially kept warp slots: parity + timing A/B
timeout 900 python tools/fuzz_parity.py 30 21 > gpurun_out/fuzz_x.txt 2>&1
FUZZ_KINDS=RZ,RY,RX,CNOT,CZ,H,SWAP,CR timeout 900 python tools/fuzz_parity.py 20 22 >> gpurun_out/fuzz_x.txt 2>&1
for v in "HQ_KEEP_WARPS=0" "HQ_KEEP_WARPS=1" "HQ_WARP_SYNC=0"; do
  echo "== c128 $v" >> gpurun_out/probe_x.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c128 >> gpurun_out/probe_x.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_x.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_x.log
