# complex64 with warp-group transitions + DP warp slots by default; dot chains on top (one compiler)
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_WARP_SYNC=0,HQ_KEEP_WARPS=0" "HQ_DOT_CHAINS=2" "HQ_DOT_CHAINS=3" 3 >> gpurun_out/ab_ba.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_ba.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ba.log
