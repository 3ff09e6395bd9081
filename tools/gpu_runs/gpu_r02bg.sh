# complex64 forward kernels with 5 register bits (opt-in HQ_FWD_RB=1): timing and parity
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_FWD_RB=1" "HQ_FWD_RB=1,HQ_FWD_MINB=3" 3 >> gpurun_out/ab_bg.log 2>&1
HQ_FWD_RB=1 timeout 900 python tools/fuzz_parity.py 30 41 > gpurun_out/fuzz_bg.txt 2>&1
HQ_FWD_RB=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_bg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bg.log
