# complex128 forward kernels with 4 register bits: parity and interleaved timing
timeout 1500 python tools/ab_probe.py cfg4 1024 c128 "HQ_FWD_RB=0" "-" "HQ_FWD_MINB=5" "HQ_FWD_MINB=3" 4 >> gpurun_out/ab_af.log 2>&1
timeout 900 python tools/fuzz_parity.py 30 31 > gpurun_out/fuzz_af.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_af.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_af.log
