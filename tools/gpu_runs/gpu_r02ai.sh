# split complex128 forward kernels + one-warp tiles fix: fuzz and the whole GPU suite
timeout 900 python tools/fuzz_parity.py 30 31 > gpurun_out/fuzz_ai.txt 2>&1
timeout 900 python tools/fuzz_parity.py 30 32 >> gpurun_out/fuzz_ai.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ai.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ai.log
