# parity evidence with the final kernels: measured errors of every golden / sharded case, randomised sweep
PARITY_LOG=gpurun_out/parity_as.jsonl timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_as.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_as.log
for seed in 2024 7 21; do timeout 900 python tools/fuzz_parity.py 40 $seed >> gpurun_out/fuzz_as.txt 2>&1; done
FUZZ_KINDS=RZ,RZ,RZ,CR,CR,RY,RX,CNOT,CZ,H timeout 900 python tools/fuzz_parity.py 30 99 >> gpurun_out/fuzz_as.txt 2>&1
