# 4-bit forward kernels: uniform-branch budget (code size vs FSEL swaps), interleaved A/B
timeout 1500 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_UBRANCH=0" "HQ_UBRANCH=1" "HQ_FWD_MINB=2" 4 >> gpurun_out/ab_ak.log 2>&1
