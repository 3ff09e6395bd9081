# complex64 opt-in variants re-measured with one compiler (interleaved A/B)
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_SHFL=1" "HQ_PINGPONG=1" "HQ_DIAG_DOTS=0" "HQ_PLAN_SEARCH=0" "HQ_DEFER_PARTIAL=1" 3 >> gpurun_out/ab_be.log 2>&1
timeout 2400 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_SHFL=1" "HQ_PINGPONG=1" 3 >> gpurun_out/ab_be.log 2>&1
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_DOT_GROUP=2" 3 >> gpurun_out/ab_be.log 2>&1
