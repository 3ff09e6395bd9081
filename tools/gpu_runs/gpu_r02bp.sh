# fixed low tile bits (128-byte HBM runs) re-checked now that the kernels are FP-bound (interleaved A/B)
timeout 2400 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_FIXED_BITS=2" "HQ_FIXED_BITS=1" "HQ_FIXED_BITS=0" 3 >> gpurun_out/ab_bp.log 2>&1
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_FIXED_BITS=3" "HQ_FIXED_BITS=2" 3 >> gpurun_out/ab_bp.log 2>&1
