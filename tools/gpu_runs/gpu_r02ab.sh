# knobs re-checked under the warp-group transitions (interleaved A/B, complex128)
timeout 900 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_FWD_MINB=3" "HQ_UBRANCH=0" "HQ_UBRANCH=3" "HQ_DOT_BATCH=4" 5 >> gpurun_out/ab_ab.log 2>&1
