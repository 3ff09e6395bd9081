# shear-form deferred phases re-checked under the barrier-light transitions (interleaved A/B)
timeout 2000 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_SHEAR_FLUSH=1" "HQ_DEFER_PARTIAL=0" "HQ_DEFER_PARTIAL=1" 3 >> gpurun_out/ab_ao.log 2>&1
