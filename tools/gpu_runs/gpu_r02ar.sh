# forward kernels with CTA barriers (lockstep instruction fetch) vs warp-group transitions
timeout 2000 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_WARP_SYNC_FWD=0" 4 >> gpurun_out/ab_ar.log 2>&1
