# upper bound of the remaining transition barriers: post-store barriers removed (timing only, wrong results)
timeout 2000 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_ABLATE=16" "HQ_ABLATE=1" 3 >> gpurun_out/ab_at.log 2>&1
