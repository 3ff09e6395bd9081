# backward uniform-branch budget under the barrier-light transitions (interleaved A/B)
timeout 2000 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_UBRANCH_BWD=1" "HQ_UBRANCH_BWD=2" 3 >> gpurun_out/ab_ap.log 2>&1
