# dot accumulation chains (DFMA latency vs combining DADDs), interleaved A/B
timeout 2000 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_DOT_CHAINS=2" "HQ_DOT_CHAINS=1" "HQ_DOT_CHAINS=8" 3 >> gpurun_out/ab_am.log 2>&1
timeout 2000 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_DOT_CHAINS=2" "HQ_DOT_CHAINS=8" 3 >> gpurun_out/ab_am.log 2>&1
