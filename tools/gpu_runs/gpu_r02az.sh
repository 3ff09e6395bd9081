# knobs re-measured with ONE compiler (NVRTC 12.9 on the box and in the cache), interleaved A/B
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_WARP_SYNC=1" "HQ_WARP_SYNC=1,HQ_KEEP_WARPS=1" "HQ_KEEP_WARPS=1" "HQ_DOT_CHAINS=2" 3 >> gpurun_out/ab_az.log 2>&1
timeout 2400 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_FWD_RB=0" "HQ_WARP_SYNC=0,HQ_KEEP_WARPS=0" "HQ_UBRANCH_BWD=1" "HQ_DIAG_DOTS=0" 3 >> gpurun_out/ab_az.log 2>&1
for rep in 1 2; do for v in "HQ_DOT_GROUP=2" "HQ_DOT_GROUP=4"; do
  echo "== c128 $v" >> gpurun_out/probe_az.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c128 2>&1 | grep onchip >> gpurun_out/probe_az.log
done; done
