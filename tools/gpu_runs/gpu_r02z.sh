# interleaved A/B of the transition barriers / warp-bit assignment, both precisions
for prec in c64 c128; do
timeout 900 python tools/ab_probe.py cfg4 1024 $prec "HQ_WARP_SYNC=0,HQ_KEEP_WARPS=0" "HQ_WARP_SYNC=1,HQ_KEEP_WARPS=1" \
   "HQ_WARP_SYNC=0,HQ_KEEP_WARPS=1" "HQ_WARP_SYNC=1,HQ_KEEP_WARPS=0" 5 >> gpurun_out/ab_z.log 2>&1
done
