# complex64 with the warp-group transitions (opt-in there) and with the DP warp-bit assignment
for v in "HQ_WARP_SYNC=0" "HQ_WARP_SYNC=1 HQ_KEEP_WARPS=0" "HQ_WARP_SYNC=1 HQ_KEEP_WARPS=1" "HQ_WARP_SYNC=0 HQ_KEEP_WARPS=1"; do
  echo "== c64 $v" >> gpurun_out/probe_y.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c64 >> gpurun_out/probe_y.log 2>&1
done
