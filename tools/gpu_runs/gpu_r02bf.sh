# which opt-in variant breaks under the new defaults: shuffle transitions / ping-pong, each alone
for v in "HQ_SHFL=1" "HQ_PINGPONG=1" "HQ_SHFL=1 HQ_WARP_SYNC=0" "HQ_PINGPONG=1 HQ_KEEP_WARPS=0" "HQ_SHFL=1 HQ_FWD_RB=0"; do
  echo "== $v" >> gpurun_out/dbg_bf.log
  env $v timeout 300 python tools/fuzz_parity.py 6 5 2>&1 | grep -E "worst|MISMATCH|FAILED|Error|error" | head -3 >> gpurun_out/dbg_bf.log
done
