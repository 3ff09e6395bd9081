# warp-local window transitions: parity (random circuits) and timing A/B
timeout 900 python tools/fuzz_parity.py 30 11 > gpurun_out/fuzz_v.txt 2>&1
FUZZ_KINDS=RZ,RZ,CR,RY,RX,CNOT,CZ,H,SWAP timeout 900 python tools/fuzz_parity.py 20 12 >> gpurun_out/fuzz_v.txt 2>&1
for prec in c128 c64; do
for v in "HQ_WARP_SYNC=0 HQ_KEEP_WARPS=0" "HQ_WARP_SYNC=1 HQ_KEEP_WARPS=0" "HQ_WARP_SYNC=1 HQ_KEEP_WARPS=1"; do
  echo "== $prec $v" >> gpurun_out/probe_v.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 $prec >> gpurun_out/probe_v.log 2>&1
done
done
