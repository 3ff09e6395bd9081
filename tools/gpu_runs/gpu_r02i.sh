timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "readout_invariant or lazy" 2>&1 | tail -3 > gpurun_out/t_r02i.log
timeout 600 python -m pytest tests/test_gpu_noise.py -q -x 2>&1 | tail -3 >> gpurun_out/t_r02i.log
for pr in c128 c64; do
  for kv in "X=0" "HQ_FWD_MINB=2" "HQ_FWD_MINB=4" "HQ_FWD_MINB=5"; do
    echo "== $pr $kv"; env $kv timeout 300 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -1
  done
done > gpurun_out/fwdminb_r02i.log 2>&1
cat gpurun_out/t_r02i.log gpurun_out/fwdminb_r02i.log
