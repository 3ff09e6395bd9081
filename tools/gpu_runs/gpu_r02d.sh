set -x
export PARITY_LOG=gpurun_out/parity_r02d.jsonl
rm -f $PARITY_LOG
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -x 2>&1 | tail -30 > gpurun_out/gputest_r02d.log
for sh in 0 1; do
  for pr in c128 c64; do
    echo "== HQ_SHFL=$sh $pr"
    HQ_SHFL=$sh timeout 600 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -2
  done
done > gpurun_out/shfl_r02d.log 2>&1
bash tools/gpu_r02c.sh
timeout 1500 python tools/cfg5_sharded.py > gpurun_out/cfg5_r02d.json 2> gpurun_out/cfg5_r02d.err
tail -3 gpurun_out/gputest_r02d.log
