export PARITY_LOG=gpurun_out/parity_r02g.jsonl
rm -f $PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gputest_r02g.log
for pr in c128 c64; do
  for kv in "X=0" "HQ_NO_DROP=1"; do
    echo "== $pr $kv"; env $kv timeout 600 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -2
  done
done > gpurun_out/drop_r02g.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
tail -3 gpurun_out/gputest_r02g.log; cat gpurun_out/drop_r02g.log
