# schedule search (first-pass cap by a windows + passes cost model)
for pr in c128 c64; do
  for v in 1 0 1 0; do
    echo "== $pr HQ_PLAN_SEARCH=$v"; HQ_PLAN_SEARCH=$v timeout 300 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -2
  done
done > gpurun_out/search_r02s.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or random_layers or natural" 2>&1 | tail -3 >> gpurun_out/search_r02s.log
for v in 1 0; do echo "== cfg5 HQ_PLAN_SEARCH=$v"; HQ_PLAN_SEARCH=$v timeout 900 python tools/cfg5_single_gpu.py --grad 2>&1 | cut -c1-400; done >> gpurun_out/search_r02s.log 2>&1
grep -v "^n=" gpurun_out/search_r02s.log
