for kv in "X=0" "HQ_FWD_MINB=3" "HQ_NO_DROP=1" "HQ_FWD_MINB=3 HQ_NO_DROP=1"; do
  echo "== $kv"; env $kv timeout 600 python tools/qae_bench.py 2>&1 | cut -c1-200
done > gpurun_out/qae_knobs_r02n.log 2>&1
cat gpurun_out/qae_knobs_r02n.log
