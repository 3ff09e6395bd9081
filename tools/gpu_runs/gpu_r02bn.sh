# cfg5 forward+adjoint: schedule search forced on long plans, dot chains 4 vs 2
for v in "HQ_PLAN_SEARCH=1" "HQ_PLAN_SEARCH=2" "HQ_DOT_CHAINS=4" "HQ_PLAN_SEARCH=2 HQ_DOT_CHAINS=4"; do
  echo "== $v" >> gpurun_out/cfg5_bn.log
  env $v timeout 900 python tools/cfg5_single_gpu.py --grad 2>&1 | cut -c1-260 >> gpurun_out/cfg5_bn.log
done
