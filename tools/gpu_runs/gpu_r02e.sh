# complex128 occupancy / tile knobs on the cfg4 plan (pass_probe: one forward+adjoint, B=1024)
for kv in "X=0" "HQ_TILE_BITS=10" "HQ_REG_ACC=0" "HQ_REG_ACC=16" "HQ_BWD_MINB=3" "HQ_FWD_MINB=4" "HQ_MAX_PASS_OPS=100"; do
  echo "== $kv"
  env $kv timeout 600 python tools/pass_probe.py cfg4 1024 c128 2>&1 | tail -2
done > gpurun_out/knobs_c128_r02e.log 2>&1
cat gpurun_out/knobs_c128_r02e.log
python tools/pass_probe.py cfg4 128 c128 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(b2|f2|b0)$" -c 3 \
    -o gpurun_out/ncu_c128_r02e python tools/pass_probe.py cfg4 128 c128 > gpurun_out/ncu_c128_r02e.log 2>&1
echo ncu rc=$?
