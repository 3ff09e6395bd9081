nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_occ tools/dfma_occupancy.cu && /tmp/dfma_occ > gpurun_out/dfma_occ.log 2>&1
cat gpurun_out/dfma_occ.log
export HQ_PINGPONG=1
python tools/pass_probe.py cfg4 128 c128 > gpurun_out/plain_pp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_b2$" -c 1 \
    -o gpurun_out/ncu_pp_r02l python tools/pass_probe.py cfg4 128 c128 > gpurun_out/ncu_pp_r02l.log 2>&1
echo "ncu rc=$?"
