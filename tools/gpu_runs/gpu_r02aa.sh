# warp-group transitions: bench, its launch list, one full capture of the c128 pass kernels
timeout 900 python bench.py > gpurun_out/bench_aa.json 2> gpurun_out/bench_aa.err
python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu > gpurun_out/plain_bench_aa.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv \
    --log-file gpurun_out/launches_aa.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu \
    > gpurun_out/ncu_launches_aa.log 2>&1
python tools/pass_probe.py cfg4 128 c128 > gpurun_out/plain_probe_aa.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(b2|f2|b0)$" -c 3 \
    -o gpurun_out/ncu_c128_aa python tools/pass_probe.py cfg4 128 c128 > gpurun_out/ncu_c128_aa.log 2>&1
echo "ncu rc=$?"
