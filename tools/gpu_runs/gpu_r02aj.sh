# bench with the split complex128 forward kernels, its launch list, and a full capture of one forward kernel
timeout 900 python bench.py > gpurun_out/bench_aj.json 2> gpurun_out/bench_aj.err
python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu > gpurun_out/plain_bench_aj.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv \
    --log-file gpurun_out/launches_aj.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu \
    > gpurun_out/ncu_launches_aj.log 2>&1
python tools/pass_probe.py cfg4 128 c128 > gpurun_out/plain_probe_aj.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(f2|b2)$" -c 2 \
    -o gpurun_out/ncu_c128_aj python tools/pass_probe.py cfg4 128 c128 > gpurun_out/ncu_c128_aj.log 2>&1
echo "ncu rc=$?"
