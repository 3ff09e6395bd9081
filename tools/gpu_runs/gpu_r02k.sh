# robustness sweep of the planner / generator options, then the bench launch list
timeout 1200 python tools/fuzz_parity.py 60 77 > gpurun_out/fuzz_default_r02k.txt 2>&1
HQ_SHFL=1 timeout 900 python tools/fuzz_parity.py 30 78 > gpurun_out/fuzz_shfl_r02k.txt 2>&1
HQ_PINGPONG=1 timeout 900 python tools/fuzz_parity.py 30 79 > gpurun_out/fuzz_pp_r02k.txt 2>&1
tail -2 gpurun_out/fuzz_*_r02k.txt
python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv \
    --log-file gpurun_out/launches_r02k.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu \
    > gpurun_out/ncu_launches_r02k.log 2>&1
echo "ncu rc=$?"
