# defaults after the one-compiler re-measurement: GPU suite, bench, launch list
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_bc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bc.log
timeout 900 python bench.py > gpurun_out/bench_bc.json 2> gpurun_out/bench_bc.err
python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu > gpurun_out/plain_bench_bc.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv \
    --log-file gpurun_out/launches_bc.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu \
    > gpurun_out/ncu_launches_bc.log 2>&1
echo "ncu rc=$?"
