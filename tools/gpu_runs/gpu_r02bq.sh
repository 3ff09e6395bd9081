# complex128 with 2 fixed tile bits (6 passes on cfg4): GPU suite, bench, cfg5 one GPU, launch list
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_bq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bq.log
timeout 900 python bench.py > gpurun_out/bench_bq.json 2> gpurun_out/bench_bq.err
timeout 600 python tools/cfg5_single_gpu.py > gpurun_out/cfg5_1gpu_bq.jsonl 2>&1
timeout 900 python tools/cfg5_single_gpu.py --grad >> gpurun_out/cfg5_1gpu_bq.jsonl 2>&1
python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu > gpurun_out/plain_bench_bq.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv \
    --log-file gpurun_out/launches_bq.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-companion --no-cpu \
    > gpurun_out/ncu_launches_bq.log 2>&1
echo "ncu rc=$?"
