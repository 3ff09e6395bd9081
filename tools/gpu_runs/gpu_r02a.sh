set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PARITY_LOG=gpurun_out/parity_r02a.jsonl
rm -f $PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/gputest_r02a.log
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02a.json 2>&1
tail -3 gpurun_out/gputest_r02a.log
