export PARITY_LOG=gpurun_out/parity_r02j.jsonl
rm -f $PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gputest_r02j.log
timeout 900 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err
cat gpurun_out/gputest_r02j.log
