export PARITY_LOG=gpurun_out/parity_r02q.jsonl
rm -f $PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gputest_r02q.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02q.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r02q.log
timeout 900 python bench.py > gpurun_out/bench_r02q.json 2> gpurun_out/bench_r02q.err
cat gpurun_out/gputest_r02q.log gpurun_out/smoke_r02q.log
