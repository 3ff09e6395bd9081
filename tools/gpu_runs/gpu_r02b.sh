set -x
export PARITY_LOG=gpurun_out/parity_r02b.jsonl
rm -f $PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gputest_r02b.log
timeout 1200 python tools/cfg5_sharded.py > gpurun_out/cfg5_r02b.json 2> gpurun_out/cfg5_r02b.err
tail -3 gpurun_out/gputest_r02b.log
