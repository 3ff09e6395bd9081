# final-state validation: smoke, GPU suite, bench (N=1), the torchrun launch path at one rank
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_aq.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_aq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_aq.log
timeout 900 python bench.py > gpurun_out/bench_aq.json 2> gpurun_out/bench_aq.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 3 --warmup 3 --no-companion > gpurun_out/bench_torchrun_aq.json 2> gpurun_out/bench_torchrun_aq.err
