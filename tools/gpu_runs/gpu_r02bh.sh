# final build: smoke, GPU suite, bench (N=1)
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_bh.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_bh.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bh.log
timeout 900 python bench.py > gpurun_out/bench_bh.json 2> gpurun_out/bench_bh.err
