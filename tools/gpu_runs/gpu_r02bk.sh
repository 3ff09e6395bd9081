# every config with the final kernels (latency-bound ones: 100 steps, median of 5)
timeout 1200 python tools/bench_all.py > gpurun_out/all_configs_bk.jsonl 2> gpurun_out/all_configs_bk.err
