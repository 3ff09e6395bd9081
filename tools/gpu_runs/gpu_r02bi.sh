# every config with the final kernels
timeout 900 python tools/bench_all.py > gpurun_out/all_configs_bi.jsonl 2> gpurun_out/all_configs_bi.err
timeout 600 python tools/qae_bench.py > gpurun_out/qae_bi.jsonl 2>&1
timeout 900 python tools/cfg5_single_gpu.py --grad > gpurun_out/cfg5_1gpu_bi.jsonl 2>&1
