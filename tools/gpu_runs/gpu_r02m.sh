# round-2 refresh of every config's throughput (one GPU)
timeout 900 python tools/bench_all.py > gpurun_out/all_configs_r02m.jsonl 2> gpurun_out/all_configs_r02m.err
timeout 600 python tools/cfg5_single_gpu.py > gpurun_out/cfg5_1gpu_r02m.jsonl 2>&1
timeout 900 python tools/cfg5_single_gpu.py --grad >> gpurun_out/cfg5_1gpu_r02m.jsonl 2>&1
timeout 600 python tools/qae_bench.py > gpurun_out/qae_r02m.jsonl 2>&1
timeout 600 python tools/hybrid_cnn.py > gpurun_out/hybrid_r02m.json 2>&1
cat gpurun_out/all_configs_r02m.jsonl gpurun_out/cfg5_1gpu_r02m.jsonl | cut -c1-300
