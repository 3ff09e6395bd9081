# refresh every config after the barrier-light transitions (one GPU)
timeout 900 python tools/bench_all.py > gpurun_out/all_configs_ac.jsonl 2> gpurun_out/all_configs_ac.err
timeout 600 python tools/cfg5_single_gpu.py > gpurun_out/cfg5_1gpu_ac.jsonl 2>&1
timeout 900 python tools/cfg5_single_gpu.py --grad >> gpurun_out/cfg5_1gpu_ac.jsonl 2>&1
timeout 1500 python tools/cfg5_sharded.py > gpurun_out/cfg5_virtual8_ac.json 2> gpurun_out/cfg5_virtual8_ac.err
timeout 600 python tools/qae_bench.py > gpurun_out/qae_ac.jsonl 2>&1
