# host-bound configs re-run (cfg1 / cfg2 / QAE were slower in bi: host speed?)
nproc > gpurun_out/host_bj.txt; lscpu | grep -E "Model name|MHz" >> gpurun_out/host_bj.txt
timeout 900 python tools/bench_all.py > gpurun_out/all_configs_bj.jsonl 2> gpurun_out/all_configs_bj.err
timeout 600 python tools/qae_bench.py > gpurun_out/qae_bj.jsonl 2>&1
