# cfg5 with the final kernels: one GPU (forward, forward+adjoint) and 8 virtual ranks
timeout 600 python tools/cfg5_single_gpu.py > gpurun_out/cfg5_1gpu_bm.jsonl 2>&1
timeout 900 python tools/cfg5_single_gpu.py --grad >> gpurun_out/cfg5_1gpu_bm.jsonl 2>&1
timeout 1500 python tools/cfg5_sharded.py > gpurun_out/cfg5_virtual8_bm.json 2> gpurun_out/cfg5_virtual8_bm.err
