# complex128 occupancy / tile variants under the barrier-light transitions (interleaved A/B)
timeout 1500 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_TILE_BITS=12" "HQ_BWD_MINB=3,HQ_REG_ACC=0" "HQ_REG_ACC=0" 4 >> gpurun_out/ab_ae.log 2>&1
