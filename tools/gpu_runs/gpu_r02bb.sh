# complex64 knobs re-measured with one compiler (round-1 decisions were confounded by NVRTC 12.8 vs 12.9)
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_UBRANCH=0" "HQ_UBRANCH=3" "HQ_FWD_MINB=3" "HQ_BWD_MINB=1" "HQ_TILE_BITS=11" 3 >> gpurun_out/ab_bb.log 2>&1
timeout 2400 python tools/ab_probe.py cfg4 1024 c64 "-" "HQ_TILE_BITS=13" "HQ_REG_BITS=3" "HQ_DEFER_RZ=0" 3 >> gpurun_out/ab_bb.log 2>&1
timeout 2400 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_DOT_CHAINS=2" "HQ_FWD_MINB=3" "HQ_SHEAR_FLUSH=1" 3 >> gpurun_out/ab_bb.log 2>&1
