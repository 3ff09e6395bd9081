for v in "HQ_REG_BITS=3" "HQ_REG_BITS=4"; do echo "== $v"; env $v HQ_FWD_RB=0 timeout 300 python tools/dbg_rb4.py 9 2>&1 | tail -4; done > gpurun_out/dbg_ah.log
