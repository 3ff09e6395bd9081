# first-pass cap re-checked with the barrier-light transitions and 4-bit forward windows (interleaved A/B)
timeout 2000 python tools/ab_probe.py cfg4 1024 c128 "-" "HQ_PLAN_SEARCH=0" "HQ_FIRST_PASS_OPS=130" "HQ_FIRST_PASS_OPS=112" "HQ_FIRST_PASS_OPS=105" 3 >> gpurun_out/ab_al.log 2>&1
