# debug: complex128 forward kernels with 4 register bits at tile 9 (one warp per tile)
T="tests/test_gpu_parity.py::test_random_layers_vs_oracle[c128-9-None]"
for v in "HQ_FWD_RB=0" "HQ_FWD_RB=1" "HQ_FWD_RB=0 HQ_REG_BITS=4" "HQ_WARP_SYNC=0" "HQ_UBRANCH=0" "HQ_DEFER_RZ=0" "HQ_NO_PERM=1" "HQ_NO_FOLD=1"; do
  echo "== $v" >> gpurun_out/dbg_ag.log
  env $v timeout 300 python -m pytest "$T" -x -q 2>&1 | grep -E "passed|failed|assert 0|Error" | head -3 >> gpurun_out/dbg_ag.log
done
