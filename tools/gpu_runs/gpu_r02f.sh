# branch / deferral knobs (pass_probe: one forward+adjoint of cfg4, B=1024)
for pr in c128 c64; do
for kv in "X=0" "HQ_UBRANCH_BWD=1" "HQ_UBRANCH_BWD=2" "HQ_UBRANCH=0" "HQ_UBRANCH=1" "HQ_DEFER_PARTIAL=0" "HQ_DEFER_PARTIAL=4" "HQ_DEFER_RZ=0"; do
  echo "== $pr $kv"
  env $kv timeout 600 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -1
done
done > gpurun_out/knobs2_r02f.log 2>&1
cat gpurun_out/knobs2_r02f.log
