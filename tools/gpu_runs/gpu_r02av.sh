# batched dot reduction: partials kept per warp (4 default / 2 / 1); separate processes, alternating
# (jit_layout reads HQ_DOT_GROUP at launch too, so ab_probe's per-plan env cannot vary it)
for rep in 1 2; do for v in "HQ_DOT_GROUP=4" "HQ_DOT_GROUP=2" "HQ_DOT_GROUP=1"; do
  echo "== $v" >> gpurun_out/probe_av.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c128 2>&1 | grep onchip >> gpurun_out/probe_av.log
done; done
