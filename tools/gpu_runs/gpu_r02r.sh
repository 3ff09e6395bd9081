# first-pass-only op cap (code size of the largest pass kernels)
for pr in c64 c128; do
  for v in 0 120 90 100; do
    echo "== $pr HQ_FIRST_PASS_OPS=$v"
    if [ $v = 0 ]; then timeout 300 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -1;
    else HQ_FIRST_PASS_OPS=$v timeout 300 python tools/pass_probe.py cfg4 1024 $pr 2>&1 | tail -1; fi
  done
done > gpurun_out/firstpass_r02r.log 2>&1
cat gpurun_out/firstpass_r02r.log
