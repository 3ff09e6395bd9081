# c128 cfg4 backward-pass ablations: upper bounds of what removing window
# transitions (1), gate math (2) or derivative dots (4) would save
for ab in 0 1 2 4; do
  echo "== HQ_ABLATE=$ab"
  HQ_ABLATE=$ab timeout 600 python tools/pass_probe.py cfg4 1024 c128 2>&1 | tail -1
done > gpurun_out/ablate_c128_r02c.log 2>&1
for ab in 0 1; do
  echo "== c64 HQ_ABLATE=$ab"
  HQ_ABLATE=$ab timeout 600 python tools/pass_probe.py cfg4 1024 c64 2>&1 | tail -1
done >> gpurun_out/ablate_c128_r02c.log 2>&1
cat gpurun_out/ablate_c128_r02c.log
