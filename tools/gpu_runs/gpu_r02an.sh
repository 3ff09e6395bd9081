# complex64 pass kernels: one full capture (first backward, a middle backward, a forward)
python tools/pass_probe.py cfg4 256 c64 > gpurun_out/plain_probe_an.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(b0|b2|f2)$" -c 3 \
    -o gpurun_out/ncu_c64_an python tools/pass_probe.py cfg4 256 c64 > gpurun_out/ncu_c64_an.log 2>&1
echo "ncu rc=$?"
