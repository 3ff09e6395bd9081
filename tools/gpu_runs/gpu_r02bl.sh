# complex64 pass kernels with the final defaults (warp-group transitions, 2 dot chains): one full capture
python tools/pass_probe.py cfg4 256 c64 > gpurun_out/plain_probe_bl.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(b0|b2|f2)$" -c 3 \
    -o gpurun_out/ncu_c64_bl python tools/pass_probe.py cfg4 256 c64 > gpurun_out/ncu_c64_bl.log 2>&1
echo "ncu rc=$?"
