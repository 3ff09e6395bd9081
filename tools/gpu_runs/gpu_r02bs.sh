# final complex128 plan (6 passes, 2 fixed tile bits): one full capture of a forward, a backward and the first backward
python tools/pass_probe.py cfg4 128 c128 > gpurun_out/plain_probe_bs.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(b0|b2|f2)$" -c 3 \
    -o gpurun_out/ncu_c128_bs python tools/pass_probe.py cfg4 128 c128 > gpurun_out/ncu_c128_bs.log 2>&1
echo "ncu rc=$?"
