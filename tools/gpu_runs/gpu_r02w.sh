# warp-local transitions (complex128 default): GPU suite, bench, ncu of the c128 pass kernels
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_w.log
timeout 900 python bench.py > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err
python tools/pass_probe.py cfg4 128 c128 > gpurun_out/plain_probe_w.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hq_(b2|f2|b0)$" -c 3 \
    -o gpurun_out/ncu_c128_w python tools/pass_probe.py cfg4 128 c128 > gpurun_out/ncu_c128_w.log 2>&1
echo "ncu rc=$?"
