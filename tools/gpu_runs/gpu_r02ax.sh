# complex64: precompiled cubins vs the same kernels compiled on the box (empty cache), alternating
for rep in 1 2; do
  echo "== c64 precompiled" >> gpurun_out/probe_ax.log
  timeout 600 python tools/pass_probe.py cfg4 1024 c64 2>&1 | grep onchip >> gpurun_out/probe_ax.log
  rm -rf /tmp/hqc_empty; mkdir -p /tmp/hqc_empty
  echo "== c64 box-compiled" >> gpurun_out/probe_ax.log
  HQ_JIT_CACHE=/tmp/hqc_empty timeout 900 python tools/pass_probe.py cfg4 1024 c64 2>&1 | grep onchip >> gpurun_out/probe_ax.log
done
ls -la /tmp/hqc_empty | head -3 >> gpurun_out/probe_ax.log
md5sum /tmp/hqc_empty/*.cubin | sort > gpurun_out/box_md5.txt
