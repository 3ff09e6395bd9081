# NVRTC pinned to the toolkit's 12.9: box-compiled cubins must equal the precompiled ones
rm -rf /tmp/hqc_empty; mkdir -p /tmp/hqc_empty
echo "== c64 box-compiled (12.9 pinned)" >> gpurun_out/probe_ay.log
HQ_JIT_CACHE=/tmp/hqc_empty timeout 900 python tools/pass_probe.py cfg4 1024 c64 2>&1 | grep onchip >> gpurun_out/probe_ay.log
echo "== c64 precompiled" >> gpurun_out/probe_ay.log
timeout 600 python tools/pass_probe.py cfg4 1024 c64 2>&1 | grep onchip >> gpurun_out/probe_ay.log
md5sum /tmp/hqc_empty/*.cubin | sort > gpurun_out/box_md5_ay.txt
