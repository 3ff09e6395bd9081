# complex128 kernels: NVRTC 12.9 (toolkit, default) vs 12.8 (torch wheel), separate processes alternating
W=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_nvrtc/lib/libnvrtc.so.12
for rep in 1 2; do
  echo "== c128 nvrtc 12.9" >> gpurun_out/probe_bd.log
  timeout 600 python tools/pass_probe.py cfg4 1024 c128 2>&1 | grep onchip >> gpurun_out/probe_bd.log
  echo "== c128 nvrtc 12.8" >> gpurun_out/probe_bd.log
  HQ_NVRTC=$W timeout 900 python tools/pass_probe.py cfg4 1024 c128 2>&1 | grep onchip >> gpurun_out/probe_bd.log
done
