# shared diagonal derivative dots: parity (RZ/CR-heavy random circuits) and timing; FSEL ablation
export FUZZ_KINDS=RZ,RZ,RZ,CR,CR,RY,RX,CNOT,CZ,H
timeout 900 python tools/fuzz_parity.py 30 77 > gpurun_out/fuzz_diag_u.txt 2>&1
unset FUZZ_KINDS
timeout 600 python tools/fuzz_parity.py 20 5 >> gpurun_out/fuzz_diag_u.txt 2>&1
for v in "HQ_DIAG_DOTS=0" "HQ_DIAG_DOTS=1" "HQ_ABLATE=8"; do
  echo "== $v" >> gpurun_out/probe_u.log
  env $v timeout 600 python tools/pass_probe.py cfg4 1024 c128 >> gpurun_out/probe_u.log 2>&1
done
