# last check on the final commit: smoke + GPU suite
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_bo.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_bo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bo.log
