timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_rm.log 2>&1; echo all=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
