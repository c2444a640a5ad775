timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_fz.log 2>&1; echo all=$?
