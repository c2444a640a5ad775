set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mx4" > gpurun_out/mx_parity.log 2>&1; echo parity=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo all=$?
