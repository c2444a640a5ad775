set -x
timeout 600 python -m pytest tests/test_gpu_edges.py -x -q -k "mxfp4" > gpurun_out/mx_edges.log 2>&1; echo edges=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mx4" > gpurun_out/mx_parity.log 2>&1; echo parity=$?
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -k "mx4" > gpurun_out/mx_loop.log 2>&1; echo loop=$?
