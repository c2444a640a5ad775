set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_loopback.py -x -q -k "mx4 or mxfp4" > gpurun_out/mx_tests.log 2>&1; echo t=$?
timeout 900 python bench.py --config 4 --variant mx4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline > gpurun_out/bench_cfg4_mx4.log 2>&1; echo b1=$?
