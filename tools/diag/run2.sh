set -x
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/pytest_loopback.log 2>&1; echo loop=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-peaks --no-fp64-baseline --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_bf16.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_class -c 1 -o gpurun_out/prof_cfg3_bf16 python bench.py $ARGS > gpurun_out/ncu_bf16.log 2>&1; echo ncu=$?
