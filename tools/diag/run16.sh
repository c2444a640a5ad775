set -x
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo b=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-peaks --no-fp64-baseline --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_bf16.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_class -c 1 -o gpurun_out/prof_cfg3_bf16m python bench.py $ARGS > gpurun_out/ncu_bf16.log 2>&1; echo ncu=$?
