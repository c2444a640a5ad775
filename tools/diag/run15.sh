set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_fin.log 2>&1; echo all=$?
A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
timeout 600 python bench.py $A > gpurun_out/ab_fin_1.log 2>&1
ARGS="--steps 1 --warmup 0 --no-e2e --no-peaks --no-fp64-baseline --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
