set -x
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mxf4_probe mxf4_probe.cu && timeout 60 ./mxf4_probe > ../../gpurun_out/mxf4_probe.log 2>&1; echo probe=$?; cd ../..
ARGS="--steps 1 --warmup 0 --no-e2e --no-peaks --no-fp64-baseline --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
