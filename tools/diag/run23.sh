set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_sw.log 2>&1; echo all=$?
A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
for r in 1 2; do
timeout 600 python bench.py $A > gpurun_out/ab_w256_$r.log 2>&1
timeout 600 python bench.py $A --flags 16384 > gpurun_out/ab_w128_$r.log 2>&1
done
