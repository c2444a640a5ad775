A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
timeout 600 python bench.py $A > gpurun_out/gap_2.log 2>&1
