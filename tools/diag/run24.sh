A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
for r in 1 2; do
timeout 600 python bench.py $A > gpurun_out/ab_def_$r.log 2>&1
timeout 600 python bench.py $A --flags 64 > gpurun_out/ab_mc_$r.log 2>&1
done
