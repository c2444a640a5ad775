A="--config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
for r in 1 2; do
timeout 600 python bench.py $A > gpurun_out/c4_def_$r.log 2>&1
timeout 600 python bench.py $A --flags 32 > gpurun_out/c4_pair_$r.log 2>&1
done
