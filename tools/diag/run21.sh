set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_dyn.log 2>&1; echo all=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
for r in 1 2; do
timeout 600 python bench.py $A > gpurun_out/ab_dyn_$r.log 2>&1
timeout 600 python bench.py $A --flags 8192 > gpurun_out/ab_sta_$r.log 2>&1
done
ARGS="--steps 1 --warmup 0 --no-e2e --no-peaks --no-fp64-baseline --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/plain_bf16.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:k_tc_class -c 1 -o gpurun_out/prof_cfg3_dyn python bench.py $ARGS > gpurun_out/ncu_dyn.log 2>&1; echo ncu=$?
