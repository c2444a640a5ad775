A="--steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 1 2 3; do
GMP_STEP_LOG=1 timeout 900 $TR --master-port 2954$r bench.py --gpus 4 $A > gpurun_out/ce_rep_$r.log 2>&1; echo ce=$?
done
