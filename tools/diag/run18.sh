set -x
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_ce.log 2>&1; echo multi=$?
A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 1 2; do
timeout 900 $TR --master-port 2952$r bench.py --gpus 4 $A > gpurun_out/ab_ce_$r.log 2>&1; echo ce=$?
timeout 900 $TR --master-port 2953$r bench.py --gpus 4 $A --flags 4096 > gpurun_out/ab_nccl_$r.log 2>&1; echo nccl=$?
done
