timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_ce2.log 2>&1; echo multi=$?
A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29571 bench.py --gpus 4 $A > gpurun_out/ce_n4_final.log 2>&1; echo ce=$?
