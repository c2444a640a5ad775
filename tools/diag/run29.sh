A="--steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 $A > gpurun_out/own_auto4.log 2>&1; echo a=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 $A > gpurun_out/own_auto2.log 2>&1; echo b=$?
