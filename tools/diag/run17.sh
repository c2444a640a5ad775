set -x
nvidia-smi --query-gpu=index,name,clocks.sm,power.limit --format=csv
A="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
timeout 900 python bench.py --gpus 1 $A > gpurun_out/scale_n1.log 2>&1; echo n1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 $A > gpurun_out/scale_n2.log 2>&1; echo n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 $A > gpurun_out/scale_n4.log 2>&1; echo n4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 $A --config 4 > gpurun_out/scale_cfg4_n4.log 2>&1; echo c4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 $A --config 4 --variant mx4 > gpurun_out/scale_cfg4mx_n4.log 2>&1; echo c4m=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus 4 $A --sender > gpurun_out/scale_n4_sender.log 2>&1; echo n4s=$?
