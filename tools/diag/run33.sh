TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --ownership balanced > gpurun_out/full_n4_bal.log 2>&1; echo b=$?
