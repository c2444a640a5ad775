# cfg4 (E4M3 on, tol 1e-2) at 4 GPUs and 1 GPU with the round-2 code
A="--config 4 --steps 5 --warmup 3 --no-cpu-baseline"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 $A > gpurun_out/cfg4_n4.json 2> gpurun_out/cfg4_n4.err
timeout 600 python bench.py $A > gpurun_out/cfg4_n1.json 2> gpurun_out/cfg4_n1.err
