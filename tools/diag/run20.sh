TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 2 --master-port 29562 bench.py --gpus 2 > gpurun_out/full_n2.log 2>&1; echo n2=$?
timeout 1500 $TR --nproc-per-node 4 --master-port 29561 bench.py --gpus 4 > gpurun_out/full_n4.log 2>&1; echo n4=$?
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_ce.log 2>&1; echo multi=$?
