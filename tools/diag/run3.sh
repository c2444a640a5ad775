# 4-GPU call: multi-GPU NCCL parity on HEAD (incl. NEXT-3 balanced owners), then cfg3 at N=4 block-cyclic vs balanced
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,power.limit --format=csv
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_r02.log 2>&1; echo multi=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
timeout 900 $TR bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_cfg3_n4_cyclic.log 2>&1; echo b1=$?
timeout 900 $TR bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-peaks --no-fp64-baseline --balance > gpurun_out/bench_cfg3_n4_balanced.log 2>&1; echo b2=$?
timeout 900 $TR bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-peaks --no-fp64-baseline > gpurun_out/bench_cfg3_n4_cyclic2.log 2>&1; echo b3=$?
timeout 900 $TR bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-peaks --no-fp64-baseline --balance > gpurun_out/bench_cfg3_n4_balanced2.log 2>&1; echo b4=$?
