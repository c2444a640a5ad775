# 4 GPUs at HEAD: multi-rank parity tests, then cfg3 N=4 bench line (default flags)
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_gpu_multi_r02_final4.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_multi_r02_final4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 > gpurun_out/final_cfg3_n4.json 2> gpurun_out/final_cfg3_n4.err; echo bench=$?
