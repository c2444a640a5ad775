cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_loopback.py -x -q > gpurun_out/v4_pytest_multi.log 2>&1
echo "rc=$?" >> gpurun_out/v4_pytest_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 > gpurun_out/v4_bench.json 2> gpurun_out/v4_bench.err
echo "bench rc=$?" >> gpurun_out/v4_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --ownership balanced --no-e2e > gpurun_out/v4_bench_bal.json 2> gpurun_out/v4_bench_bal.err
echo "bench rc=$?" >> gpurun_out/v4_bench_bal.err
