set -x
timeout 900 python bench.py --config 4 --variant mx4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_mx4.log 2>&1; echo b1=$?
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline > gpurun_out/bench_cfg4.log 2>&1; echo b2=$?
