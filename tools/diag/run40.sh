# 2-GPU: multi-rank parity tests at HEAD, then cfg4 N=1 with the pure-FP16 comparison leg
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_gpu_multi_r02_final.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_multi_r02_final.log
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg4_n1_fp16leg.json 2> gpurun_out/cfg4_n1_fp16leg.err; echo bench=$?
