cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/v_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/v_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/v_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/v_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/v_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err
echo "bench rc=$?" >> gpurun_out/v_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err
echo "ref rc=$?" >> gpurun_out/v_ref.err
