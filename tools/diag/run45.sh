# final round-2 evidence at HEAD: smoke, GPU suite, default bench, reference arm
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo smoke=$? >> gpurun_out/smoke_final.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02_final.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_r02_final.log
timeout 600 python bench.py > gpurun_out/final2_cfg3_n1.json 2> gpurun_out/final2_cfg3_n1.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref=$?
