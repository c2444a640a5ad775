timeout 1500 python tools/paper_sweep.py --out gpurun_out/paper_sweep_r02 > gpurun_out/paper_sweep_r02.log 2>&1; echo ps=$?
