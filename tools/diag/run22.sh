timeout 2400 python tools/config_sweep.py --reps 3 > gpurun_out/config_sweep_r02.jsonl 2> gpurun_out/config_sweep_r02.err; echo sweep=$?
