# round-2 final evidence: default bench (cfg3, N=1), cfg2 bench, then the cfg3 ncu launch list
timeout 600 python bench.py > gpurun_out/final_cfg3_n1.json 2> gpurun_out/final_cfg3_n1.err; echo bench=$?
timeout 600 python bench.py --config 2 > gpurun_out/final_cfg2_n1.json 2> gpurun_out/final_cfg2_n1.err; echo bench2=$?
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3_final.csv python bench.py $ARGS > gpurun_out/ncu_launch_final.log 2>&1; echo ncu=$?
