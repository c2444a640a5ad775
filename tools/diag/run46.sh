# W evict_first L2 policy (default build) vs plain W accesses (-DGMP_W_EVICT_NORMAL) at cfg3, device leg
for rep in 1 2 3; do
  for lib in exp/libgemm_mp_wnormal.so paper_2508_14848_b200/libgemm_mp.so; do
GMP_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['value'],1), 'cls', [round(x,1) for x in d['class_ms_rank0'][1:4]], 'fin', round(d['exec_other_ms_rank0']['finalize'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))" >> gpurun_out/wpol_ab.log 2>&1
  done
done
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
GMP_LIB_PATH=$PWD/exp/libgemm_mp_wnormal.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tc_class --csv --log-file gpurun_out/wpol_normal.csv python bench.py $ARGS > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tc_class --csv --log-file gpurun_out/wpol_first.csv python bench.py $ARGS > /dev/null 2>&1
