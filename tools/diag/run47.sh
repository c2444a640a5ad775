# SM-pair kernel (GMP_FLAG_TC_PAIR = 32) vs default at cfg3 with the final code: class times
for rep in 1 2; do
  for fl in 0 32; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline --flags $fl 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('flags $fl', round(d['value'],1), 'cls', [round(x,1) for x in d['class_ms_rank0'][1:4]], 'mhz', d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'), 'launches', d.get('gpu_launches_per_step'))" >> gpurun_out/pair_ab_final.log 2>&1
  done
done
