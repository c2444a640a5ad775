# same-box A/B at cfg4 (E4M3-dominant): 1-SM k_tc_class (default) vs SM-pair k_tc2_class (GMP_FLAG_TC_PAIR = 32)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2 3; do
  for fl in 0 32; do
    timeout 400 python bench.py --config 4 --flags $fl --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline --steps 3 --warmup 2 2>/dev/null > gpurun_out/p8_${fl}_${rep}.json
    python -c "
import json,sys
d=json.loads(open('gpurun_out/p8_${fl}_${rep}.json').read().strip().splitlines()[-1])
print('cfg4 flags=$fl rep$rep', round(d['value'],1), 'phases', {k: round(v,1) for k,v in d['phases_ms'].items()}, 'class_ms', [round(x,1) for x in d['class_ms_rank0']], 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w_median'))" >> gpurun_out/p8_ab.txt 2>&1
  done
done
cat gpurun_out/p8_ab.txt
