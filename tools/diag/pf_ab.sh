# same-box A/B of the tcgen05 producer's L2 prefetch distance (GMP_TC_PF K blocks; 0 = off)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for pf in 0 8 16 4; do
    for cfg in 3 4; do
      GMP_TC_PF=$pf timeout 400 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline --steps 3 --warmup 2 2>/dev/null > gpurun_out/pf_${cfg}_${pf}_${rep}.json
      python -c "
import json,sys
d=json.loads(open('gpurun_out/pf_${cfg}_${pf}_${rep}.json').read().strip().splitlines()[-1])
print('cfg$cfg pf=$pf rep$rep', round(d['value'],1), 'phases', {k: round(v,1) for k,v in d['phases_ms'].items()}, 'class_ms', [round(x,1) for x in d['class_ms_rank0']], 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w_median'))" >> gpurun_out/pf_ab.txt 2>&1
    done
  done
done
cat gpurun_out/pf_ab.txt
