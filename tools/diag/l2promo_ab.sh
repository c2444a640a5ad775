# same-box A/B of the class arenas' TMA L2 promotion (GMP_TC_L2PROMO: 0 none, 2 128 B, 3 256 B)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for pr in 3 0 2; do
    for cfg in 3 4; do
      GMP_TC_L2PROMO=$pr timeout 400 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline --steps 3 --warmup 2 2>/dev/null > gpurun_out/l2p_${cfg}_${pr}_${rep}.json
      python -c "
import json,sys
d=json.loads(open('gpurun_out/l2p_${cfg}_${pr}_${rep}.json').read().strip().splitlines()[-1])
print('cfg$cfg promo=$pr rep$rep', round(d['value'],1), 'phases', {k: round(v,1) for k,v in d['phases_ms'].items()}, 'class_ms', [round(x,1) for x in d['class_ms_rank0']], 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w_median'))" >> gpurun_out/l2p_ab.txt 2>&1
    done
  done
done
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
for pr in 3 0; do
GMP_TC_L2PROMO=$pr timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_tc_class --csv --log-file gpurun_out/l2p_ncu_$pr.csv python bench.py $ARGS > /dev/null 2>&1
done
cat gpurun_out/l2p_ab.txt
