# same-box A/B of bench.py variants (device leg only): ARGS_A vs ARGS_B, REPS times
for rep in $(seq ${REPS:-2}); do
  for v in "$ARGS_A" "$ARGS_B"; do
    python bench.py --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline --steps 3 --warmup 2 $v 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', round(d['value'],1), 'phases', {k: round(v,1) for k,v in d['phases_ms'].items()}, 'class_ms', [round(x,1) for x in d['class_ms_rank0']], 'mhz', d['clocks']['sm_mhz'])"
  done
done
