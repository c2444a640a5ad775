#!/bin/bash
# Strong-scaling table on one box: bench.py --config c at N = 1, 2, 4 GPUs
# (no e2e, no CPU baseline), one JSON line per run into gpurun_out/scaling.jsonl.
out=gpurun_out/scaling.jsonl
: > $out
port=29700
for c in 2 3 4; do
  for n in 1 2 4; do
    port=$((port+1))
    if [ $n -eq 1 ]; then
      timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" >> $out
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $n --config $c --steps 3 --warmup 3 --no-e2e 2>/dev/null | grep "^{" >> $out
    fi
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/scaling.jsonl"):
    r = json.loads(l)
    print(r["config"]["workload"], r["n_gpus"], round(r["value"], 1), round(r["ms_per_step"], 2), r["phases_ms"],
          r.get("imbalance"), r["clocks"]["sm_mhz"], round(r["precision_mix_roofline"]["frac_of_step"], 3))
PY
