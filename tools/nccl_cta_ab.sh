#!/bin/bash
# A/B of the NCCL CTA budget of the SUMMA row/column communicators at 4 GPUs:
# default, GMP_NCCL_MAX_CTAS=4, GMP_NCCL_CTA_POLICY=2 (NCCL_CTA_POLICY_ZERO).
out=gpurun_out/nccl_cta_ab.jsonl
: > $out
port=29800
run() {  # $1 label, $2 config, rest: env assignments
  local label=$1 cfg=$2; shift 2
  port=$((port+1))
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --config $cfg --steps 5 --warmup 3 --no-e2e 2>/dev/null | grep "^{" | \
    python -c "import json,sys; r=json.loads(sys.stdin.read()); r['ab']='$label'; print(json.dumps(r))" >> $out
}
for rep in 1 2; do
  run default 2 X=0
  run maxctas4 2 GMP_NCCL_MAX_CTAS=4
  run policy_zero 2 GMP_NCCL_CTA_POLICY=2
done
run default 3 X=0
run maxctas4 3 GMP_NCCL_MAX_CTAS=4
run policy_zero 3 GMP_NCCL_CTA_POLICY=2
python - <<'PY'
import json
for l in open("gpurun_out/nccl_cta_ab.jsonl"):
    r = json.loads(l)
    print(r["ab"], r["config"]["workload"], round(r["value"], 1), round(r["ms_per_step"], 2), r["phases_ms"],
          r.get("imbalance"), r["clocks"]["sm_mhz"])
PY
