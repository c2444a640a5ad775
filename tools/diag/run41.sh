# vectorised k_shadow_t: GPU tests, then cfg3 convert breakdown (2 runs)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_shadowt.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_shadowt.log
for rep in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), d['convert_ms_rank0'], d['exec_other_ms_rank0'], [s for s in d['steps_ms']], d['clocks']['sm_mhz'])" >> gpurun_out/shadowt_ab.log 2>&1
done
