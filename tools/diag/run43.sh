# leaner k_tile_stats (pointer walk, integer maxabs) + batched k_c_finalize loads: GPU tests, cfg3 A/B
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_stats.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_stats.log
for rep in 1 2; do
  for lib in exp/libgemm_mp_head.so paper_2508_14848_b200/libgemm_mp.so; do
GMP_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['value'],1), 'plan', [s[0] for s in d['steps_ms']], 'conv', {k: round(v,2) for k,v in d['convert_ms_rank0'].items()}, 'fin', round(d['exec_other_ms_rank0']['finalize'],2), d['clocks']['sm_mhz'])" >> gpurun_out/stats_ab.log 2>&1
  done
done
