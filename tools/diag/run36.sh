# k_dmma mbarrier stage hand-off (default) vs the CTA-barrier ring (-DGMP_DMMA_SYNC) at cfg2, then the GPU tests
A="--config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks"
for rep in 1 2; do
  for lib in exp/libgemm_mp_dmma_sync.so paper_2508_14848_b200/libgemm_mp.so; do
    GMP_LIB_PATH=$PWD/$lib timeout 600 python bench.py $A 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['value'],2), 'fp64cls_ms', [round(x,2) for x in d['class_ms_rank0']], 'allfp64', d.get('all_fp64'), 'mhz', d['clocks']['sm_mhz'], 'roof', d['roofline']['frac'], d['roofline']['kernel'])" >> gpurun_out/dmma_ab2.log 2>&1
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_dmma2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_dmma2.log
