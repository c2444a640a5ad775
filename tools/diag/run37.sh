# k_dmma shape A/B at cfg2 (mbarrier hand-off): 128x64 ST4 (default), 128x128 16 warps ST6 / ST5, 128x64 ST3
A="--config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks"
for rep in 1 2; do
  for lib in paper_2508_14848_b200/libgemm_mp.so exp/libgemm_mp_dmma_w4s6.so exp/libgemm_mp_dmma_w4s5.so exp/libgemm_mp_dmma_st3.so; do
    GMP_LIB_PATH=$PWD/$lib timeout 600 python bench.py $A 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['value'],2), 'cls_ms', [round(x,2) for x in d['class_ms_rank0'][:3]], 'allfp64', round(d['all_fp64']['value'],2), 'mhz', d['clocks']['sm_mhz'], 'roof', round(d['roofline']['frac'],4))" >> gpurun_out/dmma_ab3.log 2>&1
  done
done
