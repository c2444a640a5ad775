set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -k "mx4 or mxfp4" > gpurun_out/mx_tests.log 2>&1; echo t=$?
A="--config 4 --variant mx4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
for r in 1 2; do
timeout 600 python bench.py $A > gpurun_out/ab_st6_$r.log 2>&1
GMP_LIB_PATH=$PWD/exp/libgemm_mp_mx4st.so timeout 600 python bench.py $A > gpurun_out/ab_st4_$r.log 2>&1
done
