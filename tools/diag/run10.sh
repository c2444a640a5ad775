A="--config 4 --variant mx4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
timeout 600 python bench.py $A > gpurun_out/plain_mx.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mx -c 1 -o gpurun_out/prof_kmx python bench.py $A > gpurun_out/ncu_kmx.log 2>&1; echo ncu=$?
