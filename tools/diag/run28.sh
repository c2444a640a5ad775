A="--steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks --no-fp64-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for r in 1 2; do
timeout 900 $TR --master-port 2958$r bench.py --gpus 4 $A > gpurun_out/bal_cyc_$r.log 2>&1; echo c=$?
timeout 900 $TR --master-port 2959$r bench.py --gpus 4 $A --balance > gpurun_out/bal_bal_$r.log 2>&1; echo b=$?
done
